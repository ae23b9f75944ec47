mkdir -p gpurun_out
O=gpurun_out/f32mm_unroll.log
M="python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 64 --k 8 --ell 16"
echo "--- unroll 2 (default)" > $O; timeout 300 $M >> $O 2>&1
for u in 1 4; do
  FMOE_NVCC_EXTRA=-DFMOE_F32MM_UNROLL=$u timeout 600 python paper_2502_05370_b200/build.py --force > gpurun_out/build_u$u.log 2>&1
  echo "--- unroll $u" >> $O; timeout 300 $M >> $O 2>&1
done
echo done
