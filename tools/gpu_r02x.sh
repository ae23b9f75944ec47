mkdir -p gpurun_out
O=gpurun_out/f32mm_2cta.log
M="python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 64 --k 8 --ell 16"
echo "--- 1 CTA/SM (default)" > $O; timeout 300 $M >> $O 2>&1
echo "--- 2 CTA/SM" >> $O; FMOE_F32MM_2CTA=1 timeout 300 $M >> $O 2>&1
FMOE_F32MM_2CTA=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "batched or blend_cos or semantic or trajectory" > gpurun_out/gputest_2cta.log 2>&1
echo done
