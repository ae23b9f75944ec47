mkdir -p gpurun_out
O=gpurun_out/sem_trace.log
timeout 600 python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 64 --k 8 --ell 16 > gpurun_out/f32mm_micro2.log 2>&1
M="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic"
echo "--- TN=256 NO_EPI" > gpurun_out/tiled_exp.log
FMOE_UMMA_TN=256 FMOE_NO_EPI=1 timeout 300 $M >> gpurun_out/tiled_exp.log 2>&1
echo "--- TN=256 NO_EPI TILED_B_EXP" >> gpurun_out/tiled_exp.log
FMOE_UMMA_TN=256 FMOE_NO_EPI=1 FMOE_TILED_B_EXP=1 timeout 300 $M >> gpurun_out/tiled_exp.log 2>&1
echo "--- TN=512 NO_EPI NO_A_RELOAD" >> gpurun_out/tiled_exp.log
FMOE_NO_EPI=1 FMOE_NO_A_RELOAD=1 timeout 300 $M >> gpurun_out/tiled_exp.log 2>&1
timeout 300 python tools/trace.py --mode sem --n 2000000 --D 4096 --B 256 --k 8 > $O 2>&1
FMOE_NVCC_EXTRA=-DFMOE_EPI_PROFILE timeout 600 python paper_2502_05370_b200/build.py --force > gpurun_out/build_prof.log 2>&1
timeout 300 python tools/trace.py --mode sem --n 2000000 --D 4096 --B 256 --k 8 >> $O 2>&1
echo done
