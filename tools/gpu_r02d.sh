# C5 semantic scan anatomy at the per-rank 2M shard, B = 256 (semantic_cos = the bench's call)
mkdir -p gpurun_out
M="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,blend_cos,semantic"
timeout 300 $M > gpurun_out/sem_anat.log 2>&1
echo "--- FMOE_NO_EPI=1" >> gpurun_out/sem_anat.log
FMOE_NO_EPI=1 timeout 300 $M >> gpurun_out/sem_anat.log 2>&1
echo "--- FMOE_FAKE_LOADS=1" >> gpurun_out/sem_anat.log
FMOE_FAKE_LOADS=1 timeout 300 $M >> gpurun_out/sem_anat.log 2>&1
echo "--- FMOE_FAKE_LOADS=1 FMOE_NO_EPI=1" >> gpurun_out/sem_anat.log
FMOE_FAKE_LOADS=1 FMOE_NO_EPI=1 timeout 300 $M >> gpurun_out/sem_anat.log 2>&1
echo "--- FMOE_UMMA_TN=256" >> gpurun_out/sem_anat.log
FMOE_UMMA_TN=256 timeout 300 $M >> gpurun_out/sem_anat.log 2>&1
echo "--- FMOE_NO_APPROX=1" >> gpurun_out/sem_anat.log
FMOE_NO_APPROX=1 timeout 300 $M >> gpurun_out/sem_anat.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:scan_umma -c 1 \
  -o gpurun_out/r02_sem_cos_2M python tools/batched_micro.py --n 2000000 --B 256 --k 8 --once --only semantic_cos \
  > gpurun_out/ncu_sem.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:scan_umma --launch-skip 2 -c 1 \
  -o gpurun_out/r02_blend_cos_2M python tools/batched_micro.py --n 2000000 --B 256 --k 8 --once --only semantic_cos,blend_cos \
  > gpurun_out/ncu_blend.log 2>&1
echo done
