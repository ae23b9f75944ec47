mkdir -p gpurun_out
M="python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 64 --k 8 --ell 16"
timeout 300 $M > gpurun_out/f32mm_final.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py -m gpu -q -p no:cacheprovider -k "f32 or setup0 or setup3 or mid3 or mid4" > gpurun_out/gputest_f32.log 2>&1
echo done
