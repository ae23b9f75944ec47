mkdir -p gpurun_out
timeout 300 python tools/sweep_micro.py --n 1000000,4000000 --kernels row,reg,tma > gpurun_out/sweep_micro.log 2>&1
timeout 600 python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 64 --k 8 --ell 16 > gpurun_out/f32mm_micro.log 2>&1
timeout 300 python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 8 --k 8 --ell 16 --only semantic,trajectory >> gpurun_out/f32mm_micro.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "sweep or batched or blend_cos or insert or semantic or trajectory" > gpurun_out/gputest2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_midsize.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider >> gpurun_out/gputest2.log 2>&1
echo done
