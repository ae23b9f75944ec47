mkdir -p gpurun_out
timeout 300 python tools/sweep_micro.py --n 1000000,4000000 --kernels row,reg > gpurun_out/sweep_micro2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "sweep" > gpurun_out/gputest4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "sweep" >> gpurun_out/gputest4.log 2>&1
bash tools/gpu_r02d.sh
