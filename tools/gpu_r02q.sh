mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider -k "insert or rdy or resolve or victims or dist or two_ranks or nccl" > gpurun_out/gputest_resolve.log 2>&1
NCCL_DEBUG=INFO timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -p no:cacheprovider -k nccl -s > gpurun_out/nccl_info.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c5_r.json 2> gpurun_out/bench_c5_r.err
echo done
