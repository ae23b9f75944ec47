mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py -m gpu -q -x -p no:cacheprovider -k "batched or session or blend or semantic or merge or rdy or insert" > gpurun_out/gputest_merge.log 2>&1
timeout 600 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3_m.json 2> gpurun_out/bench_c3_m.err
FMOE_PROFILE_RANGE=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_m.csv python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3_m.log 2>&1
echo done
