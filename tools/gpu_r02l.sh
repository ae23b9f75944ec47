mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_full.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5_b.json 2> gpurun_out/bench_c5_b.err
timeout 600 python bench.py --config C2 > gpurun_out/bench_c2_b.json 2> gpurun_out/bench_c2_b.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5.log 2>&1
echo done
