mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5_final.json 2> gpurun_out/bench_c5_final.err
timeout 600 python bench.py --config C2 > gpurun_out/bench_c2_final.json 2> gpurun_out/bench_c2_final.err
FMOE_PROFILE_RANGE=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2_final.log 2>&1
FMOE_PROFILE_RANGE=1 timeout 1200 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5_final.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
