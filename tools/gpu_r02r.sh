mkdir -p gpurun_out
FMOE_PROFILE_RANGE=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
echo done
