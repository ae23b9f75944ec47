mkdir -p gpurun_out
FMOE_NVCC_EXTRA=-DFMOE_EPI_PROFILE timeout 600 python paper_2502_05370_b200/build.py --force > gpurun_out/build_prof.log 2>&1
timeout 300 python tools/trace.py --mode blend_cos --ell 31 --n 2000000 --D 4096 --B 256 --k 8 > gpurun_out/blend_trace.log 2>&1
python paper_2502_05370_b200/build.py --force > gpurun_out/build_prof2.log 2>&1
# one pass of ncu metrics on the FULL C5 bench step (16M maps): dominant-kernel traffic and tensor-pipe activity
timeout 1500 /usr/local/cuda/bin/ncu --clock-control none -k regex:scan_umma -c 4 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/c5_ncu_metrics.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/c5_ncu_bench.log 2>&1
echo done
