mkdir -p gpurun_out
O=gpurun_out/sweep_chunk.log
echo "--- chunk 16" > $O; FMOE_SWEEP_CHUNK=16 timeout 300 python tools/sweep_micro.py --n 1000000,4000000 --kernels row >> $O 2>&1
echo "--- chunk 8" >> $O; FMOE_SWEEP_CHUNK=8 timeout 300 python tools/sweep_micro.py --n 1000000,4000000 --kernels row >> $O 2>&1
timeout 600 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
echo done
