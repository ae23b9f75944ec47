mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_v.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5_v.json 2> gpurun_out/bench_c5_v.err
timeout 600 python bench.py --config C2 > gpurun_out/bench_c2_v.json 2> gpurun_out/bench_c2_v.err
timeout 600 python bench.py --config C3 > gpurun_out/bench_c3_v.json 2> gpurun_out/bench_c3_v.err
timeout 600 python bench.py --config C4 > gpurun_out/bench_c4_v.json 2> gpurun_out/bench_c4_v.err
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:rowmajor -c 1 -o gpurun_out/r02_sweep_row_1M python tools/sweep_micro.py --n 1000000 --kernels row --reps 1 > gpurun_out/ncu_sweep.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:f32mm_kernel -c 1 -o gpurun_out/r02_f32mm_sem64 python tools/batched_micro.py --dtype f32 --n 1000000 --D 2048 --L 24 --E 60 --B 64 --k 8 --once --only semantic > gpurun_out/ncu_f32mm.log 2>&1
echo done
