mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_z.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5_z.json 2> gpurun_out/bench_c5_z.err
echo done
