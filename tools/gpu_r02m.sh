mkdir -p gpurun_out
B="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,blend_cos"
O=gpurun_out/cos_bound.log
echo "--- COS_BOUND=1 (default)" > $O; timeout 300 $B >> $O 2>&1
echo "--- COS_BOUND=0" >> $O; FMOE_COS_BOUND=0 timeout 300 $B >> $O 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "blend or insert or rdy or batched" > gpurun_out/gputest_bound.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_midsize.py -m gpu -q -x -p no:cacheprovider -k "blend or rdy" >> gpurun_out/gputest_bound.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider >> gpurun_out/gputest_bound.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5_c.json 2> gpurun_out/bench_c5_c.err
FMOE_BENCH_DEVICE=0 FMOE_DIST_TRANSPORT=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C2 --steps 5 --warmup 3 > gpurun_out/bench_c2_2ranks.json 2> gpurun_out/bench_c2_2ranks.err
echo done
