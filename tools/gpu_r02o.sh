mkdir -p gpurun_out
B="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,blend_cos"
O=gpurun_out/cos_bound2.log
echo "--- COS_BOUND=1 (default)" > $O; timeout 300 $B >> $O 2>&1
echo "--- COS_BOUND=0" >> $O; FMOE_COS_BOUND=0 timeout 300 $B >> $O 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "blend or insert or rdy or batched or cos" > gpurun_out/gputest_bound2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_midsize.py -m gpu -q -x -p no:cacheprovider -k "blend or rdy" >> gpurun_out/gputest_bound2.log 2>&1
bash tools/gpu_r02n.sh
echo done
