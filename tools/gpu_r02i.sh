mkdir -p gpurun_out
B="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,blend_cos"
O=gpurun_out/cos_tiled.log
echo "--- base" > $O; timeout 300 $B >> $O 2>&1
echo "--- COS_TILED_EXP=1" >> $O; FMOE_COS_TILED_EXP=1 timeout 300 $B >> $O 2>&1
echo "--- COS_TILED_EXP=1 L2PF=2" >> $O; FMOE_L2PF=2 FMOE_COS_TILED_EXP=1 timeout 300 $B >> $O 2>&1
B2="python tools/batched_micro.py --n 16000000 --B 256 --k 8 --reps 3 --only semantic_cos,blend_cos"
echo "--- 16M base" >> $O; timeout 600 $B2 >> $O 2>&1
echo "--- 16M COS_TILED_EXP=1" >> $O; FMOE_COS_TILED_EXP=1 timeout 600 $B2 >> $O 2>&1
echo done
