mkdir -p gpurun_out
M="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic"
O=gpurun_out/tiled2.log
echo "--- TN=512 NO_EPI" > $O; FMOE_NO_EPI=1 timeout 300 $M >> $O 2>&1
echo "--- TN=512 NO_EPI TILED=1" >> $O; FMOE_NO_EPI=1 FMOE_TILED_B_EXP=1 timeout 300 $M >> $O 2>&1
echo "--- TN=512 NO_EPI TILED=2" >> $O; FMOE_NO_EPI=1 FMOE_TILED_B_EXP=2 timeout 300 $M >> $O 2>&1
echo "--- TN=256 NO_EPI TILED=2" >> $O; FMOE_UMMA_TN=256 FMOE_NO_EPI=1 FMOE_TILED_B_EXP=2 timeout 300 $M >> $O 2>&1
echo "--- TN=512 TILED=2 (with epilogue; garbage)" >> $O; FMOE_TILED_B_EXP=2 timeout 300 $M >> $O 2>&1
B="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,blend_cos"
for r in 3 4 5; do echo "--- COS_RING=$r" >> $O; FMOE_COS_RING=$r timeout 300 $B >> $O 2>&1; done
echo done
