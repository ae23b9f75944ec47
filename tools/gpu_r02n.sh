mkdir -p gpurun_out
B="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,semantic"
O=gpurun_out/stages4.log
echo "--- base" > $O; timeout 300 $B >> $O 2>&1
echo "--- COS_DIRECT" >> $O; FMOE_COS_DIRECT=1 timeout 300 $B >> $O 2>&1
echo "--- EXTRA=4 SMEM=218 COS_DIRECT (4 stages)" >> $O; FMOE_APPROX_EXTRA=4 FMOE_UMMA_SMEM_KB=218 FMOE_COS_DIRECT=1 timeout 300 $B >> $O 2>&1
echo "--- EXTRA=4 SMEM=218" >> $O; FMOE_APPROX_EXTRA=4 FMOE_UMMA_SMEM_KB=218 timeout 300 $B >> $O 2>&1
echo "--- EXTRA=4" >> $O; FMOE_APPROX_EXTRA=4 timeout 300 $B >> $O 2>&1
echo done
