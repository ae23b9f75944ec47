mkdir -p gpurun_out
M="python tools/batched_micro.py --n 2000000 --B 256 --k 8 --reps 5 --only semantic_cos,semantic"
O=gpurun_out/l2pf.log
echo "--- base (flush after tempty)" > $O
timeout 300 $M >> $O 2>&1
for pf in 2 3 4 6 8 12; do echo "--- FMOE_L2PF=$pf" >> $O; FMOE_L2PF=$pf timeout 300 $M >> $O 2>&1; done
echo "--- FMOE_UMMA_STAGES=2" >> $O; FMOE_UMMA_STAGES=2 timeout 300 $M >> $O 2>&1
echo "--- FMOE_UMMA_STAGES=2 FMOE_L2PF=4" >> $O; FMOE_UMMA_STAGES=2 FMOE_L2PF=4 timeout 300 $M >> $O 2>&1
echo "--- NO_EPI FMOE_L2PF=4" >> $O; FMOE_NO_EPI=1 FMOE_L2PF=4 timeout 300 $M >> $O 2>&1
timeout 300 python tools/trace.py --mode sem --n 2000000 --D 4096 --B 256 --k 8 > gpurun_out/sem_trace2.log 2>&1
FMOE_L2PF=4 timeout 300 python tools/trace.py --mode sem --n 2000000 --D 4096 --B 256 --k 8 >> gpurun_out/sem_trace2.log 2>&1
echo done
