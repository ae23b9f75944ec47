mkdir -p gpurun_out
O=gpurun_out/c3_trace.log
timeout 300 python tools/trace.py --mode session --ell 3 --n 1000000 --D 8 --E 60 --L 24 --B 64 --k 8 > $O 2>&1
timeout 300 python tools/trace.py --mode session --ell 20 --n 1000000 --D 8 --E 60 --L 24 --B 64 --k 8 >> $O 2>&1
FMOE_NVCC_EXTRA=-DFMOE_EPI_PROFILE timeout 600 python paper_2502_05370_b200/build.py --force > gpurun_out/build_prof3.log 2>&1
timeout 300 python tools/trace.py --mode session --ell 3 --n 1000000 --D 8 --E 60 --L 24 --B 64 --k 8 >> $O 2>&1
timeout 300 python tools/trace.py --mode session --ell 20 --n 1000000 --D 8 --E 60 --L 24 --B 64 --k 8 >> $O 2>&1
echo done
