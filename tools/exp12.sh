FRS_LIB_PATH=scratch/lib_oldprod.so FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp12_oldprod.txt 2>&1
FRS_LIB_PATH=scratch/lib_head.so FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp12_head.txt 2>&1
