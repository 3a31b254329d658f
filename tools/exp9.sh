FRS_LIB_PATH=scratch/lib_head.so FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp9_head.txt 2>&1
FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp9_cur.txt 2>&1
FRS_LIB_PATH=scratch/lib_head.so timeout 120 python tools/fast_diag.py --calls 200 > gpurun_out/exp9_head_diag.json 2>&1
timeout 120 python tools/fast_diag.py --calls 200 > gpurun_out/exp9_cur_diag.json 2>&1
