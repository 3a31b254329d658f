FRS_EXP_NO_PDL_FB=1 FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp7_trace_nopdl.txt 2>&1
FRS_EXP_NO_PDL_FB=1 timeout 120 python tools/fast_diag.py --calls 200 > gpurun_out/exp7_diag_nopdl.json 2>&1
