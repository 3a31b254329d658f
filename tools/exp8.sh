for pre in 1 4 0; do
FRS_EXP_PRE=$pre FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp8_trace_pre$pre.txt 2>&1
done
