for v in latelaunch finnopdl; do
FRS_LIB_PATH=scratch/lib_$v.so FRS_TRACE=1 timeout 120 python tools/fast_trace.py > gpurun_out/exp11_$v.txt 2>&1
done
