set -u
OUT=gpurun_out; mkdir -p $OUT
FRS_TRACE=1 python tools/fast_trace.py > $OUT/exp2_trace.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_finalize -s 5 -c 1 -o $OUT/prof_fin_exp2 -f python tools/fast_diag.py --calls 10 > $OUT/exp2_ncu.log 2>&1
