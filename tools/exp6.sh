set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:'k_fast_finalize' -s 10 -c 1 -o $OUT/prof_exp6 -f python tools/fast_diag.py --calls 10 > $OUT/exp6_ncu.log 2>&1
