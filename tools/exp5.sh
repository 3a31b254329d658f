set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_fast_(finalize|main)' -s 10 -c 2 -o $OUT/prof_exp5 -f python tools/fast_diag.py --calls 10 > $OUT/exp5_ncu.log 2>&1
