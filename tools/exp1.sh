set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/fast_diag.py --calls 200 > $OUT/exp1_rowmajor.json 2>&1
FRS_EXPERIMENT_TILED=1 python tools/fast_diag.py --calls 200 > $OUT/exp1_tiled.json 2>&1
FRS_EXPERIMENT_TILED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_fast_main -s 20 -c 3 --csv python tools/fast_diag.py --calls 30 > $OUT/exp1_tiled_ncu.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_fast_main -s 20 -c 3 --csv python tools/fast_diag.py --calls 30 > $OUT/exp1_rm_ncu.csv 2>&1
