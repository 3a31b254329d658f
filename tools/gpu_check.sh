#!/usr/bin/env bash
# One gpurun pass: GPU parity tests, a bench line, the ncu launch list and one full capture
# of the FAST draft-head kernel. Usage (from the repo root, under gpurun):
#   bash tools/gpu_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python tools/fast_diag.py --calls 400 > $OUT/diag_$TAG.json 2> $OUT/diag_$TAG.err
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(fast|hsplit|exact|softmax|argmax|slab|accept|gather)' -s 20 -c 40 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_main -s 5 -c 2 \
    -o $OUT/prof_fast_$TAG -f python bench.py --steps 10 --warmup 5 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo done
