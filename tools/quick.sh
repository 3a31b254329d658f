# quick GPU pass: parity tests, trace, diag (usage: bash tools/quick.sh TAG [pytest-args])
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 420 python -m pytest tests -m gpu -x -q -s "$@" > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_$TAG.log
FRS_TRACE=1 timeout 120 python tools/fast_trace.py > $OUT/trace_$TAG.txt 2>&1
timeout 180 python tools/fast_diag.py --calls 400 > $OUT/diag_$TAG.json 2>&1
timeout 60 ./tools/hbm_probe > $OUT/probe_$TAG.txt 2>&1
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.mem,clocks.max.sm,power.draw,temperature.gpu --format=csv >> $OUT/probe_$TAG.txt 2>&1
