#!/usr/bin/env bash
# Draft-layer check under gpurun: layer/attention/exact parity tests, one forward timing, the
# ncu launch list of one 10-row forward, and a full capture of the first exact GEMV launch of
# a 10-row forward (launch 196: after the 512-row context forward's 32 passes x 6 projections
# plus q/k/v/o). Usage: bash tools/layer_check.sh [tag]
TAG=${1:-layer}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "layer or attention or exact" > gpurun_out/${TAG}_tests.log 2>&1
tail -1 gpurun_out/${TAG}_tests.log
timeout 300 python tools/layer_probe.py 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/layer_probe.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_exact_gemv -s 196 -c 1 -o gpurun_out/${TAG}_gemv -f python tools/layer_probe.py > /dev/null 2>&1
