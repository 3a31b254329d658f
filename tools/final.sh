#!/usr/bin/env bash
# Round-end pass: gpu_check + sweeps + the reference arm + the draft-layer launch list.
TAG=${1:-r01e}
bash tools/gpu_check.sh $TAG
timeout 1200 python tools/sweep.py --exact > gpurun_out/sweep_$TAG.jsonl 2> gpurun_out/sweep_$TAG.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/layer_launches_$TAG.csv python tools/layer_probe.py > /dev/null 2>&1
tail -2 gpurun_out/pytest_gpu_$TAG.log
cat gpurun_out/bench_$TAG.json | cut -c1-400
