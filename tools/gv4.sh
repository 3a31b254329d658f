timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py > gpurun_out/sanitize_racecheck2.log 2>&1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 5 python tools/sanitize.py > gpurun_out/sanitize_initcheck2.log 2>&1
tail -n 2 gpurun_out/sanitize_racecheck2.log gpurun_out/sanitize_initcheck2.log
timeout 300 python tools/layer_probe.py 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q -k "layer or exact or attention or verify" 2>&1 | tail -1
