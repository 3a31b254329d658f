mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "layer or attention" > gpurun_out/gv7_tests.log 2>&1; echo rc=$? >> gpurun_out/gv7_tests.log
tail -2 gpurun_out/gv7_tests.log
timeout 300 python tools/layer_probe.py 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gv7_layer_launches.csv python tools/layer_probe.py > /dev/null 2>&1
python - <<'PY'
import csv, io
lines=[l for l in open('gpurun_out/gv7_layer_launches.csv') if not l.startswith('==')]
rows=list(csv.DictReader(io.StringIO(''.join(lines))))
for r in rows[-19:]: print(r['Kernel Name'][:50], r['Metric Value'])
PY
