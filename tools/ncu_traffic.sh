#!/usr/bin/env bash
# dram__bytes of k_fast_main per launch for the CURRENT build (run under gpurun): writes
# profiles/ncu_fast_bf16_summary.json tagged with the kernel sources' sha256 (bench.py reports
# the traffic only when the tag matches the sources it runs).
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_fast_main -s 10 -c 5 --csv --log-file $OUT/ncu_traffic.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-decode --no-verify --no-sweep --no-batched > /dev/null 2>&1
python - <<'PY'
import csv, hashlib, json, statistics
rows = list(csv.reader(open("gpurun_out/ncu_traffic.csv")))
hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hdr]
vals = {}
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(d.get("Metric Unit", ""), 1)
    vals.setdefault(d["Metric Name"], []).append(float(d["Metric Value"].replace(",", "")) * scale)
rd = statistics.median(vals["dram__bytes_read.sum"])
wr = statistics.median(vals["dram__bytes_write.sum"])
import sys; sys.path.insert(0, ".")
from bench import source_sha256
sha = source_sha256()
out = {"kernel": "k_fast_main<16,1,0>", "source": "tools/ncu_traffic.sh (ncu --metrics dram__bytes_*, C2, 5 launches, median)",
       "source_sha256": sha, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
       "gpu_time_ns_median": statistics.median(vals.get("gpu__time_duration.sum", [0]))}
json.dump(out, open("profiles/ncu_fast_bf16_summary.json", "w"), indent=1)
json.dump(out, open("gpurun_out/ncu_fast_bf16_summary.json", "w"), indent=1)  # merged back by gpurun
print(json.dumps(out))
PY
