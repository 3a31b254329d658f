set -u
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
done
