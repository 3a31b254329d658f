# bench us/step under each FRS_ABLATE diagnostic (usage: bash tools/ablate.sh TAG "0 1 3 7 13")
TAG=$1; LIST=${2:-"0 1 3 7 13"}
for a in $LIST; do
  FRS_ABLATE=$a timeout 200 python bench.py --no-cpu-baseline --no-verify --steps 1000 > gpurun_out/abl_${TAG}_$a.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/abl_${TAG}_$a.json').read().strip().splitlines()[-1]); print('ablate $a', round(d['us_per_step'],2))" >> gpurun_out/abl_$TAG.txt
done
