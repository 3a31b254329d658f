# quick GPU pass + a bench line (usage: bash tools/quick2.sh TAG)
set -u
TAG=$1; shift
bash tools/quick.sh $TAG "$@"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
