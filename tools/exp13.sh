for a in 0 1 2 3; do
FRS_ABLATE=$a timeout 200 python tools/loop_probe.py > gpurun_out/exp13_ablate$a.txt 2>&1
done
