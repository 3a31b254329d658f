for a in 0 4 5; do
FRS_ABLATE=$a timeout 200 python tools/loop_probe.py > gpurun_out/exp14_ablate$a.txt 2>&1
done
