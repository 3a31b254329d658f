mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gv_layer_launches.csv python tools/layer_probe.py > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_exact_gemv -s 196 -c 2 -o gpurun_out/gv_full -f python tools/layer_probe.py > gpurun_out/gv_ncu.log 2>&1
tail -3 gpurun_out/gv_ncu.log
