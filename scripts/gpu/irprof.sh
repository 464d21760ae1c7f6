IRGC_ONLY=t256_tid0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_tp -s 1 -c 1 -o gpurun_out/irgc -f python scripts/diag/ir_latency_gc.py 5000 > gpurun_out/irgc.log 2>&1
ncu -i gpurun_out/irgc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/irgc_src.csv 2>/dev/null
ncu -i gpurun_out/irgc.ncu-rep --page source --csv --print-source sass > gpurun_out/irgc_sass.csv 2>/dev/null
tail -2 gpurun_out/irgc.log
