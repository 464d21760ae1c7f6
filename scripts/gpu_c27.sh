GEVO_CTA_CLOCK=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:interp_tp -s 1 -c 1 -o gpurun_out/c27 -f python scripts/diag/one_c4.py 27 > gpurun_out/c27.log 2>&1
ncu -i gpurun_out/c27.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c27_src.csv 2>/dev/null
ncu -i gpurun_out/c27.ncu-rep --page details --csv > gpurun_out/c27_details.csv 2>/dev/null
tail -3 gpurun_out/c27.log
