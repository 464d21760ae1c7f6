# ncu of one config-4 candidate alone: C4_SEED / C4_IDX select it (default seed 1, index 27)
S=${C4_SEED:-1}; I=${C4_IDX:-27}
C4_SEED=$S timeout 120 python scripts/diag/one_c4.py $I 2>&1 | grep -E "spins|test|device_ms"
C4_SEED=$S GEVO_SPIN_THRESHOLD=0 timeout 300 python scripts/diag/one_c4.py $I 2>&1 | grep -E "spins|test|device_ms"
GEVO_RECONV=0 C4_SEED=$S timeout 120 python scripts/diag/one_c4.py $I 2>&1 | grep -E "spins|test|device_ms"
C4_SEED=$S GEVO_CTA_CLOCK=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp_tp -s 1 -c 1 -o gpurun_out/c4one -f python scripts/diag/one_c4.py $I > gpurun_out/c4one.log 2>&1
ncu -i gpurun_out/c4one.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c4one_src.csv 2>/dev/null
ncu -i gpurun_out/c4one.ncu-rep --page raw --csv > gpurun_out/c4one_raw.csv 2>/dev/null
tail -2 gpurun_out/c4one.log
