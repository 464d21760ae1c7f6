# Config-4 interpreter study: test-lane mapping A/B and one ncu --set full
# capture of a representative batch launch (the second interp_tp launch: the
# first is the suite's oracle generation).
mkdir -p gpurun_out
for ln in 32 1; do
  GEVO_TP_LANES=$ln timeout 600 python scripts/bench_configs.py config4 --pop 1024 --steps 1 --cpu-seconds 0 > gpurun_out/c4_ln$ln.json 2>&1; tail -1 gpurun_out/c4_ln$ln.json
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp_tp --launch-skip 1 -c 1 -o gpurun_out/c4b -f python scripts/bench_configs.py config4 --pop 296 --steps 1 --cpu-seconds 0 > gpurun_out/c4bncu.log 2>&1; tail -2 gpurun_out/c4bncu.log
timeout 900 python -m pytest tests/test_gpu_authored.py tests/test_gpu_parity.py -k "golden or nsga" -x -q 2>&1 | tail -5
