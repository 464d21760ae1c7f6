timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_spin.py tests/test_gpu_authored.py tests/test_gpu_wide_conflicts.py tests/test_gpu_shapes.py -x -q 2>&1 | tail -2
for e in "GEVO_TP_PERSIST=1" "GEVO_TP_PERSIST=0"; do
echo "== $e"
env $e timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -1 | cut -c1-260
env $e timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120
done
