timeout 300 python scripts/diag/one_c4.py 696 353 2>&1 | grep -E "test|device_ms"
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_spin.py tests/test_gpu_authored.py tests/test_gpu_wide_conflicts.py -x -q 2>&1 | tail -2
timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -9 | cut -c1-260
timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120
