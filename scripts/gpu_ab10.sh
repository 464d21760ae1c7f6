mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_spin.py tests/test_gpu_fuzz.py tests/test_gpu_authored.py tests/test_gpu_wide_conflicts.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -12 | cut -c1-260
timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120
