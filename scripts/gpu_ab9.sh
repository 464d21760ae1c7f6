mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -7 | cut -c1-250
timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120
GEVO_TRACE=1 timeout 1200 python scripts/search_time.py > gpurun_out/search_time3.log 2>&1; grep "gevo trace" gpurun_out/search_time3.log | cut -c1-300
