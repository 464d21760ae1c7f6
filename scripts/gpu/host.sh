timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_search.py tests/test_conformance.py tests/test_gpu_nsga_large.py -x -q 2>&1 | tail -3
GEVO_TRACE=1 timeout 600 python scripts/search_time.py --ref 2>&1 | grep -v "^$" | cut -c1-700
timeout 300 python scripts/nsga_bench.py --sizes 512,5120 --no-ref 2>&1 | tail -6
