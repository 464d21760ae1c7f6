timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_search.py tests/test_conformance.py -x -q 2>&1 | tail -3
GEVO_TRACE=1 timeout 600 python scripts/search_time.py --ref 2>&1 | grep -v "^$" | cut -c1-700
