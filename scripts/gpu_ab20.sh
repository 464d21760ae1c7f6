timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | cut -c1-330
