timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python scripts/diag/slow_variants.py nw-sync 65536 1 3 2>&1 | cut -c1-250
timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -1 | cut -c1-200
timeout 300 python scripts/diag/one_c4.py 3810 2752 2>&1 | grep -E "spins|test|device_ms"
for e in "GEVO_RECONV=0" "GEVO_SPIN_THRESHOLD=0"; do echo "== $e"; env $e timeout 300 python scripts/diag/one_c4.py 3810 2>&1 | grep -E "spins|test\"\: 0|device_ms"; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bp.json; python -c "import json; d=json.load(open('gpurun_out/bp.json')); print('c4', d['value'], d['ms_per_step'], 'c2', d['secondary']['value'], d['secondary']['ms_per_step'])"
