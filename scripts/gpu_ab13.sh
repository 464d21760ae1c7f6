timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for e in "GEVO_STAGE=1" "GEVO_STAGE=0"; do
echo "== $e"
env $e timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -1 | cut -c1-200
env $e timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-100
env $e timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bp.json; python -c "import json; d=json.load(open('gpurun_out/bp.json')); print('c4', d['value'], d['ms_per_step'], 'c2', d['secondary']['value'], d['secondary']['ms_per_step'])"
done
timeout 900 python scripts/diag/slow_variants.py nw-sync 65536 1 6 2>&1 | cut -c1-400
