mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for e in "GEVO_RECONV=-" "GEVO_RECONV=0"; do
  echo "== $e"
  env $e timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -1 | cut -c1-250
  env $e timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120
done
for e in "GEVO_RECONV=-" "GEVO_RECONV=1"; do
env $e timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_perf.json; python -c "import json; d=json.load(open('gpurun_out/bench_perf.json')); print('$e c4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'c2', d['secondary']['value'], d['secondary']['ms_per_step'], 'rank', d['rank_select_ms'])"
done
GEVO_TRACE=1 timeout 1200 python scripts/search_time.py --ref > gpurun_out/search_time.log 2>&1; grep -v "^\[gevo" gpurun_out/search_time.log | cut -c1-330; grep "gevo trace" gpurun_out/search_time.log | cut -c1-300
