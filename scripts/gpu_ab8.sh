mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
AB="GEVO_LIB=$PWD/paper_2004_08140_b200/libgevo_b200_ab.so"
for e in "GEVO_X=1" "$AB"; do
  echo "== $e"
  env $e timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -1 | cut -c1-250
  env $e timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120
done
GEVO_TRACE=1 timeout 1200 python scripts/search_time.py > gpurun_out/search_time2.log 2>&1; grep "gevo trace" gpurun_out/search_time2.log | cut -c1-300
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bench_perf.json; python -c "import json; d=json.load(open('gpurun_out/bench_perf.json')); print('c4', d['value'], d['ms_per_step'], 'dev_ir/s', d['device_ir_per_s'], 'ref_ir/s', d['ir_per_s'], json.dumps(d['roofline'])[:500])"
