# quick A/B of an interpreter change: per-IR latency, config-4 sets, bench (config 4 + config 2), config 3
timeout 300 python scripts/diag/ir_latency_gc.py 20000 2>&1 | tail -4 | cut -c1-140
timeout 400 python scripts/diag/c4_sets.py 1,2,5,8 2>&1 | python -c "import sys,json; print(' '.join('%d:%.0f' % (json.loads(l)['seed'], json.loads(l)['device_ms'][0]) for l in sys.stdin if l.startswith('{')))"
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/ab.json; python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('c4', round(d['value'],1), 'c2', round(d['secondary']['value']), round(d['secondary']['ms_per_step'],4))"
timeout 300 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-90
