mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('c4', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline'], 'c2', d['secondary']['value'], d['secondary']['ms_per_step'], 'clocks', d['clocks'])"
timeout 1800 python scripts/nsga_bench.py > gpurun_out/nsga.jsonl 2> gpurun_out/nsga.err; tail -3 gpurun_out/nsga.err; cat gpurun_out/nsga.jsonl
