timeout 300 python -m pytest tests/test_gpu_tp.py tests/test_gpu_wide_conflicts.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_spin.py tests/test_gpu_authored.py tests/test_gpu_shapes.py tests/test_gpu_fuzz.py tests/test_gpu_conflicts.py -x -q 2>&1 | tail -2
timeout 120 python scripts/diag/one_c4.py 27 353 1856 2>&1 | grep -E "spins|test\"\: 0"
timeout 300 python scripts/diag/c4_tail.py 4096 2>&1 | grep -E "variants|active|late_cta" | head -6 | cut -c1-300
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bp.json; python -c "import json; d=json.load(open('gpurun_out/bp.json')); print('c4', d['value'], d['ms_per_step'], 'c2', d['secondary']['value'], d['secondary']['ms_per_step'])"
GEVO_FOCUS=0 timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bp0.json; python -c "import json; d=json.load(open('gpurun_out/bp0.json')); print('nofocus c4', d['value'], d['ms_per_step'])"
timeout 300 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-100
