timeout 1500 python -m pytest tests/test_gpu_spin.py tests/test_gpu_fuzz.py tests/test_gpu_authored.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
AB="GEVO_LIB=$PWD/paper_2004_08140_b200/libgevo_b200_ab.so"
for e in "GEVO_X=1" "$AB"; do echo "== $e"
env $e timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | grep -E "variants" | cut -c1-200
env $e timeout 300 python scripts/diag/one_c4.py 3810 2752 2>&1 | grep -E "spins|test\"\: 0"
env $e timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-100
env $e timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/bp.json; python -c "import json; d=json.load(open('gpurun_out/bp.json')); print('c4', d['value'], d['ms_per_step'], 'c2', d['secondary']['value'], d['secondary']['ms_per_step'])"
done
