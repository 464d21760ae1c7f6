mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conflicts.py tests/test_gpu_wide_conflicts.py tests/test_gpu_parity.py tests/test_gpu_spin.py tests/test_gpu_authored.py -x -q 2>&1 | tail -4
for L in libgevo_b200.so libgevo_b200_ab.so; do
  echo "== $L"
  GEVO_LIB=$PWD/paper_2004_08140_b200/$L timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | cut -c1-400
  GEVO_LIB=$PWD/paper_2004_08140_b200/$L GEVO_SCRATCH_GB=64 timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | head -1
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['secondary']['value'], d['secondary']['ms_per_step'])"
GEVO_LIB=$PWD/paper_2004_08140_b200/libgevo_b200_ab.so timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['secondary']['value'], d['secondary']['ms_per_step'])"
