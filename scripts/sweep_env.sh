# bench.py under several env settings (no cpu baseline): sweep_env.sh "VAR=a VAR2=b" ...
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'evals/s', round(d['ms_per_step'],3), 'ms', d['step_ms'])"
done
