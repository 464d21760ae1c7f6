for e in "GEVO_SPIN_THRESHOLD=256" "GEVO_SPIN_THRESHOLD=0" "GEVO_SPIN_THRESHOLD=2048" "GEVO_SPIN_THRESHOLD=16384"; do echo "== $e"
env $e timeout 900 python scripts/diag/c4_tail.py 4096 2>&1 | grep -E "variants" | cut -c1-200
env $e timeout 600 python scripts/bench_configs.py config3 --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-100
done
