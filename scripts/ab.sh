# A/B: default library vs paper_2004_08140_b200/libgevo_b200_ab.so on the
# config-2 bench, a config-3 slice and the lone-lane IR latency
AB="GEVO_LIB=$PWD/paper_2004_08140_b200/libgevo_b200_ab.so"
bash scripts/sweep_env.sh "GEVO_TP=1" "$AB" "GEVO_TP=1" "$AB"
for e in "GEVO_TP=1" "$AB"; do echo "== $e"; env $e timeout 300 python scripts/bench_configs.py config3 --pop ${CFG3_POP:-512} --steps 2 --cpu-seconds 0 2>&1 | tail -1 | cut -c1-120; done
for e in "GEVO_SPIN_THRESHOLD=0" "GEVO_SPIN_THRESHOLD=0 $AB"; do echo "== $e"; env $e python scripts/ir_latency.py 20000 | cut -c1-100; done
