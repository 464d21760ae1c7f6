# A/B over several library builds: ab_multi.sh libA.so libB.so ... (paths
# relative to paper_2004_08140_b200/; "default" = libgevo_b200.so). Per lib:
# config-2 bench, lone-lane IR latency, nw-sync/hot-branch batch probe.
P=$PWD/paper_2004_08140_b200
for lib in "$@"; do
  [ "$lib" = default ] && lib=libgevo_b200.so
  echo "######## $lib"
  export GEVO_LIB=$P/$lib
  bash scripts/sweep_env.sh "GEVO_TP=1" "GEVO_TP=1"
  GEVO_SPIN_THRESHOLD=0 timeout 300 python scripts/ir_latency.py 20000 2>&1 | cut -c1-110
done
