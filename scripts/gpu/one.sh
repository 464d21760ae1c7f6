# one config-4 candidate alone under knobs: C4_SEED / C4_IDX
S=${C4_SEED:-1}; I=${C4_IDX:-27}
for env in "" "GEVO_SPIN_THRESHOLD=0" "GEVO_SPIN_PAY=0" "GEVO_SPIN_PAY=4096" "GEVO_RECONV=0"; do
  echo "== $env"; env $env C4_SEED=$S timeout 200 python scripts/diag/one_c4.py $I 2>&1 | grep -E "spins|device_ms|test\": 0"
done
