#!/usr/bin/env bash
# Regenerates the committed golden fixtures under tests/golden/ from the
# reference compiled in place (oracle/_ref, see oracle/Makefile). Needs
# /root/reference (this container only). TEST INFRASTRUCTURE.
set -euo pipefail
cd "$(dirname "$0")"
make -s ref
OUT=../tests/golden
mkdir -p "$OUT" "$OUT/runs"
./_ref/ref_dump corpus  | gzip -9n > "$OUT/corpus.jsonl.gz"
./_ref/ref_dump vmcases | gzip -9n > "$OUT/vmcases.jsonl.gz"
./_ref/ref_dump mutants 400 | gzip -9n > "$OUT/mutants.jsonl.gz"
./_ref/ref_dump mutants 150 20000 | gzip -9n > "$OUT/mutants_budget20k.jsonl.gz"
./_ref/ref_dump nsga 300 | gzip -9n > "$OUT/nsga.jsonl.gz"
# Search trajectories (reference CLI artefacts): config 1 and small runs of
# every corpus kernel in both modes.
run() { # name bench seed pop gens mode train heldout
  local d="$OUT/runs/$1"; rm -rf "$d"; mkdir -p "$d"
  ./_ref/ref_dump run "$2" "$3" "$4" "$5" "$6" "$7" "$8" "$d" > /dev/null
  rm -f "$d/best.ir" "$d/best.patch.json"
}
run config1_nw-sync nw-sync 1 32 5 default 3 3
for b in bfs-load hot-branch hot-memo lud-store lud-unroll nw-sync; do
  run small_${b}_default $b 7 16 4 default 3 2
  run small_${b}_mo $b 3 16 4 mo 3 2
done
echo "golden fixtures written to $OUT"
