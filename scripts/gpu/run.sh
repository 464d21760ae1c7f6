#!/bin/bash
# Rebuild in-tree (the built .so travels with the snapshot), then run a
# command on the B200 box: scripts/gpu/run.sh <timeout_s> '<command>'
set -e
cd "$(dirname "$0")/../.."
make -C oracle -j8 >/dev/null
make -C paper_2004_08140_b200 -j8 >/dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
