#!/bin/bash
# Run the reference's unit suites built against libgevo_b200.so (see
# oracle/Makefile "conformance"). Exit status: number of failing suites.
cd "$(dirname "$(readlink -f "$0")")"
fail=0
for t in test_*; do
  [ -x "$t" ] || continue
  out=$(./"$t" 2>&1); rc=$?
  echo "$t: $(echo "$out" | tail -1)"
  [ $rc -ne 0 ] && { echo "$out" | head -40; fail=$((fail+1)); }
done
exit $fail
