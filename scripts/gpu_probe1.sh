for e in "GEVO_RECONV=1" "GEVO_RECONV=0"; do echo "== $e"; env $e timeout 300 python scripts/diag/one_c4.py 696 353 2>&1 | grep -v "^  \|^kernel\|^[a-z]*:$\|^}" ; done
env GEVO_RECONV=1 timeout 300 python scripts/diag/one_c4.py 696 2>&1 | head -100
