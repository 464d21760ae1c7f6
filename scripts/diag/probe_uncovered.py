"""Budget-exceeding instances the spin accelerator did not jump (per-test
record jumps == 0), for a registry benchmark's candidate sample."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

bench, n = sys.argv[1], int(sys.argv[2])
cands = gevo.sample_candidates(bench, n, 1, 4)
suite = gevo.Suite.from_benchmark(bench, 1, gevo.train_seed(1))
b = suite.batch()
for c in cands:
    b.add_patch(c)
_, t, st = b.eval(suite.exec_config(), tests=True)
bud = [(i, int(t[i, 0]["pad"][0])) for i in range(len(cands)) if int(t[i, 0]["status"]) == 2]
unc = [i for i, j in bud if j == 0]
print(bench, "budget", len(bud), "not jumped", len(unc), "ms", st.device_ms)
with open(os.path.join(ROOT, "gpurun_out", "uncovered_%s.txt" % bench), "w") as f:
    for i in unc[:6]:
        f.write("# %d\n%s\n" % (i, gevo.apply_patch(gevo.benchmark_ir(bench), cands[i])[0]))
