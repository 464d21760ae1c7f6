"""Status / IR profile of an authored config's candidates (which ones are slow)."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

name, pop = sys.argv[1], int(sys.argv[2])
ir, gen = gevo.authored_kernel(name)
suite = gevo.Suite.from_spec(ir, gen, 1, gevo.train_seed(1))
cfg = suite.exec_config()
cands = gevo.sample_candidates_ir(ir, pop, 1, 3)
times = []
for i, c in enumerate(cands):
    b = suite.batch().add_patch(c)
    v, t, st = b.eval(cfg, tolerance=0.01, tests=True)
    r = t[0, 0]
    times.append((st.device_ms, i, int(r["status"]), int(r["code"]), int(r["ir"]), int(r["pad"][0])))
times.sort(reverse=True)
print(json.dumps(collections.Counter((x[2], x[3]) for x in times).most_common()))
for x in times[:10]:
    print(x)
with open(os.path.join(ROOT, "gpurun_out", "cfg_slow_%s.txt" % name), "w") as f:
    for x in times[:4]:
        f.write("# %s\n%s\n" % (x, gevo.apply_patch(ir, cands[x[1]])[0]))
