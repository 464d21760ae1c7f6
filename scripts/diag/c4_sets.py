"""GPU probe: config-4 step time of each committed candidate set
(bench_data/cand_conv-bn_s<seed>.txt.gz; rank r of a multi-GPU bench reads
seed 1 + r): device ms of one early-exit evaluation (minimum of 3), the
reference-equivalent executions, and the longest CTA of the set."""
import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

ir, gen = gevo.authored_kernel("conv-bn")
suite = gevo.Suite.from_spec(ir, gen, 3, gevo.train_seed(1))
cfg = suite.exec_config()
for seed in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,5,6,7,8").split(",")]:
    with gzip.open(os.path.join(ROOT, "bench_data", "cand_conv-bn_s%d.txt.gz" % seed), "rt") as f:
        cands = [x for x in f.read().splitlines() if x.strip()]
    b = suite.batch()
    for c in cands:
        b.add_patch(c)
    b.make_resident()
    v, _ = b.eval_resident(cfg, tolerance=0.01, early_exit=True, records=True)
    ms = sorted(b.eval_resident(cfg, tolerance=0.01, early_exit=True)[1].device_ms for _ in range(3))
    execs = int(v["execs_ref"].sum())
    print(json.dumps({"seed": seed, "variants": len(cands), "device_ms": ms, "executions": execs,
                      "evals_per_s": execs / (ms[0] / 1e3),
                      "budget_variants": int((v["code"] == 29).sum()) if "code" in v.dtype.names else None}),
          flush=True)
    del b
