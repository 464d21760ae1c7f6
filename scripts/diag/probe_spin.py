"""GPU probe: per-IR latency of a lone spinning lane and the spinners the
exact accelerator does not cover. Writes gpurun_out/spin_probe.json and the
uncovered kernels' IR to gpurun_out/uncovered_<bench>.ir."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

out = {}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for bench in ("hot-branch", "nw-sync", "bfs-load"):
    cands = gevo.sample_candidates(bench, 1024, 1, 4)
    suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
    cfg = suite.exec_config()
    b = suite.batch()
    for c in cands:
        b.add_patch(c)
    t0 = time.time()
    v, t, st = b.eval(cfg, tests=True)
    budget = t["status"] == 2
    jumped = t["pad"][:, :, 0] > 0
    unc = budget & ~jumped
    rows = sorted(set(int(i) for i in unc.nonzero()[0]))
    import collections
    why = collections.Counter(int(x) for x in t["pad"][:, :, 1][unc])
    ir_unc = t["ir"][unc]
    out[bench] = {"device_ms": st.device_ms, "budget_lanes": int(budget.sum()),
                  "jumped_lanes": int((budget & jumped).sum()),
                  "uncovered_lanes": int(unc.sum()), "uncovered_variants": len(rows),
                  "uncovered_ir_max": int(ir_unc.max()) if len(ir_unc) else 0,
                  "abandon_reasons": {hex(k): v for k, v in why.most_common()}}
    with open(os.path.join(ROOT, "gpurun_out", "uncovered_%s.ir" % bench), "w") as f:
        for r in rows[:12]:
            ir, _ = gevo.apply_patch(gevo.benchmark_ir(bench), cands[r])
            f.write("# variant %d tests %s\n%s\n" % (r, unc[r].nonzero()[0].tolist(), ir))
    # lone spinner latency: one uncovered variant, one test
    if rows:
        s1 = gevo.Suite.from_benchmark(bench, 1, gevo.train_seed(1))
        b1 = s1.batch().add_patch(cands[rows[0]])
        b1.make_resident()
        for _ in range(2):
            vr, st1 = b1.eval_resident(s1.exec_config(), records=True)
        vr, st1 = b1.eval_resident(s1.exec_config(), records=True)
        ir = int(vr["ir_ref"][0])
        out[bench]["lone_spinner"] = {"ms": st1.device_ms, "ir": ir,
                                      "cycles_per_ir_at_1965MHz": st1.device_ms * 1.965e6 / max(ir, 1)}
    print(bench, json.dumps(out[bench]), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "spin_probe.json"), "w"), indent=1)
