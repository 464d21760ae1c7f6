"""GPU probe: which variants set the interpreter launch's tail. Times every
candidate of the bench workload alone (batch of one, all tests, early exit)
and dumps the slowest ones (records + IR) to gpurun_out/tail_<bench>.txt."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

BENCHES = sys.argv[1:] or ["hot-branch", "nw-sync", "bfs-load"]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
summary = {}
for bench in BENCHES:
    cands = gevo.sample_candidates(bench, 1024, 1, 4)
    suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
    cfg = suite.exec_config()
    times, seq_times, reruns = [], [], []
    for i, c in enumerate(cands):
        b = suite.batch()
        b.add_patch(c)
        b.eval(cfg, early_exit=True)
        gevo.tp_counters(reset=True)
        _, _, st = b.eval(cfg, early_exit=True)
        reruns.append(gevo.tp_counters(reset=True)[0])
        times.append((st.device_ms, i))
        _, _, st = b.eval(cfg, early_exit=True, sequential=True)
        seq_times.append(st.device_ms)
    # one empty-ish batch: launch overhead floor
    b = suite.batch()
    b.add_ir(gevo.benchmark_ir(bench))
    b.eval(cfg, early_exit=True)
    _, _, st0 = b.eval(cfg, early_exit=True)
    times.sort(reverse=True)
    tot = sum(t for t, _ in times)
    summary[bench] = {"sum_ms": tot, "seq_sum_ms": sum(seq_times), "original_ms": st0.device_ms,
                      "median_ms": sorted(t for t, _ in times)[len(times) // 2],
                      "seq_median_ms": sorted(seq_times)[len(seq_times) // 2],
                      "variants_rerun": sum(1 for r in reruns if r),
                      "top": [(round(t, 3), i, reruns[i]) for t, i in times[:20]],
                      "n_over_1ms": sum(1 for t, _ in times if t > 1.0)}
    print(bench, json.dumps(summary[bench]), flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "tail_%s.txt" % bench), "w") as f:
        for t, i in times[:8]:
            b = suite.batch()
            b.add_patch(cands[i])
            v, tr, st = b.eval(cfg, early_exit=False, tests=True)
            ir, _ = gevo.apply_patch(gevo.benchmark_ir(bench), cands[i])
            f.write("# variant %d  %.3f ms\n# patch %s\n" % (i, t, cands[i]))
            for k in range(tr.shape[1]):
                r = tr[0, k]
                f.write("#  test %d status %d code %d ir %d jumps %d why %d\n" %
                        (k, r["status"], r["code"], r["ir"], r["pad"][0], r["pad"][1]))
            f.write(ir + "\n")
json.dump(summary, open(os.path.join(ROOT, "gpurun_out", "tail_probe.json"), "w"), indent=1)
