"""Throughput of the authored workloads (BASELINE.json configs 3 and 4) and the
config-5 sweep, beside bench.py's config-2 headline line.

  python scripts/bench_configs.py config3 [--pop 1024] [--steps 2]
  python scripts/bench_configs.py config4 [--pop 4096] [--steps 1]
  python scripts/bench_configs.py sweep   [--pops 64,256,1024,4096] [--tests 1,4,16]

config3: SVM RBF kernel row on a9a-shaped data (X 32561x123 f32 ~ U[0,1), q[123],
gamma 1/128, exp by range reduction + degree-6 polynomial, 256 simulated
threads), pop validated mutants x 3 test queries, tolerance 0.01, early exit.
config4: conv3x3 (+bias) and batch-norm (per-channel scale/shift) on a
CIFAR-shaped tensor (in 3x32x32, w 64x3x3x3, out 64x32x32), 256 threads.
One JSON line per config: evaluations/s (reference-equivalent executions, as
bench.py), dynamic IR/s, device ms per step (CUDA events around the
resident-batch evaluation), and the reference CPU path (oracle/_ref/ref_bench on
the same candidate file) timed on a bounded sample with every host core."""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
CONFIGS = {
    "config3": {"kernel": "svm-rbf", "tests": 3, "tol": 0.01, "pop": 1024,
                "workload": "config3: SVM RBF kernel row, a9a-shaped X[32561x123] f32 U[0,1), "
                            "256 simulated threads, validated mutants x 3 queries, tol 0.01"},
    "config4": {"kernel": "conv-bn", "tests": 3, "tol": 0.01, "pop": 4096,
                "workload": "config4: conv3x3+bias+batch-norm, CIFAR-shaped in[3x32x32] -> "
                            "out[64x32x32] f32, 256 simulated threads, validated mutants x 3 inputs, "
                            "tol 0.01"},
}


def cpu_reference(kernel, cands, tests, seed, tol, seconds):
    if not os.path.exists(REF_BENCH):
        return None
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(cands) + "\n")
        path = f.name
    threads = os.cpu_count() or 1
    out = subprocess.run([REF_BENCH, "file:" + os.path.join(gevo.KERNEL_DIR, kernel), path,
                          str(tests), str(seed), str(threads), str(seconds), "1000000", str(tol)],
                         check=True, capture_output=True, text=True,
                         env=dict(os.environ, REF_BENCH_NOCOUNT="1")).stdout
    os.unlink(path)
    r = json.loads(out.strip().splitlines()[-1])
    return {"value": r["executions"] / r["seconds"], "unit": "evals/s", "cores": threads,
            "kind": "reference", "sample": "%d of %d candidates x %d tests, %.0f s bound" %
            (r["variants"], len(cands), tests, seconds)}


def run_config(name, pop, steps, cpu_seconds):
    c = CONFIGS[name]
    ir, gen = gevo.authored_kernel(c["kernel"])
    seed = gevo.train_seed(1)
    suite = gevo.Suite.from_spec(ir, gen, c["tests"], seed)
    cfg = suite.exec_config()
    cands = gevo.sample_candidates_ir(ir, pop, 1, 3)
    batch = suite.batch()
    for p in cands:
        batch.add_patch(p)
    batch.make_resident()
    v, _ = batch.eval_resident(cfg, tolerance=c["tol"], early_exit=True, records=True)  # warm-up
    execs = int(v["execs_ref"].sum())
    ir_ref = int(v["ir_ref"].sum())
    ms = []
    for _ in range(steps):
        _, st = batch.eval_resident(cfg, tolerance=c["tol"], early_exit=True, records=True)
        ms.append(st.device_ms)
    t = statistics.mean(ms)
    line = {"metric": "variant x input evaluations/s", "value": execs / (t / 1e3), "unit": "evals/s",
            "config": {"workload": c["workload"], "variants": pop, "tests": c["tests"]},
            "ms_per_step": t, "steps": steps, "executions_per_step": execs,
            "ir_per_s": ir_ref / (t / 1e3), "accepted": int(v["accepted"].sum()),
            "tp_reruns": gevo.tp_counters(reset=True)[0]}
    if cpu_seconds > 0:
        line["cpu_baseline"] = cpu_reference(c["kernel"], cands[:max(8, min(64, pop))], c["tests"],
                                             seed, c["tol"], cpu_seconds)
    print(json.dumps(line), flush=True)
    return line


def run_sweep(pops, tests_list, kernels):
    for k in kernels:
        for T in tests_list:
            suite = gevo.Suite.from_benchmark(k, T, gevo.train_seed(1))
            cfg = suite.exec_config()
            for P in pops:
                cands = gevo.sample_candidates(k, P, 1, 4)
                b = suite.batch()
                for c in cands:
                    b.add_patch(c)
                b.make_resident()
                v, _ = b.eval_resident(cfg, early_exit=True, records=True)
                ms = []
                for _ in range(3):
                    _, st = b.eval_resident(cfg, early_exit=True, records=True)
                    ms.append(st.device_ms)
                t = min(ms)
                print(json.dumps({"sweep": k, "pop": P, "tests": T, "ms": round(t, 4),
                                  "evals_per_s": int(v["execs_ref"].sum()) / (t / 1e3)}),
                      flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["config3", "config4", "sweep"])
    ap.add_argument("--pop", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=30.0)
    ap.add_argument("--pops", default="64,256,1024,4096,16384")
    ap.add_argument("--tests", default="1,4,16,64")
    ap.add_argument("--kernels", default="nw-sync,hot-branch,bfs-load")
    a = ap.parse_args()
    if a.what == "sweep":
        run_sweep([int(x) for x in a.pops.split(",")], [int(x) for x in a.tests.split(",")],
                  a.kernels.split(","))
    else:
        run_config(a.what, a.pop or CONFIGS[a.what]["pop"], a.steps, a.cpu_seconds)


if __name__ == "__main__":
    main()
