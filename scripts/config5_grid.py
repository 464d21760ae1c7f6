"""Config 5 (BASELINE.json configs[4]): throughput grid pop x tests on one
B200 with the reference's CPU path beside every cell.

  python scripts/config5_grid.py [--kernels nw-sync,bfs-load] [--pops ...]
                                 [--tests ...] [--cpu-seconds 2] > grid.jsonl

Per corpus kernel and variant mix, per test count T (generate_tests(b, T,
train_seed(1))) and population P:
  raw   = P validated candidate mutants (seeded random walks of up to 4
          edits: trapping, over-tolerance and budget-spinning variants as the
          search produces them),
  clean = P accepted individuals (raw candidates that pass every test of the
          suite, cycled to P).
Device: the batch is made resident and evaluated with early exit; the cell's
time is the minimum of 3 CUDA-event timed evaluations; evals/s counts the
reference-equivalent executions. CPU: oracle/_ref/ref_bench (the reference's
evaluate_fitness, /root/reference/proj/src compiled in place) on the same
candidates with every host core, a bounded sample per cell. SM clocks are
sampled with nvidia-smi while each (kernel, mix, T) row runs."""
import argparse
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (ClockSampler)
import paper_2004_08140_b200 as gevo  # noqa: E402

REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


def cpu_cell(kernel, cands, tests, seed, seconds):
    if not os.path.exists(REF_BENCH) or seconds <= 0:
        return None
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(cands[:4096]) + "\n")
        path = f.name
    threads = os.cpu_count() or 1
    try:
        out = subprocess.run([REF_BENCH, kernel, path, str(tests), str(seed), str(threads),
                              str(seconds), "1000000", "0"], check=True, capture_output=True,
                             text=True, env=dict(os.environ, REF_BENCH_NOCOUNT="1")).stdout
    finally:
        os.unlink(path)
    r = json.loads(out.strip().splitlines()[-1])
    return {"value": r["executions"] / r["seconds"], "unit": "evals/s", "cores": threads,
            "kind": "reference", "sample": "%d variants x %d tests, %.1f s bound" %
            (r["variants"], tests, seconds)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", default="nw-sync,hot-branch,bfs-load")
    ap.add_argument("--pops", default="64,256,1024,4096,16384,65536")
    ap.add_argument("--tests", default="1,4,16,64,256")
    ap.add_argument("--mixes", default="raw,clean")
    ap.add_argument("--cpu-seconds", type=float, default=2.0)
    a = ap.parse_args()
    pops = [int(x) for x in a.pops.split(",")]
    seed = gevo.train_seed(1)
    for k in a.kernels.split(","):
        raw = gevo.sample_candidates(k, max(pops), 1, 4)
        for T in [int(x) for x in a.tests.split(",")]:
            suite = gevo.Suite.from_benchmark(k, T, seed)
            cfg = suite.exec_config()
            mixes = {}
            if "raw" in a.mixes:
                mixes["raw"] = raw
            if "clean" in a.mixes:
                # accepted individuals of this suite, cycled to the largest pop
                probe = suite.batch()
                for c in raw[:8192]:
                    probe.add_patch(c)
                v, _, _ = probe.eval(cfg, early_exit=True)
                ok = [raw[i] for i in range(len(v)) if v["accepted"][i]]
                del probe
                if ok:
                    mixes["clean"] = [ok[i % len(ok)] for i in range(max(pops))]
            for mix, pool in mixes.items():
                with bench.ClockSampler(int(os.environ.get("GEVO_DEVICE", "0"))) as ck:
                    rows = []
                    for P in pops:
                        b = suite.batch()
                        for c in pool[:P]:
                            b.add_patch(c)
                        b.make_resident()
                        v, _ = b.eval_resident(cfg, early_exit=True, records=True)
                        ms = min(b.eval_resident(cfg, early_exit=True)[1].device_ms for _ in range(3))
                        execs = int(v["execs_ref"].sum())
                        rows.append({"config": "config5", "kernel": k, "mix": mix, "pop": P,
                                     "tests": T, "ms": round(ms, 4),
                                     "evals_per_s": execs / (ms / 1e3),
                                     "ir_per_s": int(v["ir_ref"].sum()) / (ms / 1e3),
                                     "executions": execs, "n_gpus": 1})
                        del b
                clocks = ck.summary()
                for r in rows:
                    r["clocks"] = clocks
                    r["cpu_baseline"] = cpu_cell(k, pool[:r["pop"]], T, seed, a.cpu_seconds)
                    if r["cpu_baseline"]:
                        r["vs_cpu"] = r["evals_per_s"] / r["cpu_baseline"]["value"]
                    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
