"""Wall time of a whole seeded GEVO search (config 1 / config 2) through the
product engine, with device/host split, and byte-equality with the reference's
trajectory when the golden run exists. With --ref, the reference CLI itself
(oracle/_ref/ref_dump run: src/cli_app.cpp cmd_run compiled in place) runs the
same search at jobs = nproc on this host, its log.csv compared byte for byte."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

RUNS = {"config1_nw-sync": ("nw-sync", 1, 32, 5, "default", 3, 3)}
for b in ("nw-sync", "bfs-load", "hot-branch", "hot-memo"):
    RUNS["config2_" + b] = (b, 1, 256, 50, "mo" if b == "hot-memo" else "default", 16, 3)
jobs = os.cpu_count() or 8
out = {}
# one untimed search first: CUDA context, module load and host pool start-up
gevo.run_search(*RUNS["config1_nw-sync"][:5], -1.0, *RUNS["config1_nw-sync"][5:], jobs=jobs)
import subprocess  # noqa: E402
import tempfile  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "ref_dump")
with_ref = "--ref" in sys.argv
names = [a for a in sys.argv[1:] if not a.startswith("--")]
for name in names or list(RUNS):
    bench, seed, pop, gens, mode, train, held = RUNS[name]
    t0 = time.time()
    log, rep, st = gevo.run_search(bench, seed, pop, gens, mode, -1.0, train, held, jobs=jobs)
    wall = time.time() - t0
    d = os.path.join(ROOT, "tests", "golden", "runs", name)
    same = None
    if os.path.isdir(d):
        same = log == open(os.path.join(d, "log.csv")).read()
    out[name] = {"wall_s": wall, "device_ms": st.device_ms, "host_gen_ms": st.host_gen_ms,
                 "candidates": st.candidates, "executions": st.executions, "batches": st.batches,
                 "launches": st.launches, "log_matches_reference": same, "jobs": jobs}
    if with_ref and os.path.exists(REF):
        with tempfile.TemporaryDirectory() as d:
            t0 = time.time()
            subprocess.run([REF, "run", bench, str(seed), str(pop), str(gens), mode, str(train),
                            str(held), d, str(jobs)], check=True, capture_output=True)
            ref_wall = time.time() - t0
            ref_log = open(os.path.join(d, "log.csv")).read()
        out[name]["reference_wall_s"] = ref_wall
        out[name]["reference_jobs"] = jobs
        out[name]["log_equals_reference_run"] = ref_log == log
        out[name]["speedup_vs_reference"] = ref_wall / wall
    print(name, json.dumps(out[name]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "search_time.json"), "w"), indent=1)
