"""Benchmark of the GEVO fitness-evaluation hot path on B200.

Headline workload (BASELINE.json configs[3], "config 4", the largest
single-GPU configuration): a candidate batch of 4096 validated mutants
(seeded random walks of up to 3 edits, the search's candidate stream;
bench_data/cand_conv-bn_s1.txt.gz) of the authored conv3x3 + bias + batch-norm
IR kernel (paper_2004_08140_b200/data/kernels/conv-bn: CIFAR-shaped
in[3x32x32] f32, w[64x3x3x3] -> out[64x32x32], 256 simulated threads) on the 3
seeded train inputs of generate_tests_for(kernel, spec, 3, train_seed(1)),
budget 10^6 instructions per simulated thread, tolerance 0.01, early exit
(the reference's evaluate_fitness stops at a variant's first failing test).
One step = evaluate_fitness of the whole batch on the device.

metric: variant x input evaluations/s = reference-equivalent executions (the
tests the reference's evaluate_fitness runs: all of an accepted variant's,
else up to and including the first failing one) per second; IR instrs/s is
reported beside it (reference-equivalent, and device-executed).
`value`: device-resident batch, CUDA events on the launching stream (the
caller's stream: the library launches on it, gevo_set_stream), L2 flushed by a
512 MiB write on that stream before every timed step. `e2e`: the same through
the C ABI with host bytecode -- H2D of the batch image and D2H of the records
inside the timed region. Validation is outside both arms' timed regions.

Config 2 (configs[1]: hot-branch / nw-sync / bfs-load, 1024 mutants each x 16
tests, tol 0) is measured in the same run and reported in `secondary`.

--impl reference times the reference's own CPU implementation
(oracle/_ref/ref_bench: /root/reference/proj/src compiled in place,
evaluate_fitness) on the same committed candidates with every host core, each
step a bounded sample; that arm never loads the product library.

Multi-GPU (torchrun, one process per GPU, NCCL): weak scaling -- rank r
evaluates its own 4096-candidate batch (seed 1 + r); the per-variant fitness
rows are exchanged with an NCCL all-gather, then rank_population +
select_best of the gathered pool run on the GPU (the north star's only
exchange step).
"""
from __future__ import annotations

import argparse
import gzip
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "variant x input evaluations/s"
UNIT = "evals/s"
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
ISSUE_PROFILE = os.path.join(ROOT, "profiles", "issue_per_launch.json")
BENCH_DATA = os.path.join(ROOT, "bench_data")
KERNEL_DIR = os.path.join(ROOT, "paper_2004_08140_b200", "data", "kernels")
MASTER_SEED = 1

C4 = {"name": "config4", "kernel": "conv-bn", "variants": 4096, "tests": 3, "tol": 0.01,
      "budget": 1_000_000, "depth": 3}
C2 = {"name": "config2", "kernels": ("hot-branch", "nw-sync", "bfs-load"), "variants": 1024,
      "tests": 16, "tol": 0.0, "budget": 1_000_000, "depth": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="bound of the cpu_baseline sample")
    ap.add_argument("--ref-step-seconds", type=float, default=8.0,
                    help="--impl reference: bound of each step's sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--profile-step", choices=["config4", "config2"],
                    help="one untimed step of that workload between cudaProfilerStart/Stop "
                         "(ncu --profile-from-start off), then exit")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def splitmix64(x):
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def train_seed(master):
    """src/cli_app.cpp:193-201 (the product exports the same as gevo_train_seed)."""
    return splitmix64(master ^ 0x7261696E5F736574)


def c4_config(world, backend="nccl"):
    return {
        "workload": "config4: GEVO candidate batch of %d validated mutants of the conv3x3+bias+"
                    "batch-norm IR kernel (CIFAR-shaped in[3x32x32] -> out[64x32x32] f32, 256 "
                    "simulated threads) x %d synthetic inputs, budget 1e6, tol %g, early exit, "
                    "seed %d" % (C4["variants"], C4["tests"], C4["tol"], MASTER_SEED),
        "kernel": C4["kernel"],
        "variants_per_gpu": C4["variants"],
        "tests": C4["tests"],
        "budget": C4["budget"],
        "tolerance": C4["tol"],
        "parallelism": "population-sharded dp%d (fitness rows all-gathered over %s, GPU "
                       "rank_population + select_best of the gathered pool)" %
                       (world, "NCCL" if backend == "nccl" else backend),
        "l2": "flushed before every timed step (512 MiB write on the launching stream)",
    }


def committed_candidates(kind, seed=MASTER_SEED):
    path = os.path.join(BENCH_DATA, "cand_%s_s%d.txt.gz" % (kind, seed))
    if not os.path.exists(path):
        return None
    with gzip.open(path, "rt") as f:
        return [ln for ln in f.read().splitlines() if ln.strip()]


def run_ref_bench(target, cand_lines, n_tests, seed, threads, seconds, budget, tol, start=0,
                  count=True):
    """The reference's evaluate_fitness over candidates (oracle/_ref/ref_bench)."""
    if not os.path.exists(REF_BENCH):
        raise RuntimeError("oracle/_ref/ref_bench missing: run __graft_entry__.build() in the "
                           "container that has /root/reference (it travels with the repo)")
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(cand_lines) + "\n")
        path = f.name
    try:
        env = dict(os.environ)
        if not count:
            env["REF_BENCH_NOCOUNT"] = "1"
        out = subprocess.run([REF_BENCH, target, path, str(n_tests), str(seed), str(threads),
                              str(seconds), str(budget), str(tol), str(start)],
                             check=True, capture_output=True, text=True, env=env).stdout
    finally:
        os.unlink(path)
    return json.loads(out.strip().splitlines()[-1])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path, no product code loaded


def reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    cands = committed_candidates(C4["kernel"])
    if cands is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "bench_data/cand_conv-bn_s1.txt.gz missing"}))
        return
    threads = os.cpu_count() or 1
    target = "file:" + os.path.join(KERNEL_DIR, C4["kernel"])
    seed = train_seed(MASTER_SEED)
    tot = {"executions": 0, "ir": 0, "seconds": 0.0, "variants": 0}
    ir_s = None
    # each step: a bounded sample of the batch, starting at a different variant
    stride = 97
    for i in range(args.warmup + args.steps):
        r = run_ref_bench(target, cands, C4["tests"], seed, threads, args.ref_step_seconds,
                          C4["budget"], C4["tol"], start=(i * stride) % len(cands),
                          count=i == args.warmup)
        if i == args.warmup:
            ir_s = r["ir"] / r["seconds"]
        if i >= args.warmup:
            for k in tot:
                tot[k] += r[k]
    value = tot["executions"] / tot["seconds"]
    sample = ("per step %.0f variants of the %d-candidate batch (from a rotating start) x %d "
              "inputs, reference evaluate_fitness with early exit (validation untimed), "
              "%d threads, %.0f s bound" % (tot["variants"] / max(args.steps, 1), len(cands),
                                            C4["tests"], threads, args.ref_step_seconds))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * tot["seconds"] / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32",
        "data": "synthetic (seeded generate_tests_for inputs, committed seeded mutant walks)",
        "config": c4_config(1),
        "ir_per_s": ir_s,  # IR counted (untimed re-run at unit cost) on the first timed step
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------
# B200 arm


def issue_profile(workload):
    if not os.path.exists(ISSUE_PROFILE):
        return None
    prof = json.load(open(ISSUE_PROFILE))
    return prof.get("workloads", {}).get(workload)


def useful_ir_fraction(v, t):
    """Reference-equivalent instructions of the tests the reference runs (each
    variant's tests up to its first failing one; all of them when it passes) /
    those of every test the device ran, from one pass with per-test records."""
    import numpy as np
    ir = t["ir"].astype(np.float64)
    ff = v["failing_test"].astype(np.int64)
    idx = np.arange(ir.shape[1])[None, :]
    ref_run = (ff[:, None] < 0) | (idx <= ff[:, None])
    total = float(ir.sum())
    return float(ir[ref_run].sum()) / total if total > 0 else None


def roofline_of(workload, step_ms, f_mhz, ir_ref_step, ir_dev_step):
    """Issue-slot roofline: the interpreter is integer dispatch
    with per-test working sets on chip. achieved = SASS warp instructions the
    step's interpreter launches issue (ncu smsp__inst_executed.sum summed over
    the launches of one step, profiles/issue_per_launch.json) / the step's
    CUDA-event time; peak = 148 SM x 4 schedulers x 1 warp-instruction/cycle at
    the median SM clock under load."""
    peak = 148 * 4 * f_mhz * 1e6 / 1e9
    prof = issue_profile(workload)
    out = {"bound": "issue", "achieved": None, "peak": peak, "unit": "Gwarp-inst/s",
           "frac": None, "traffic": None, "traffic_unit": "DRAM bytes per step (ncu)",
           "note": "peak = 148 SM x 4 schedulers x 1 warp-inst/cycle x median SM clock"}
    if not prof or not step_ms:
        return out
    achieved = prof["warp_inst"] / (step_ms / 1e3) / 1e9
    out.update({"achieved": achieved, "frac": achieved / peak, "traffic": prof.get("dram_bytes"),
                "launches_profiled": prof.get("launches"),
                "lanes_per_warp_inst": (prof["thread_inst"] / prof["warp_inst"])
                if prof.get("thread_inst") else None,
                "ncu_ms_per_step": prof.get("ncu_ms")})
    # device-executed (interpreted) instructions per issued warp instruction,
    # and the issue fraction scaled to the reference-equivalent work: the
    # reference runs ir_ref instructions for this step, the device
    # interpreted ir_dev (jumps make it smaller, discarded speculative work
    # larger)
    if ir_dev_step:
        out["interpreted_ir_per_step"] = ir_dev_step
        out["warp_inst_per_interpreted_ir"] = prof["warp_inst"] / ir_dev_step
        out["reference_ir_per_interpreted_ir"] = ir_ref_step / ir_dev_step
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, src = peaks["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        hbm_peak, src = 7700.0, "B200_PROFILING.md fallback"
    if prof.get("dram_bytes") is not None:
        gbs = prof["dram_bytes"] / (step_ms / 1e3) / 1e9
        out["hbm_view"] = {"achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak,
                           "peak_source": src}
    return out


def b200_arm(args):
    import numpy as np
    import torch
    import paper_2004_08140_b200 as gevo
    from paper_2004_08140_b200 import dist as gdist

    rank, local, world = dist_env()
    shared = world > torch.cuda.device_count()
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    os.environ["GEVO_DEVICE"] = str(local)
    backend = os.environ.get("BENCH_DIST_BACKEND", "gloo" if shared else "nccl")
    coll_dev = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    # every library launch goes to this stream, so CUDA events recorded on it
    # bracket the work (and the L2 flush on it precedes the work)
    stream = torch.cuda.Stream()
    gevo.set_stream(stream.cuda_stream)
    seed = gevo.train_seed(MASTER_SEED)
    assert seed == train_seed(MASTER_SEED)

    # ---- config 4 batch
    ir, gen = gevo.authored_kernel(C4["kernel"])
    cands = committed_candidates(C4["kernel"], MASTER_SEED + rank)
    if cands is None:
        cands = gevo.sample_candidates_ir(ir, C4["variants"], MASTER_SEED + rank, C4["depth"])
    suite = gevo.Suite.from_spec(ir, gen, C4["tests"], seed)
    cfg = suite.exec_config().with_(budget=C4["budget"])
    batch = suite.batch()
    for line in cands:
        batch.add_patch(line)
    batch.make_resident()

    # ---- config 2 batches (secondary)
    c2 = {}
    if not args.no_secondary and not args.profile_step == "config4":
        for k in C2["kernels"]:
            lines = committed_candidates(k, MASTER_SEED + rank) or \
                gevo.sample_candidates(k, C2["variants"], MASTER_SEED + rank, C2["depth"])
            s2 = gevo.Suite.from_benchmark(k, C2["tests"], seed)
            b2 = s2.batch()
            for line in lines:
                b2.add_patch(line)
            b2.make_resident()
            c2[k] = (s2, b2, s2.exec_config())

    if args.profile_step:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        if args.profile_step == "config4":
            batch.eval_resident(cfg, tolerance=C4["tol"], early_exit=True, records=True)
        else:
            for k in C2["kernels"]:
                c2[k][1].eval_resident_async(c2[k][2], tolerance=C2["tol"], early_exit=True)
            for k in C2["kernels"]:
                c2[k][1].wait(records=True)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"profile_step": args.profile_step}))
        return

    # untimed pass with per-test records: reference-equivalent and
    # device-executed work of one step
    gevo.spin_counters(reset=True)
    gevo.work_counters(reset=True)
    v, t, _ = batch.eval(cfg, tolerance=C4["tol"], early_exit=True, tests=True)
    execs_step = int(v["execs_ref"].sum())
    ir_ref_step = int(v["ir_ref"].sum())
    # instructions the device actually interpreted in the step: spin jumps
    # excluded, speculative tests / aborted threads / re-runs included
    ir_dev_step = gevo.work_counters(reset=True)
    spins = gevo.spin_counters(reset=True)
    useful = useful_ir_fraction(v, t)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def exchange(vrec):
        # NCCL all-gather of per-variant fitness (cost_mean, error_max,
        # accepted), then rank_population + select_best of the gathered pool
        rows = gdist.fitness_rows(vrec)
        g = gdist.allgather_fitness(rows, device=coll_dev) if world > 1 else rows
        cost, err, _ = gdist.accepted_fitness(g)
        keep = len(cost) * 4 // 5
        return gevo.select_best(cost, err, keep)

    def timed(step_fn, k, w):
        for _ in range(w):
            step_fn(None)
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(k)]
        for i in range(k):
            step_fn(ev[i])
        barrier()
        return [a.elapsed_time(b) for a, b in ev]

    lib_ms, launches, rank_ms = [], [0], []

    def step_resident(ev):
        with torch.cuda.stream(stream):
            flush.fill_(1)
            if ev:
                ev[0].record(stream)
            vrec, st = batch.eval_resident(cfg, tolerance=C4["tol"], early_exit=True, records=True)
            if ev:
                ev[1].record(stream)
                lib_ms.append(st.device_ms)
                launches[0] += st.launches
        _, ms = exchange(vrec)
        if ev:
            rank_ms.append(ms)

    with ClockSampler(local) as clocks:
        step_ms = timed(step_resident, args.steps, args.warmup)
    dev_ms = sum(step_ms)

    h2d = d2h = 0
    e2e_launches = [0]

    def step_e2e(ev):
        nonlocal h2d, d2h
        with torch.cuda.stream(stream):
            flush.fill_(2)
            if ev:
                ev[0].record(stream)
            batch.eval_resident_async(cfg, tolerance=C4["tol"], early_exit=True, upload=True)
            _, st = batch.wait(records=True)
            if ev:
                ev[1].record(stream)
                h2d, d2h = st.h2d_bytes, st.d2h_bytes
                e2e_launches[0] += st.launches

    e2e_ms = sum(timed(step_e2e, args.steps, args.warmup))

    # host pipeline beside it (diagnostic, wall clock, one pass): patches ->
    # apply_patch + encode -> H2D -> evaluate -> records
    t0 = time.perf_counter()
    b_host = suite.batch()
    for line in cands:
        b_host.add_patch(line)
    t1 = time.perf_counter()
    b_host.eval(cfg, tolerance=C4["tol"], early_exit=True)
    t2 = time.perf_counter()
    host_pipeline = {"encode_s": t1 - t0, "eval_s": t2 - t1,
                     "value": execs_step / (t2 - t0), "unit": UNIT,
                     "note": "patches applied, encoded, uploaded and evaluated through the C ABI "
                             "(wall clock, one pass)"}
    del b_host

    sec = None
    if c2:
        sec = secondary_config2(args, gevo, torch, stream, flush, c2, barrier, world)

    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = tt.tolist()

    total_execs = execs_step * args.steps * world
    value = total_execs / (dev_ms / 1000.0)
    e2e_value = total_execs / (e2e_ms / 1000.0)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    ck = clocks.summary()
    f_mhz = ck["sm_mhz"] or 1965.0
    roofline = roofline_of("config4", dev_ms / args.steps, f_mhz, ir_ref_step, ir_dev_step)
    if roofline.get("frac") is not None and useful is not None:
        # the share of the step's work the reference also does: tests up to and
        # including each variant's first failing test (the rest is speculative
        # work early exit discards), in reference-equivalent instructions
        roofline["useful_ir_frac"] = useful
        roofline["useful_frac"] = roofline["frac"] * useful
    roofline["lib_ms_per_step"] = statistics.mean(lib_ms) if lib_ms else None

    cpu = None
    if not args.no_cpu_baseline and world == 1 and os.path.exists(REF_BENCH):
        threads = os.cpu_count() or 1
        r = run_ref_bench("file:" + os.path.join(KERNEL_DIR, C4["kernel"]), cands, C4["tests"],
                          seed, threads, args.cpu_seconds, C4["budget"], C4["tol"], count=False)
        cpu = {"value": r["executions"] / r["seconds"], "unit": UNIT, "cores": threads,
               "kind": "reference",
               "sample": "first %d of %d candidates x %d inputs, reference evaluate_fitness "
                         "(validation untimed), %.0f s bound" %
                         (r["variants"], len(cands), C4["tests"], args.cpu_seconds)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32 (IEEE, no FMA) + f64 error",
        "data": "synthetic (seeded generate_tests_for inputs, committed seeded mutant walks)",
        "config": c4_config(world, backend),
        "executions_per_step": execs_step * world,
        "ir_per_s": ir_ref_step * args.steps * world / (dev_ms / 1000.0),
        "device_ir_per_s": ir_dev_step * args.steps * world / (dev_ms / 1000.0),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches[0],
        "gpu_launches_e2e": e2e_launches[0],
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": ck,
        "step_ms": [round(x, 3) for x in step_ms],
        "rank_select_ms": round(statistics.mean(rank_ms), 4) if rank_ms else None,
        "host_pipeline": host_pipeline,
        "spin_accelerator": {"loops_jumped_per_step": spins[0],
                             "instructions_skipped_per_step": spins[1]},
        "secondary": sec,
    }
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def secondary_config2(args, gevo, torch, stream, flush, c2, barrier, world):
    """Config 2: the three corpus batches evaluated concurrently (each on its
    own stream, ordered after the caller's stream) -- value and e2e."""
    ks = C2["kernels"]
    execs = ir_ref = 0
    for k in ks:
        s2, b2, cfg2 = c2[k]
        v, _, _ = b2.eval(cfg2, tolerance=C2["tol"], early_exit=True)
        execs += int(v["execs_ref"].sum())
        ir_ref += int(v["ir_ref"].sum())

    def run(upload, ev):
        with torch.cuda.stream(stream):
            flush.fill_(3)
            if ev:
                ev[0].record(stream)
            for k in ks:
                c2[k][1].eval_resident_async(c2[k][2], tolerance=C2["tol"], early_exit=True,
                                             upload=upload)
            sts = [c2[k][1].wait(records=True)[1] for k in ks]
            if ev:
                ev[1].record(stream)
        return sts

    def timed(upload):
        for _ in range(args.warmup):
            run(upload, None)
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        live = []
        for i in range(args.steps):
            sts = run(upload, ev[i])
            live.append(max(s.device_ms for s in sts))
        barrier()
        return [a.elapsed_time(b) for a, b in ev], live

    steps, live = timed(False)
    e2e_steps, _ = timed(True)
    ms = statistics.mean(steps)
    return {
        "workload": "config2: hot-branch/nw-sync/bfs-load, %d validated mutants each x %d "
                    "synthetic inputs, budget 1e6, tol 0, the three batches concurrently" %
                    (C2["variants"], C2["tests"]),
        "value": execs * world / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
        "e2e": {"value": execs * world / (statistics.mean(e2e_steps) / 1e3), "unit": UNIT},
        "ir_per_s": ir_ref * world / (ms / 1e3),
        "executions_per_step": execs * world,
        # per step: the longest batch's own device span next to the step's
        # window (the batches run inside the window: live <= step)
        "step_ms": [round(x, 4) for x in steps],
        "batch_live_ms": [round(x, 4) for x in live],
        "live_within_step": all(l <= s + 1e-3 for l, s in zip(live, steps)),
        "roofline": roofline_of("config2", ms, 1965.0, ir_ref, None),
    }


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
