"""Benchmark of the GEVO fitness-evaluation hot path on B200.

Workload (BASELINE.json configs[1], "config 2"): the Rodinia-style corpus
kernels hot-branch (hotspot), nw-sync (nw) and bfs-load (bfs); per kernel one
candidate batch of 1024 validated mutants -- the ~1016 `sanity_check` calls of
one pop-256 generation -- drawn as seeded random walks by the
product host, evaluated on the 16 synthetic train inputs of
generate_tests(b, 16, train_seed(1)) with the default 10^6 instruction budget
and tolerance 0 (mode default). One step = evaluate_fitness of all three
batches (3 x 1024 variants x 16 tests) on the device.

metric: variant x input evaluations/s = reference-equivalent executions
(tests the reference's evaluate_fitness runs: all of an accepted variant's,
else up to and including the first failing one) per second; IR instrs/s is
reported beside it. `value` times device-resident batches (CUDA events on the
launch stream, L2 flushed between steps); `e2e` times the C-ABI call with
host bytecode (H2D of the batch, D2H of the records inside the timed region).
The three batches are independent and are evaluated concurrently, each on its
own stream (gevo_eval_resident_async / _wait), so their launch tails overlap.

--impl reference times the reference's own CPU path (oracle/_ref/ref_bench:
validate + evaluate_fitness from /root/reference/proj/src compiled in place)
on the same candidate files with every host core.

Multi-GPU (torchrun, one process per GPU, NCCL): weak scaling -- each rank
evaluates its own candidate batches (seed 1 + rank); the per-variant fitness
records are exchanged with an NCCL all-gather and the gathered population is
ranked by the GPU non-dominated sort (the north star's only exchange step).
"""
from __future__ import annotations

import argparse
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

KERNELS = ("hot-branch", "nw-sync", "bfs-load")
N_VARIANTS = 1024
N_TESTS = 16
MASTER_SEED = 1
MAX_DEPTH = 4
METRIC = "variant x input evaluations/s"
UNIT = "evals/s"
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
ISSUE_PROFILE = os.path.join(ROOT, "profiles", "issue_per_launch.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--variants", type=int, default=N_VARIANTS)
    ap.add_argument("--tests", type=int, default=N_TESTS)
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="bound of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def workload_config(args, world, backend="nccl"):
    return {
        "workload": "config2: GEVO candidate batches, Rodinia-style IR kernels "
                    "hot-branch/nw-sync/bfs-load, %d validated mutants per kernel x %d "
                    "synthetic test inputs, budget 1e6, tol 0, seed %d" %
                    (args.variants, args.tests, MASTER_SEED),
        "kernels": list(KERNELS),
        "variants_per_kernel_per_gpu": args.variants,
        "tests": args.tests,
        "budget": 1_000_000,
        "tolerance": 0.0,
        "parallelism": "population-sharded dp%d (fitness records all-gathered over %s)" %
                       (world, "NCCL" if backend == "nccl" else backend),
        "l2": "flushed between timed steps (512 MiB write)",
    }


def write_candidates(gevo, seed, n, outdir):
    files = {}
    for k in KERNELS:
        lines = gevo.sample_candidates(k, n, seed, MAX_DEPTH)
        path = os.path.join(outdir, "cand_%s_%d.txt" % (k, seed))
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
        files[k] = (path, lines)
    return files


def run_ref_bench(files, n_tests, test_seed, threads, max_seconds):
    """Reference CPU path over every kernel's candidates; returns totals."""
    if not os.path.exists(REF_BENCH):
        raise RuntimeError("oracle/_ref/ref_bench missing: run __graft_entry__.build() "
                           "in the container that has /root/reference")
    tot = {"executions": 0, "ir": 0, "seconds": 0.0, "variants": 0}
    per = max_seconds / len(files)
    for k, (path, _) in files.items():
        out = subprocess.run([REF_BENCH, k, path, str(n_tests), str(test_seed), str(threads),
                              str(per)], check=True, capture_output=True, text=True).stdout
        r = json.loads(out.strip().splitlines()[-1])
        for key in tot:
            tot[key] += r[key]
    return tot


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


def reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import paper_2004_08140_b200 as gevo
    threads = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as tmp:
        files = write_candidates(gevo, MASTER_SEED, args.variants, tmp)
        seed = gevo.train_seed(MASTER_SEED)
        budget = max(args.cpu_seconds, 5.0) * 3
        for _ in range(args.warmup):
            run_ref_bench(files, args.tests, seed, threads, budget)
        tot = {"executions": 0, "ir": 0, "seconds": 0.0, "variants": 0}
        for _ in range(args.steps):
            r = run_ref_bench(files, args.tests, seed, threads, budget)
            for k in tot:
                tot[k] += r[k]
    value = tot["executions"] / tot["seconds"]
    sample = ("%d of %d candidates per step (3 kernels x %d) x %d tests, evaluate_fitness "
              "with early exit, %d threads" % (tot["variants"] // max(args.steps, 1),
                                               3 * args.variants, args.variants, args.tests,
                                               threads))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * tot["seconds"] / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32",
        "data": "synthetic", "config": workload_config(args, 1),
        "ir_per_s": tot["ir"] / tot["seconds"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def b200_arm(args):
    import numpy as np
    import torch
    import paper_2004_08140_b200 as gevo
    from paper_2004_08140_b200 import dist as gdist

    rank, local, world = dist_env()
    # one process per GPU; more ranks than GPUs (a functional check of the
    # N > 1 path on a smaller box) share devices round-robin
    shared = world > torch.cuda.device_count()
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    os.environ["GEVO_DEVICE"] = str(local)
    # NCCL needs a distinct GPU per rank: ranks sharing a device exchange over gloo
    backend = os.environ.get("BENCH_DIST_BACKEND", "gloo" if shared else "nccl")
    coll_dev = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.current_stream()
    gevo.set_stream(stream.cuda_stream)

    tmp = tempfile.mkdtemp(prefix="gevo_bench_")
    files = write_candidates(gevo, MASTER_SEED + rank, args.variants, tmp)
    seed = gevo.train_seed(MASTER_SEED)
    suites, batches, cfgs = {}, {}, {}
    for k in KERNELS:
        suites[k] = gevo.Suite.from_benchmark(k, args.tests, seed)
        cfgs[k] = suites[k].exec_config()
        b = suites[k].batch()
        for line in files[k][1]:
            b.add_patch(line)
        b.make_resident()
        batches[k] = b

    gevo.spin_counters(reset=True)
    # One untimed pass with per-test records: device-executed IR (speculative
    # work included) for the issue-rate roofline.
    dev_ir = 0
    ref_execs_step = ref_ir_step = 0
    for k in KERNELS:
        v, t, _ = batches[k].eval(cfgs[k], tolerance=0.0, early_exit=True, tests=True)
        dev_ir += int(t["ir"].sum())
        ref_execs_step += int(v["execs_ref"].sum())
        ref_ir_step += int(v["ir_ref"].sum())

    spins = gevo.spin_counters(reset=True)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    gathered_front = None

    def exchange(vrec_list):
        # NCCL all-gather of per-variant fitness (cost_mean, error_max, accepted)
        # then the GPU non-dominated sort of the gathered population.
        nonlocal gathered_front
        rows = gdist.fitness_rows(np.concatenate(vrec_list))
        g = gdist.allgather_fitness(rows, device=coll_dev) if world > 1 else rows
        cost, err, _ = gdist.accepted_fitness(g)
        front, _, _ = gevo.rank(cost, err)
        gathered_front = front

    timed_launches = [0]
    kernel_ms = {k: [] for k in KERNELS}

    # launch order of the concurrent batches (records are still gathered in
    # KERNELS order)
    order = os.environ.get("BENCH_LAUNCH_ORDER", ",".join(KERNELS)).split(",")

    def step_resident():
        # the three batches are independent: each runs on its own stream and
        # their launches (and launch tails) overlap on the GPU
        for k in order:
            batches[k].eval_resident_async(cfgs[k], tolerance=0.0, early_exit=True)
        recs = []
        for k in KERNELS:
            v, st = batches[k].wait(records=True)
            timed_launches[0] += st.launches
            kernel_ms[k].append(st.device_ms)
            recs.append(v)
        return recs

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        exchange(step_resident())
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    timed_launches[0] = 0
    for k in KERNELS:
        kernel_ms[k].clear()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            recs = step_resident()
            ev[i][1].record(stream)
            exchange(recs)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    dev_ms = sum(step_ms)

    # e2e through the C ABI with host bytecode (H2D + kernels + D2H records)
    def step_e2e():
        for k in order:
            batches[k].eval_resident_async(cfgs[k], tolerance=0.0, early_exit=True, upload=True)
        return [batches[k].wait(records=True)[1] for k in KERNELS]

    for _ in range(args.warmup):
        step_e2e()
    barrier()
    h2d = d2h = 0
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches = 0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev2[i][0].record(stream)
        h2d = d2h = 0
        # C-ABI evaluations with the host bytecode uploaded inside the timed
        # region and the records read back, the three batches concurrently
        for st in step_e2e():
            h2d += st.h2d_bytes
            d2h += st.d2h_bytes
            launches += st.launches
        ev2[i][1].record(stream)
    barrier()
    e2e_ms = sum(a.elapsed_time(b) for a, b in ev2)

    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = t.tolist()

    total_execs = ref_execs_step * args.steps * world
    value = total_execs / (dev_ms / 1000.0)
    e2e_value = total_execs / (e2e_ms / 1000.0)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    # Roofline: the interpreter is issue-slot bound -- integer
    # dispatch, no dense contraction, per-test working sets that live on chip.
    # achieved = SASS warp instructions the interpreter launches issue per step
    # (smsp__inst_executed.sum per launch, ncu, profiles/issue_per_launch.json)
    # / the step's CUDA-event time measured here (the batches run concurrently); peak = 148 SM x 4
    # schedulers x 1 warp instruction per cycle at the median SM clock under
    # load. traffic = DRAM bytes per launch of the dominant (hot-branch) launch.
    ck = clocks.summary()
    f_mhz = ck["sm_mhz"] or 1965.0
    peak = 148 * 4 * f_mhz * 1e6 / 1e9
    achieved = traffic = None
    per_kernel = {}
    if os.path.exists(ISSUE_PROFILE):
        prof = json.load(open(ISSUE_PROFILE))["kernels"]
        inst = sum(prof[k]["warp_inst"] for k in KERNELS if k in prof)
        # the three batches overlap on the GPU: the step time (CUDA events on
        # the launch stream) is the time their launches take together
        live_ms = dev_ms / args.steps
        if inst and live_ms and all(k in prof for k in KERNELS):
            achieved = inst / (live_ms / 1e3) / 1e9
        dom = prof.get(KERNELS[0], {})
        traffic = dom.get("dram_bytes")
        for k in KERNELS:
            if k in prof:
                per_kernel[k] = {"live_ms": round(statistics.mean(kernel_ms[k]), 4),
                                 "ncu_ms": prof[k].get("ncu_ms"),
                                 "warp_inst": prof[k]["warp_inst"],
                                 "lanes_per_warp_inst": (prof[k]["thread_inst"] /
                                                         prof[k]["warp_inst"])
                                 if prof[k].get("thread_inst") else None}
    # Secondary (HBM) view: DRAM bytes the interpreter launches move (ncu, per
    # launch) over their live time, against the measured copy bandwidth. The
    # per-test working sets (<= ~5 KB) stay in L2 / shared memory, so this is
    # tiny by construction -- the interpreter is not memory-bound.
    hbm_view = None
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, hbm_src = peaks["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        hbm_peak, hbm_src = 7700.0, "B200_PROFILING.md fallback"
    if per_kernel and os.path.exists(ISSUE_PROFILE):
        prof = json.load(open(ISSUE_PROFILE))["kernels"]
        dram = sum(prof[k].get("dram_bytes") or 0 for k in KERNELS if k in prof)
        live_ms = dev_ms / args.steps
        gbs = dram / (live_ms / 1e3) / 1e9 if live_ms else 0.0
        hbm_view = {"achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak,
                    "peak_source": hbm_src}
    roofline = {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "Gwarp-inst/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_unit": "DRAM bytes per hot-branch launch (ncu)",
                "per_kernel": per_kernel,
                "hbm_view": hbm_view,
                "note": "peak = 148 SM x 4 schedulers x 1 warp-inst/cycle x median SM clock"}

    cpu = None
    if not args.no_cpu_baseline and world == 1 and os.path.exists(REF_BENCH):
        threads = os.cpu_count() or 1
        r = run_ref_bench(files, args.tests, seed, threads, args.cpu_seconds)
        cpu = {"value": r["executions"] / r["seconds"], "unit": UNIT, "cores": threads,
               "kind": "reference",
               "sample": "%d of %d candidates (3 kernels) x %d tests, reference validate + "
                         "evaluate_fitness, %.1f s bound" % (r["variants"], 3 * args.variants,
                                                             args.tests, args.cpu_seconds),
               "ir_per_s": r["ir"] / r["seconds"]}
    shutil.rmtree(tmp, ignore_errors=True)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32 (IEEE, no FMA) + f64 error",
        "data": "synthetic (seeded generate_tests inputs, seeded mutant walks)",
        "config": workload_config(args, world, backend),
        "ir_per_s": ref_ir_step * args.steps * world / (dev_ms / 1000.0),
        "executions_per_step": ref_execs_step * world,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": timed_launches[0],
        "gpu_launches_e2e": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": ck,
        "step_ms": [round(x, 4) for x in step_ms],
        "spin_accelerator": {"loops_jumped_per_step": spins[0],
                             "instructions_skipped_per_step": spins[1]},
    }
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
