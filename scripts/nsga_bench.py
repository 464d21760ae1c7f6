"""rank_population + select_best at the pool sizes of configs 4-5 on the GPU,
beside the reference's own implementation on the host (oracle/_ref/ref_dump
nsga_bin: src/nsga.cpp compiled in place, one core -- the reference ranks on
the engine's thread, src/engine.cpp:258-262).

  python scripts/nsga_bench.py [--sizes 5120,20480,81920] [--no-ref] > nsga.jsonl

Fitness sets: oracle/gen_golden_nsga_large.fits (the same instances whose
reference digests tests/test_gpu_nsga_large.py checks). GPU time: CUDA events
around the ranking kernels (median of 7), and wall time of the C-ABI call
(H2D of the fitness vectors + kernels + D2H of the keep order)."""
import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

spec = importlib.util.spec_from_file_location(
    "gen_nsga_large", os.path.join(ROOT, "oracle", "gen_golden_nsga_large.py"))
G = importlib.util.module_from_spec(spec)
spec.loader.exec_module(G)
REF = os.path.join(ROOT, "oracle", "_ref", "ref_dump")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="5120,20480,81920")
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    for n in [int(x) for x in a.sizes.split(",")]:
        for dist in G.DISTS:
            c, e = G.fits(dist, n)
            keep = G.keep_of(n)
            gevo.select_best(c, e, keep)  # warm-up (buffers, module)
            dev, wall = [], []
            for _ in range(7):
                t0 = time.perf_counter()
                _, ms = gevo.select_best(c, e, keep)
                wall.append((time.perf_counter() - t0) * 1e3)
                dev.append(ms)
            row = {"n": n, "dist": dist, "keep": keep, "device_ms": statistics.median(dev),
                   "call_ms": statistics.median(wall)}
            if not a.no_ref and os.path.exists(REF):
                with tempfile.TemporaryDirectory() as d:
                    pin, pout = os.path.join(d, "in.bin"), os.path.join(d, "out.bin")
                    with open(pin, "wb") as f:
                        f.write(np.int64(n).tobytes() + c.tobytes() + e.tobytes())
                    r = json.loads(subprocess.run([REF, "nsga_bin", pin, str(keep), pout],
                                                  check=True, capture_output=True,
                                                  text=True).stdout)
                row["reference_ms"] = r["rank_select_s"] * 1e3
                row["speedup_call"] = row["reference_ms"] / row["call_ms"]
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
