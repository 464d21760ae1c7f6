"""Writes the committed bench workload: seeded candidate patches (validated
random-walk mutants, as the search's candidate stream) for bench.py, so the
reference arm reads the same candidates without loading the product library.

  python scripts/gen_bench_candidates.py      -> bench_data/*.txt.gz

config 4: conv-bn (authored CIFAR-shaped conv3x3+bias+batch-norm), 4096
mutants of up to 3 edits, seed 1. config 2: hot-branch / nw-sync / bfs-load,
1024 mutants of up to 4 edits each, seed 1; rank r of a multi-GPU bench reads
seed 1 + r (seeds 1-8 are committed: one node of 8 GPUs).

  python scripts/gen_bench_candidates.py [seeds, default 1-8]"""
import gzip
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

OUT = os.path.join(ROOT, "bench_data")


def candidates(kind, seed):
    if kind == "conv-bn":
        ir, _ = gevo.authored_kernel("conv-bn")
        return gevo.sample_candidates_ir(ir, 4096, seed, 3)
    return gevo.sample_candidates(kind, 1024, seed, 4)


def main():
    os.makedirs(OUT, exist_ok=True)
    seeds = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(1, 9)
    for seed in seeds:
        for k in ("conv-bn", "hot-branch", "nw-sync", "bfs-load"):
            write(k, seed)


def write(k, seed):
    lines = candidates(k, seed)
    path = os.path.join(OUT, "cand_%s_s%d.txt.gz" % (k, seed))
    with gzip.GzipFile(path, "wb", compresslevel=9, mtime=0) as f:  # (reproducible bytes)
        f.write(("\n".join(lines) + "\n").encode())
    print(path, len(lines))


if __name__ == "__main__":
    main()
