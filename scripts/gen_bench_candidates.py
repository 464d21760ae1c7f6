"""Writes the committed bench workload: seeded candidate patches (validated
random-walk mutants, as the search's candidate stream) for bench.py, so the
reference arm reads the same candidates without loading the product library.

  python scripts/gen_bench_candidates.py      -> bench_data/*.txt.gz

config 4: conv-bn (authored CIFAR-shaped conv3x3+bias+batch-norm), 4096
mutants of up to 3 edits, seed 1. config 2: hot-branch / nw-sync / bfs-load,
1024 mutants of up to 4 edits each, seed 1. Ranks > 0 of a multi-GPU bench
draw their own batches with seed 1 + rank at run time."""
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
    for k in ("conv-bn", "hot-branch", "nw-sync", "bfs-load"):
        lines = candidates(k, 1)
        path = os.path.join(OUT, "cand_%s_s1.txt.gz" % k)
        with gzip.open(path, "wt", compresslevel=9) as f:
            f.write("\n".join(lines) + "\n")
        print(path, len(lines))


if __name__ == "__main__":
    main()
