"""Builds paper_2004_08140_b200/data/corpus.json from the reference's shipped
benchmark data (/root/reference/proj/data/benchmarks/*: kernel IR, generator
spec, reach patch). The six planted-inefficiency kernels are workload DATA the
search runs on; the product embeds this file at build time. Run once here
(the reference tree is not present on the GPU box):

    python paper_2004_08140_b200/data/make_corpus_data.py
"""
import json
import os
import sys

SRC = "/root/reference/proj/data/benchmarks"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "corpus.json")


def main():
    names = sorted(f[:-3] for f in os.listdir(SRC) if f.endswith(".ir") and ".improved" not in f)
    out = []
    for n in names:
        spec = json.load(open(os.path.join(SRC, n + ".json")))
        out.append({
            "name": n,
            "class": spec["planted_class"],
            "notes": spec["notes"],
            "ir": open(os.path.join(SRC, n + ".ir")).read(),
            "reach": json.load(open(os.path.join(SRC, n + ".patch.json"))),
            "buffers": spec["buffers"],
            "scalars": spec.get("scalars", []),
        })
    with open(DST, "w") as f:
        json.dump({"benchmarks": out}, f, indent=1, sort_keys=True)
        f.write("\n")
    print("wrote", DST, len(out), "benchmarks", file=sys.stderr)


if __name__ == "__main__":
    main()
