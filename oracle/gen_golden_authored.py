"""Golden records of the authored config-3/4 kernels from the compiled
reference (oracle/_ref/ref_dump authored). TEST INFRASTRUCTURE: run in the
container that has /root/reference; writes tests/golden/authored_<name>.jsonl.gz.
Reduced sizes (40 SVM rows, 1024 conv outputs) keep the fixtures small; the
first line holds the generator spec and seed so tests regenerate the inputs.

  python oracle/gen_golden_authored.py          reduced sizes (40 mutants)
  python oracle/gen_golden_authored.py --full   BASELINE shapes (a9a 32561x123,
      CIFAR conv 64x32x32 outputs), 256 mutants + the original, 3 tests,
      budget 1e6, tol 0.01 -> tests/golden/authored_full_<name>.jsonl.gz
      (the reference runs ~1 s per execution here, so the patches are split
      over every host core, one ref_dump process per shard, records kept in
      patch order)"""
import gzip
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

SIZES = {"svm-rbf": 40, "conv-bn": 1024}
N_TESTS, SEED, BUDGET, TOL, N_MUTANTS = 2, 7, 200000, 0.01, 40


def resize(name, gen_json, scale):
    g = json.loads(gen_json)
    for b in g["buffers"]:
        if name == "svm-rbf" and b["name"] == "X":
            b["size"] = scale * 123
        if (name == "svm-rbf" and b["name"] == "K") or (name == "conv-bn" and b["name"] == "out"):
            b["size"] = scale
    for sc in g["scalars"]:
        if sc["name"] in ("n", "total"):
            sc["value"] = scale
    return json.dumps(g)


def run_sharded(ref, d, n_tests, seed, cands, budget, tol, shards):
    """ref_dump authored over contiguous shards of the patch list, in parallel."""
    per = (len(cands) + shards - 1) // shards
    procs = []
    for s in range(shards):
        part = cands[s * per:(s + 1) * per]
        if not part:
            break
        pp = os.path.join(d, "p%d.txt" % s)
        with open(pp, "w") as f:
            f.write("\n".join(part) + "\n")
        procs.append(subprocess.Popen([ref, "authored", os.path.join(d, "k.ir"), os.path.join(d, "g.json"),
                                       str(n_tests), str(seed), pp, str(budget), str(tol)],
                                      stdout=subprocess.PIPE, text=True))
    outs = []
    for s, p in enumerate(procs):
        out, _ = p.communicate()
        assert p.returncode == 0, s
        lines = out.splitlines()
        # records carry the patch index within their shard: renumber globally
        for ln in lines:
            r = json.loads(ln)
            r["i"] = r["i"] + s * per
            outs.append(json.dumps(r))
    return "\n".join(outs) + "\n"


def main_full():
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_dump")
    n_tests, seed, budget, tol, n_mut = 3, 7, 1000000, 0.01, 256
    for name in ("conv-bn", "svm-rbf"):
        ir, gen = gevo.authored_kernel(name)
        cands = ["[]"] + gevo.sample_candidates_ir(ir, n_mut, 5, 3)
        with tempfile.TemporaryDirectory() as d:
            for fn, text in (("k.ir", ir), ("g.json", gen)):
                with open(os.path.join(d, fn), "w") as f:
                    f.write(text)
            out = run_sharded(ref, d, n_tests, seed, cands, budget, tol, os.cpu_count() or 4)
        head = {"kind": "suite", "name": name, "gen": json.loads(gen), "n_tests": n_tests,
                "seed": seed, "budget": budget, "tol": tol}
        path = os.path.join(ROOT, "tests", "golden", "authored_full_%s.jsonl.gz" % name)
        with gzip.open(path, "wt", compresslevel=9) as f:
            f.write(json.dumps(head) + "\n" + out)
        print(path, len(out.splitlines()), "records", flush=True)


def main():
    if "--full" in sys.argv:
        return main_full()
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_dump")
    for name, scale in SIZES.items():
        ir, gen = gevo.authored_kernel(name)
        gen = resize(name, gen, scale)
        cands = ["[]"] + gevo.sample_candidates_ir(ir, N_MUTANTS, 3, 3)
        with tempfile.TemporaryDirectory() as d:
            for fn, text in (("k.ir", ir), ("g.json", gen), ("p.txt", "\n".join(cands) + "\n")):
                with open(os.path.join(d, fn), "w") as f:
                    f.write(text)
            out = subprocess.run([ref, "authored", os.path.join(d, "k.ir"), os.path.join(d, "g.json"),
                                  str(N_TESTS), str(SEED), os.path.join(d, "p.txt"), str(BUDGET),
                                  str(TOL)], check=True, capture_output=True, text=True).stdout
        head = {"kind": "suite", "name": name, "gen": json.loads(gen), "n_tests": N_TESTS,
                "seed": SEED, "budget": BUDGET, "tol": TOL}
        path = os.path.join(ROOT, "tests", "golden", "authored_%s.jsonl.gz" % name)
        with gzip.open(path, "wt", compresslevel=9) as f:
            f.write(json.dumps(head) + "\n" + out)
        print(path, len(out.splitlines()), "records")


if __name__ == "__main__":
    main()
