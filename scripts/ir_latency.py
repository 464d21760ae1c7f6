"""Per-IR latency of one lone interpreter lane (no other work on the GPU).

A one-thread kernel runs a counted loop whose body mixes the corpus's common
opcodes; with the spin accelerator off (GEVO_SPIN_THRESHOLD=0) every
instruction is interpreted. Prints ns and cycles per dynamic IR instruction
for the thread-parallel and the sequential-lane interpreter.
  GEVO_SPIN_THRESHOLD=0 python scripts/ir_latency.py [iterations]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
KERNELS = {
    "alu": """kernel k(a: ptr<global> f32, out: ptr<global> f32) threads=1 shared=0 {
entry:
  %0 = tid i32  #uid=0
  br loop  #uid=1
loop:
  %1 = phi i32 [0, entry], [%9, loop]  #uid=2
  %2 = phi f32 [0.0, entry], [%8, loop]  #uid=3
  %3 = add i32 %1, 7  #uid=4
  %4 = mul i32 %3, 3  #uid=5
  %5 = sub i32 %4, %1  #uid=6
  %6 = fadd f32 %2, 1.5  #uid=7
  %7 = fmul f32 %6, 0.5  #uid=8
  %8 = fadd f32 %7, %2  #uid=9
  %9 = add i32 %1, 1  #uid=10
  %10 = icmp.lt i32 %9, NITER  #uid=11
  br %10, loop, done  #uid=12
done:
  store out[%0], %8  #uid=13
  ret  #uid=14
}""",
    "mem": """kernel k(a: ptr<global> f32, out: ptr<global> f32) threads=1 shared=0 {
entry:
  %0 = tid i32  #uid=0
  br loop  #uid=1
loop:
  %1 = phi i32 [0, entry], [%9, loop]  #uid=2
  %2 = phi f32 [0.0, entry], [%8, loop]  #uid=3
  %3 = mul i32 %1, 0  #uid=4
  %4 = load f32 a[%3]  #uid=5
  %5 = fadd f32 %4, %2  #uid=6
  store out[%3], %5  #uid=7
  %6 = load f32 out[%3]  #uid=8
  %8 = fmul f32 %6, 0.5  #uid=9
  %9 = add i32 %1, 1  #uid=10
  %10 = icmp.lt i32 %9, NITER  #uid=11
  br %10, loop, done  #uid=12
done:
  store out[%0], %8  #uid=13
  ret  #uid=14
}""",
}

res = {}
for name, text in KERNELS.items():
    ir = text.replace("NITER", str(N))
    doc = {"inputs": {"a": {"type": "f32", "data": [1.0] * 4}, "out": {"type": "f32", "data": [0.0] * 4}},
           "scalars": {}, "oracle": {}}
    suite = gevo.Suite.from_json(ir, [json.dumps(doc)])
    cfg = suite.exec_config().with_(budget=100_000_000)
    b = suite.batch().add_ir(ir)
    for seq in (False, True):
        ms = []
        for _ in range(5):
            _, t, st = b.eval(cfg, tests=True, sequential=seq)
            ms.append(st.device_ms)
        n_ir = int(t[0, 0]["ir"])
        best = min(ms[1:])
        key = "%s/%s" % (name, "seq" if seq else "tp")
        res[key] = {"ir": n_ir, "ms": best, "ns_per_ir": best * 1e6 / n_ir,
                    "cycles_per_ir_1965": best * 1.965e6 / n_ir}
        print(key, json.dumps(res[key]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "ir_latency.json"), "w"), indent=1)
