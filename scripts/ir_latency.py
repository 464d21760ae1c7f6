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
    "alu16": """kernel k(a: ptr<global> f32, out: ptr<global> f32) threads=1 shared=0 {
entry:
  %0 = tid i32  #uid=0
  br loop  #uid=1
loop:
  %1 = phi i32 [0, entry], [%9, loop]  #uid=2
  %99 = add i32 %1, 1  #uid=99
  %101 = mul i32 %99, 5  #uid=101
  %102 = add i32 %101, 3  #uid=102
  %103 = mul i32 %102, 5  #uid=103
  %104 = add i32 %103, 3  #uid=104
  %105 = mul i32 %104, 5  #uid=105
  %106 = add i32 %105, 3  #uid=106
  %107 = mul i32 %106, 5  #uid=107
  %108 = add i32 %107, 3  #uid=108
  %109 = mul i32 %108, 5  #uid=109
  %110 = add i32 %109, 3  #uid=110
  %111 = mul i32 %110, 5  #uid=111
  %112 = add i32 %111, 3  #uid=112
  %113 = mul i32 %112, 5  #uid=113
  %114 = add i32 %113, 3  #uid=114
  %115 = mul i32 %114, 5  #uid=115
  %116 = add i32 %115, 3  #uid=116
  %9 = add i32 %1, 1  #uid=10
  %10 = icmp.lt i32 %9, NITER  #uid=11
  br %10, loop, done  #uid=12
done:
  ret  #uid=14
}""",
    "smem": """kernel k(a: ptr<global> f32, out: ptr<global> f32, s: ptr<shared> f32) threads=1 shared=16 {
entry:
  %0 = tid i32  #uid=0
  store s[%0], 0.0  #uid=20
  br loop  #uid=1
loop:
  %1 = phi i32 [0, entry], [%9, loop]  #uid=2
  %2 = phi f32 [0.0, entry], [%8, loop]  #uid=3
  %3 = mul i32 %1, 0  #uid=4
  %4 = load f32 s[%3]  #uid=5
  %5 = fadd f32 %4, %2  #uid=6
  store s[%3], %5  #uid=7
  %6 = load f32 s[%3]  #uid=8
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
ONLY = os.environ.get("IRLAT_ONLY")
for name, text in KERNELS.items():
    if ONLY and name != ONLY:
        continue
    ir = text.replace("NITER", str(N))
    doc = {"inputs": {"a": {"type": "f32", "data": [1.0] * 4}, "out": {"type": "f32", "data": [0.0] * 4}},
           "scalars": {}, "oracle": {}}
    suite = gevo.Suite.from_json(ir, [json.dumps(doc)])
    cfg = suite.exec_config().with_(budget=100_000_000)
    b = suite.batch().add_ir(ir)
    for seq in ((False,) if ONLY else (False, True)):
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
