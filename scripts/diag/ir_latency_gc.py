"""GPU probe: per-IR latency of one long-running simulated thread in the
thread-parallel kernel, by kernel shape: threads=1, and threads=256 (one
instance per CTA, global cells) with only tid 0 long / warp 0 long. The loop
body mimics the conv-bn inner loop (short blocks: phi, compare, branch,
bounds checks). Spin accelerator off (GEVO_SPIN_THRESHOLD=0 set here)."""
import json
import os
import sys

os.environ["GEVO_SPIN_THRESHOLD"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
BODY = """kernel k(a: ptr<global> f32, out: ptr<global> f32) threads=THREADS shared=0 {
entry:
  %0 = tid i32  #uid=0
  %1 = icmp.lt i32 %0, LONG  #uid=1
  %2 = select i32 %1, NITER, 1  #uid=2
  br loop  #uid=3
loop:
  %3 = phi i32 [0, entry], [%20, next]  #uid=4
  %4 = phi f32 [0.0, entry], [%21, next]  #uid=5
  %5 = icmp.lt i32 %3, %2  #uid=6
  br %5, body, done  #uid=7
body:
  %6 = add i32 %3, %0  #uid=8
  %7 = sub i32 %6, 1  #uid=9
  %8 = icmp.ge i32 %7, -1000000  #uid=10
  br %8, chk, next  #uid=11
chk:
  %9 = icmp.lt i32 %7, 100000000  #uid=12
  br %9, tap, next  #uid=13
tap:
  %10 = mul i32 %3, 0  #uid=14
  %11 = load f32 a[%10]  #uid=15
  %12 = fmul f32 %11, 0.5  #uid=16
  %13 = fadd f32 %4, %12  #uid=17
  br next  #uid=18
next:
  %21 = phi f32 [%4, body], [%4, chk], [%13, tap]  #uid=19
  %20 = add i32 %3, 1  #uid=20
  br loop  #uid=21
done:
  store out[%0], %4  #uid=22
  ret  #uid=23
}"""

res = {}
ONLY = os.environ.get("IRGC_ONLY")  # one shape (e.g. for an ncu capture)
for name, threads, long_ in (("t1", 1, 1), ("t256_tid0", 256, 1), ("t256_warp0", 256, 32),
                             ("t256_all", 256, 256)):
    if ONLY and name != ONLY:
        continue
    ir = BODY.replace("THREADS", str(threads)).replace("LONG", str(long_)).replace("NITER", str(N))
    doc = {"inputs": {"a": {"type": "f32", "data": [1.0] * 4},
                      "out": {"type": "f32", "data": [0.0] * threads}},
           "scalars": {}, "oracle": {}}
    suite = gevo.Suite.from_json(ir, [json.dumps(doc)])
    cfg = suite.exec_config().with_(budget=100_000_000)
    b = suite.batch().add_ir(ir)
    ms = []
    for _ in range(4):
        _, t, st = b.eval(cfg, tests=True)
        ms.append(st.device_ms)
    ir_total = int(t[0, 0]["ir"])
    per_thread = (ir_total - (threads - long_) * 12) / long_
    best = min(ms[1:])
    res[name] = {"ir_long_thread": per_thread, "ms": best, "ns_per_ir": best * 1e6 / per_thread,
                 "cycles_per_ir_1965": best * 1.965e6 / per_thread}
    print(name, json.dumps(res[name]), flush=True)
