"""Every icmp / fcmp predicate and the arithmetic ops on IEEE edge values
(NaN, signed zeros, infinities, subnormals, INT_MIN/INT_MAX wrap-around) on
the device interpreters, against the plain-C oracle and against Python's own
float32 / int32 semantics. The corpus kernels only ever compare with icmp.lt,
so these predicates are otherwise exercised only by random mutants."""
import math
import struct

import numpy as np
import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu

PREDS = ["eq", "ne", "lt", "le", "gt", "ge"]
F_PAIRS = [(float("nan"), 1.0), (1.0, float("nan")), (float("nan"), float("nan")), (0.0, -0.0),
           (-0.0, 0.0), (float("inf"), float("inf")), (-float("inf"), float("inf")),
           (1e-45, 0.0), (-1e-45, 1e-45), (1.5, 1.5), (2.0, -3.0), (-3.0, 2.0),
           (3.4e38, float("inf")), (-1.0, -1.0), (1e-38, 1.1e-38), (7.0, 6.999999)]
I_PAIRS = [(-2**31, 2**31 - 1), (2**31 - 1, -2**31), (0, 0), (-1, 0), (0, -1), (5, 5),
           (2**31 - 1, 2**31 - 1), (-2**31, -2**31), (123, -456), (-456, 123), (1, 2), (2, 1),
           (-7, -7), (65536, 65535), (-65536, 65536), (42, 43)]
T = len(F_PAIRS)
F_OPS = ["fadd", "fsub", "fmul"]
I_OPS = ["add", "sub", "mul"]
N_OUT = 2 * len(PREDS) + len(I_OPS)  # i32 words per thread in `out`


def _kernel():
    lines = ["kernel k(a: ptr<global> f32, b: ptr<global> i32, out: ptr<global> i32, "
             "fo: ptr<global> f32) threads=%d shared=0 {" % T, "entry:"]
    u = [0]

    def emit(s):
        lines.append("  %s  #uid=%d" % (s, u[0]))
        u[0] += 1

    emit("%0 = tid i32")
    emit("%1 = mul i32 %0, 2")
    emit("%2 = add i32 %1, 1")
    emit("%3 = load f32 a[%1]")
    emit("%4 = load f32 a[%2]")
    emit("%5 = load i32 b[%1]")
    emit("%6 = load i32 b[%2]")
    emit("%%7 = mul i32 %%0, %d" % N_OUT)
    v = 8
    k = 0
    # compares back to back (the straight-line run loop), then selects
    cmps = []
    for kind, (x, y) in (("fcmp", ("%3", "%4")), ("icmp", ("%5", "%6"))):
        ty = "f32" if kind == "fcmp" else "i32"
        for p in PREDS:
            emit("%%%d = %s.%s %s %s, %s" % (v, kind, p, ty, x, y))
            cmps.append(v)
            v += 1
    for c in cmps:
        emit("%%%d = select i32 %%%d, 1, 0" % (v, c))
        emit("%%%d = add i32 %%7, %d" % (v + 1, k))
        emit("store out[%%%d], %%%d" % (v + 1, v))
        v += 2
        k += 1
    for op in I_OPS:
        emit("%%%d = %s i32 %%5, %%6" % (v, op))
        emit("%%%d = add i32 %%7, %d" % (v + 1, k))
        emit("store out[%%%d], %%%d" % (v + 1, v))
        v += 2
        k += 1
    for j, op in enumerate(F_OPS):
        emit("%%%d = %s f32 %%3, %%4" % (v, op))
        emit("%%%d = mul i32 %%0, %d" % (v + 1, len(F_OPS)))
        emit("%%%d = add i32 %%%d, %d" % (v + 2, v + 1, j))
        emit("store fo[%%%d], %%%d" % (v + 2, v))
        v += 3
    emit("ret")
    lines.append("}")
    return "\n".join(lines)


def _f32_words(vals):
    return "".join("%08x" % struct.unpack("<I", struct.pack("<f", x))[0] for x in vals)


def _doc():
    a = [x for p in F_PAIRS for x in p]
    b = [x & 0xFFFFFFFF for p in I_PAIRS for x in p]
    return {"inputs": {"a": {"type": "f32", "hex": _f32_words(a)},
                       "b": {"type": "i32", "hex": "".join("%08x" % x for x in b)},
                       "out": {"type": "i32", "hex": "00000000" * (N_OUT * T)},
                       "fo": {"type": "f32", "hex": "00000000" * (len(F_OPS) * T)}},
            "scalars": {}, "oracle": {}}


def _python_expected():
    """Per-thread compare outcomes with C++ semantics (NaN: only != holds)."""
    out = []
    for (fx, fy), (ix, iy) in zip(F_PAIRS, I_PAIRS):
        fx, fy = float(np.float32(fx)), float(np.float32(fy))
        row = []
        for x, y in ((fx, fy), (ix, iy)):
            row += [int(x == y), int(x != y), int(x < y), int(x <= y), int(x > y), int(x >= y)]
        wrap = lambda z: ((z + 2**31) % 2**32) - 2**31  # noqa: E731
        row += [wrap(ix + iy) & 0xFFFFFFFF, wrap(ix - iy) & 0xFFFFFFFF, wrap(ix * iy) & 0xFFFFFFFF]
        out += row
    return out


def test_compare_and_arith_edges_match_oracle_and_python(gevo):
    ir = _kernel()
    doc = _doc()
    res = ob.execute(ob.Kernel(ir), ob.CTest(doc), ob.config(T, 0))
    assert res["status"] == "completed", res["reason"]
    got_out = [int(res["outputs"]["out"]["hex"][i:i + 8], 16)
               for i in range(0, len(res["outputs"]["out"]["hex"]), 8)]
    assert got_out == _python_expected()  # pins the oracle
    fo = res["outputs"]["fo"]["hex"]
    for t, (fx, fy) in enumerate(F_PAIRS):
        x, y = np.float32(fx), np.float32(fy)
        with np.errstate(all="ignore"):
            exp = [x + y, x - y, x * y]
        for j, e in enumerate(exp):
            w = int(fo[(t * 3 + j) * 8:(t * 3 + j + 1) * 8], 16)
            gw = struct.unpack("<I", struct.pack("<f", float(e)))[0]
            if math.isnan(float(e)):
                assert (w & 0x7F800000) == 0x7F800000 and (w & 0x7FFFFF), (t, j)
            else:
                assert w == gw, (t, j)
    doc["oracle"] = res["outputs"]
    # the oracle's own error against itself (NaN outputs count as failures)
    ref = ob.execute(ob.Kernel(ir), ob.CTest(doc), ob.config(T, 0))
    suite = gevo.Suite.from_json(ir, [doc])
    batch = suite.batch().add_ir(ir)
    # default budget: the straight-line run loop; a budget just above the
    # per-thread count: blocks that could cross it run in exact
    # per-instruction mode through the general dispatch
    for budget, seq in ((None, False), (None, True), (res["ir"] // T + 3, False),
                        (res["ir"] // T + 3, True)):
        cfg = suite.exec_config()
        if budget:
            cfg = cfg.with_(budget=budget)
        _, tr, _ = batch.eval(cfg, tests=True, sequential=seq)
        r = tr[0, 0]
        assert int(r["status"]) == 0, seq
        assert int(r["cost"]) == res["cost"] and int(r["ir"]) == res["ir"], seq
        assert hex_double(float(r["error"])) == hex_double(ref["error"]), seq
        outs = batch.outputs(cfg)
        assert outs[0][0]["out"]["hex"] == res["outputs"]["out"]["hex"], seq
