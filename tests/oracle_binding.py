"""ctypes binding of the plain-C oracle (oracle/liboracle.so). TEST
INFRASTRUCTURE: only tests/, smoke() and bench.py's cpu_baseline use it, and
only as the checker."""
import ctypes
import os
import struct

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "liboracle.so")


class Buf(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("elem", ctypes.c_int32), ("n", ctypes.c_int32),
                ("words", ctypes.POINTER(ctypes.c_uint32))]


class Scal(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("kind", ctypes.c_int32), ("bits", ctypes.c_uint32)]


class Test(ctypes.Structure):
    _fields_ = [("n_inputs", ctypes.c_int32), ("inputs", ctypes.POINTER(Buf)),
                ("n_scalars", ctypes.c_int32), ("scalars", ctypes.POINTER(Scal)),
                ("n_oracle", ctypes.c_int32), ("oracle", ctypes.POINTER(Buf))]


class Config(ctypes.Structure):
    _fields_ = [("threads", ctypes.c_int32), ("shared_words", ctypes.c_int32),
                ("budget", ctypes.c_int64), ("cost", ctypes.c_int64 * 14)]


class Result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("cost", ctypes.c_int64), ("ir", ctypes.c_int64),
                ("error", ctypes.c_double), ("reason", ctypes.c_char * 160),
                ("n_outputs", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError("oracle/liboracle.so missing: make -C oracle")
        L = ctypes.CDLL(LIB)
        L.eo_parse.restype = ctypes.c_void_p
        L.eo_parse.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]
        L.eo_free.argtypes = [ctypes.c_void_p]
        L.eo_param_count.argtypes = [ctypes.c_void_p]
        L.eo_execute.argtypes = [ctypes.c_void_p, ctypes.POINTER(Test), ctypes.POINTER(Config),
                                 ctypes.POINTER(Result), ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p]
        L.eo_evaluate_fitness.argtypes = [ctypes.c_void_p, ctypes.POINTER(Test), ctypes.c_int32,
                                          ctypes.POINTER(Config), ctypes.c_double,
                                          ctypes.POINTER(ctypes.c_int32), ctypes.c_char_p,
                                          ctypes.c_size_t, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int32)]
        L.eo_rank.restype = ctypes.c_int32
        L.eo_rank.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int32] + [ctypes.c_void_p] * 4
        L.eo_select_best.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                     ctypes.c_int32, ctypes.c_void_p]
        _lib = L
    return _lib


class Kernel:
    def __init__(self, text: str):
        err = ctypes.create_string_buffer(256)
        self._h = lib().eo_parse(text.encode(), err, 256)
        if not self._h:
            raise ValueError(err.value.decode())

    def __del__(self):
        if getattr(self, "_h", None):
            lib().eo_free(self._h)


def _words(hexstr):
    return [int(hexstr[i:i + 8], 16) for i in range(0, len(hexstr), 8)]


class CTest:
    """Owns the C structs for one TestCase JSON document (hex buffers)."""

    def __init__(self, doc):
        self._keep = []
        self.words = 0

        def bufs(section):
            items = sorted(doc.get(section, {}).items())
            arr = (Buf * max(len(items), 1))()
            for i, (name, b) in enumerate(items):
                if "hex" in b:
                    w = _words(b["hex"])
                else:
                    fmt = "<i" if b["type"] == "i32" else "<f"
                    w = [struct.unpack("<I", struct.pack(fmt, x))[0] for x in b["data"]]
                self.words += len(w)
                data = (ctypes.c_uint32 * max(len(w), 1))(*w)
                nm = name.encode()
                self._keep += [data, nm]
                arr[i] = Buf(nm, 0 if b["type"] == "i32" else 1, len(w), data)
            return arr, len(items)

        ins, ni = bufs("inputs")
        orc, no = bufs("oracle")
        sc = sorted(doc.get("scalars", {}).items())
        sarr = (Scal * max(len(sc), 1))()
        for i, (name, s) in enumerate(sc):
            kind = {"i32": 0, "f32": 1, "bool": 2}[s["type"]]
            if kind == 0:
                bits = s["value"] & 0xFFFFFFFF
            elif kind == 1:
                bits = struct.unpack("<I", struct.pack("<f", s["value"]))[0]
            else:
                bits = 1 if s["value"] else 0
            nm = name.encode()
            self._keep.append(nm)
            sarr[i] = Scal(nm, kind, bits)
        self._keep += [ins, orc, sarr]
        self.c = Test(ni, ins, len(sc), sarr, no, orc)


def config(threads, shared_words, budget=1_000_000, costs=(1, 1, 1, 1, 1, 1, 1, 1, 4, 4, 20, 20, 8, 1)):
    c = Config(threads, shared_words, budget)
    for i, v in enumerate(costs):
        c.cost[i] = v
    return c


STATUS = {0: "completed", 1: "trap", 2: "budget"}


def execute(kernel: Kernel, test: CTest, cfg: Config):
    r = Result()
    cap = max(1 << 16, test.words + 64)
    words = (ctypes.c_uint32 * cap)()
    offs = (ctypes.c_int32 * 64)()
    sizes = (ctypes.c_int32 * 64)()
    elems = (ctypes.c_int32 * 64)()
    names = (ctypes.c_char_p * 64)()
    lib().eo_execute(kernel._h, ctypes.byref(test.c), ctypes.byref(cfg), ctypes.byref(r),
                     words, cap, offs, sizes, elems, names)
    outs = {}
    if r.status == 0:
        for j in range(r.n_outputs):
            w = words[offs[j]:offs[j] + sizes[j]]
            outs[names[j].decode()] = {"type": "i32" if elems[j] == 0 else "f32",
                                       "hex": "".join("%08x" % x for x in w)}
    return {"status": STATUS[r.status], "reason": r.reason.decode(), "cost": r.cost,
            "ir": r.ir, "error": r.error, "outputs": outs}


def evaluate_fitness(kernel: Kernel, tests, cfg: Config, tolerance: float):
    arr = (Test * max(len(tests), 1))(*[t.c for t in tests])
    ft = ctypes.c_int32()
    reason = ctypes.create_string_buffer(200)
    cost, err = ctypes.c_double(), ctypes.c_double()
    ir, execs = ctypes.c_int64(), ctypes.c_int32()
    acc = lib().eo_evaluate_fitness(kernel._h, arr, len(tests), ctypes.byref(cfg), tolerance,
                                    ctypes.byref(ft), reason, 200, ctypes.byref(cost),
                                    ctypes.byref(err), ctypes.byref(ir), ctypes.byref(execs))
    return {"accepted": bool(acc), "failing_test": ft.value, "reason": reason.value.decode(),
            "cost": cost.value, "error": err.value, "ir_ref": ir.value,
            "execs_ref": execs.value}


def rank(cost, error):
    import numpy as np
    c = np.ascontiguousarray(cost, np.float64)
    e = np.ascontiguousarray(error, np.float64)
    n = len(c)
    front = np.zeros(n, np.int32)
    crowd = np.zeros(n, np.float64)
    members = np.zeros(n + 1, np.int32)
    offsets = np.zeros(n + 2, np.int32)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    nf = lib().eo_rank(vp(c), vp(e), n, vp(front), vp(crowd), vp(members), vp(offsets))
    return front, crowd, [members[offsets[f]:offsets[f + 1]].tolist() for f in range(nf)]


def select_best(cost, error, keep):
    import numpy as np
    c = np.ascontiguousarray(cost, np.float64)
    e = np.ascontiguousarray(error, np.float64)
    out = np.zeros(max(keep, 1), np.int32)
    lib().eo_select_best(c.ctypes.data_as(ctypes.c_void_p), e.ctypes.data_as(ctypes.c_void_p),
                         len(c), keep, out.ctypes.data_as(ctypes.c_void_p))
    return out[:keep].tolist()
