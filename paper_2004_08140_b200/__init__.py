"""B200-native GEVO fitness-evaluation engine (arXiv 2004.08140 hot path).

Python view of the C ABI in ``include/gevo_b200.h`` (ctypes over the in-tree
``libgevo_b200.so``). The library is the product: a C++ host that keeps the
reference ``evoir`` API (IR, mutation operators, crossover, NSGA-II, the
error-tolerance gate) and hand-written sm_100a kernels for the batched
interpreter, the fitness reduction and the non-dominated sort. This module
only marshals arguments; there is no Python or CPU evaluation path, and every
device call raises :class:`DeviceError` when no GPU is present.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Iterable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GEVO_LIB") or os.path.join(_HERE, "libgevo_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "gevo_b200.h")

# ---- record layouts (bytecode.h) ---------------------------------------------
TEST_RECORD = np.dtype([("cost", "<i8"), ("ir", "<i8"), ("error", "<f8"), ("aux", "<i4"),
                        ("status", "u1"), ("code", "u1"), ("pad", "u1", 2)])
VARIANT_RECORD = np.dtype([("cost_mean", "<f8"), ("error_max", "<f8"), ("fail_error", "<f8"),
                           ("ir_ref", "<i8"), ("failing_test", "<i4"), ("execs_ref", "<i4"),
                           ("aux", "<i4"), ("accepted", "u1"), ("code", "u1"), ("pad", "u1", 2)])
assert TEST_RECORD.itemsize == 32 and VARIANT_RECORD.itemsize == 48

STATUS_COMPLETED, STATUS_TRAP, STATUS_BUDGET, STATUS_SKIPPED = 0, 1, 2, 3
FAIL_TOLERANCE = 0xFF
EVAL_EARLY_EXIT, EVAL_TESTS, EVAL_SEQUENTIAL, EVAL_UPLOAD = 1, 2, 4, 8
COST_FIELDS = ("arith", "cmp", "select_op", "phi", "constant", "br", "intrinsic", "getindex",
               "load_shared", "store_shared", "load_global", "store_global", "sync", "ret")
DEFAULT_COSTS = (1, 1, 1, 1, 1, 1, 1, 1, 4, 4, 20, 20, 8, 1)
UNIT_COSTS = (1,) * 14


class GevoError(RuntimeError):
    pass


class DeviceError(GevoError):
    """No usable CUDA device (the product has no CPU path)."""


class InitFailure(GevoError):
    pass


class ExecConfig(ctypes.Structure):
    _fields_ = [("threads", ctypes.c_int32), ("shared_words", ctypes.c_int32),
                ("instruction_budget", ctypes.c_int64), ("cost_table", ctypes.c_int64 * 14)]

    @classmethod
    def make(cls, threads: int, shared_words: int, budget: int = 1_000_000,
             costs: Sequence[int] = DEFAULT_COSTS) -> "ExecConfig":
        c = cls()
        c.threads, c.shared_words, c.instruction_budget = threads, shared_words, budget
        for i, v in enumerate(costs):
            c.cost_table[i] = v
        return c

    def with_(self, budget: Optional[int] = None, costs: Optional[Sequence[int]] = None):
        return ExecConfig.make(self.threads, self.shared_words,
                               self.instruction_budget if budget is None else budget,
                               list(self.cost_table) if costs is None else costs)


class EvalStats(ctypes.Structure):
    _fields_ = [("device_ms", ctypes.c_float), ("h2d_bytes", ctypes.c_uint64),
                ("d2h_bytes", ctypes.c_uint64), ("launches", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class RunStats(ctypes.Structure):
    _fields_ = [("candidates", ctypes.c_int64), ("executions", ctypes.c_int64),
                ("dynamic_ir", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("batches", ctypes.c_int64), ("device_ms", ctypes.c_double),
                ("host_gen_ms", ctypes.c_double), ("seconds", ctypes.c_double)]


_c_char_pp = ctypes.POINTER(ctypes.c_char_p)
_vp = ctypes.c_void_p
_i32, _i64, _u64, _u32, _f64 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                ctypes.c_uint32, ctypes.c_double)
_str_out = ctypes.POINTER(ctypes.c_void_p)

# (name, restype, argtypes)
_SIGNATURES = [
    ("gevo_abi_version", ctypes.c_int, []),
    ("gevo_device_count", ctypes.c_int, []),
    ("gevo_last_error", ctypes.c_char_p, []),
    ("gevo_set_stream", ctypes.c_int, [_vp]),
    ("gevo_spin_counters", ctypes.c_int, [_vp, ctypes.c_int]),
    ("gevo_tp_counters", ctypes.c_int, [_vp, ctypes.c_int]),
    ("gevo_work_counters", ctypes.c_int, [_vp, ctypes.c_int]),
    ("gevo_nccl_unique_id", ctypes.c_int, [_vp]),
    ("gevo_set_nccl", ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp]),
    ("gevo_set_collective", ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp]),
    ("gevo_free", None, [_vp]),
    ("gevo_suite_from_benchmark", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _u64, ctypes.c_int,
                                                 ctypes.POINTER(_vp)]),
    ("gevo_suite_from_json", ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p),
                                            ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    ("gevo_suite_free", None, [_vp]),
    ("gevo_suite_n_tests", ctypes.c_int, [_vp]),
    ("gevo_suite_exec_config", ctypes.c_int, [_vp, ctypes.POINTER(ExecConfig)]),
    ("gevo_suite_kernel_ir", ctypes.c_int, [_vp, _str_out]),
    ("gevo_batch_create", ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    ("gevo_batch_add_ir", ctypes.c_int, [_vp, ctypes.c_char_p]),
    ("gevo_batch_add_patch", ctypes.c_int, [_vp, ctypes.c_char_p]),
    ("gevo_batch_size", ctypes.c_int, [_vp]),
    ("gevo_batch_blob", ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_size_t)]),
    ("gevo_batch_free", None, [_vp]),
    ("gevo_eval", ctypes.c_int, [_vp, ctypes.POINTER(ExecConfig), _f64, _u32, _vp, _vp,
                                 ctypes.POINTER(EvalStats)]),
    ("gevo_batch_make_resident", ctypes.c_int, [_vp]),
    ("gevo_eval_resident_async", ctypes.c_int, [_vp, ctypes.POINTER(ExecConfig), _f64, _u32]),
    ("gevo_eval_resident_wait", ctypes.c_int, [_vp, _vp, ctypes.POINTER(EvalStats)]),
    ("gevo_eval_resident", ctypes.c_int, [_vp, ctypes.POINTER(ExecConfig), _f64, _u32, _vp,
                                          ctypes.POINTER(EvalStats)]),
    ("gevo_reason", ctypes.c_int, [_vp, ctypes.c_int, _u32, _i32, _f64, _str_out]),
    ("gevo_eval_outputs_json", ctypes.c_int, [_vp, ctypes.POINTER(ExecConfig), _str_out]),
    ("gevo_execute", ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ExecConfig),
                                    _str_out]),
    ("gevo_evaluate_fitness", ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p),
                                             ctypes.c_int, ctypes.POINTER(ExecConfig), _f64,
                                             _str_out]),
    ("gevo_nsga_select", ctypes.c_int, [_vp, _vp, _i32, ctypes.c_int, _i32, _vp, _u64, _i32,
                                        _vp]),
    ("gevo_rank", ctypes.c_int, [_vp, _vp, _i32, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    ("gevo_debug_cta_clock", ctypes.c_int, [_vp, ctypes.c_size_t, _vp]),
    ("gevo_select_best", ctypes.c_int, [_vp, _vp, _i32, ctypes.c_int, _i32, _vp, _vp]),
    ("gevo_crowding", ctypes.c_int, [_vp, _vp, _i32, ctypes.c_int, _vp]),
    ("gevo_kernel_canonical", ctypes.c_int, [ctypes.c_char_p, _str_out]),
    ("gevo_kernel_validate", ctypes.c_int, [ctypes.c_char_p, _str_out]),
    ("gevo_kernel_is_valid", ctypes.c_int, [ctypes.c_char_p, _vp]),
    ("gevo_apply_patch", ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _str_out,
                                        ctypes.POINTER(_i32)]),
    ("gevo_random_mutation", ctypes.c_int, [ctypes.c_char_p, _u64, _u64, _u64, _u64, _str_out,
                                            ctypes.POINTER(_u64)]),
    ("gevo_benchmark_inputs", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _u64, _str_out]),
    ("gevo_benchmark_names", ctypes.c_int, [_str_out]),
    ("gevo_benchmark_ir", ctypes.c_int, [ctypes.c_char_p, _str_out]),
    ("gevo_sample_candidates_ir", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _u64, ctypes.c_int,
                                                 _str_out]),
    ("gevo_suite_from_spec", ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, _u64,
                                            ctypes.c_int, ctypes.POINTER(_vp)]),
    ("gevo_spec_inputs", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _u64, _str_out]),
    ("gevo_sample_candidates", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _u64, ctypes.c_int,
                                              _str_out]),
    ("gevo_train_seed", _u64, [_u64]),
    ("gevo_heldout_seed", _u64, [_u64]),
    ("gevo_run_search", ctypes.c_int, [ctypes.c_char_p, _u64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_char_p, _f64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, _str_out, _str_out,
                                       ctypes.POINTER(RunStats)]),
]

_lib = None


def exported_symbols() -> list:
    return [name for name, _, _ in _SIGNATURES]


def lib():
    """Loads the in-tree library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2004_08140_b200)")
        handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, res, args in _SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = (lib().gevo_last_error() or b"").decode()
    if rc == -2:
        raise DeviceError(msg)
    if rc == -4:
        raise InitFailure(msg)
    raise GevoError(f"gevo call failed ({rc}): {msg}")


def _take(p: ctypes.c_void_p) -> str:
    s = ctypes.string_at(p.value).decode()
    lib().gevo_free(p)
    return s


def _b(s: str) -> bytes:
    return s.encode()


# ---- host-side API -------------------------------------------------------------
def canonical(ir: str) -> str:
    out = ctypes.c_void_p()
    _check(lib().gevo_kernel_canonical(_b(ir), ctypes.byref(out)))
    return _take(out)


def validate(ir: str) -> list:
    out = ctypes.c_void_p()
    _check(lib().gevo_kernel_validate(_b(ir), ctypes.byref(out)))
    return json.loads(_take(out))


def is_valid(ir: str) -> bool:
    """is_valid (ir.hpp:258): validate(k).empty() by the verdict-only path."""
    v = ctypes.c_int32()
    _check(lib().gevo_kernel_is_valid(_b(ir), ctypes.byref(v)))
    return bool(v.value)


def apply_patch(ir: str, patch) -> tuple:
    text = patch if isinstance(patch, str) else json.dumps(patch)
    out, n = ctypes.c_void_p(), ctypes.c_int32()
    _check(lib().gevo_apply_patch(_b(ir), _b(text), ctypes.byref(out), ctypes.byref(n)))
    return _take(out), n.value


def random_mutation(ir: str, master: int, a: int, b: int, c: int) -> tuple:
    out, probe = ctypes.c_void_p(), ctypes.c_uint64()
    _check(lib().gevo_random_mutation(_b(ir), master, a, b, c, ctypes.byref(out),
                                      ctypes.byref(probe)))
    return json.loads(_take(out)), probe.value


def benchmark_names() -> list:
    out = ctypes.c_void_p()
    _check(lib().gevo_benchmark_names(ctypes.byref(out)))
    return json.loads(_take(out))


def benchmark_ir(name: str) -> str:
    out = ctypes.c_void_p()
    _check(lib().gevo_benchmark_ir(_b(name), ctypes.byref(out)))
    return _take(out)


def benchmark_inputs(name: str, count: int, seed: int) -> list:
    out = ctypes.c_void_p()
    _check(lib().gevo_benchmark_inputs(_b(name), count, seed, ctypes.byref(out)))
    return json.loads(_take(out))


def sample_candidates(bench: str, n: int, seed: int, max_depth: int = 4) -> list:
    """n validated (not evaluated) mutants of `bench` as patch JSON strings."""
    out = ctypes.c_void_p()
    _check(lib().gevo_sample_candidates(_b(bench), n, seed, max_depth, ctypes.byref(out)))
    return [line for line in _take(out).split("\n") if line]


def sample_candidates_ir(kernel_ir: str, n: int, seed: int, max_depth: int = 4) -> list:
    """n validated (not evaluated) mutants of an arbitrary kernel as patch JSON strings."""
    out = ctypes.c_void_p()
    _check(lib().gevo_sample_candidates_ir(_b(kernel_ir), n, seed, max_depth, ctypes.byref(out)))
    return [line for line in _take(out).split("\n") if line]


def spec_inputs(gen_json: str, count: int, seed: int) -> list:
    """Seeded inputs of a generator spec (TestCase JSON documents, no oracles)."""
    out = ctypes.c_void_p()
    _check(lib().gevo_spec_inputs(_b(gen_json), count, seed, ctypes.byref(out)))
    return json.loads(_take(out))


KERNEL_DIR = os.path.join(_HERE, "data", "kernels")


def authored_kernel(name: str) -> tuple:
    """(IR text, generator spec JSON) of an authored workload kernel
    (data/kernels/<name>.ir, <name>.gen.json): svm-rbf (config 3), conv-bn (config 4)."""
    with open(os.path.join(KERNEL_DIR, name + ".ir")) as f:
        ir = f.read()
    with open(os.path.join(KERNEL_DIR, name + ".gen.json")) as f:
        gen = f.read()
    return ir, gen


def set_stream(stream_ptr: int) -> None:
    """Run the library's launches on a caller's CUDA stream (0 = its own)."""
    _check(lib().gevo_set_stream(ctypes.c_void_p(stream_ptr or None)))


def tp_counters(reset: bool = False) -> tuple:
    """(instances re-run in thread-id order, instances run) by the
    thread-parallel interpreter."""
    out = (ctypes.c_uint64 * 2)()
    _check(lib().gevo_tp_counters(ctypes.cast(out, ctypes.c_void_p), 1 if reset else 0))
    return out[0], out[1]


def work_counters(reset: bool = False) -> int:
    """IR instructions the device interpreted since the last reset (jumps
    excluded, discarded work included)."""
    out = (ctypes.c_uint64 * 2)()
    _check(lib().gevo_work_counters(out, 1 if reset else 0))
    return int(out[0])


def spin_counters(reset: bool = False) -> tuple:
    """(loops jumped, instructions skipped) by the spin accelerator."""
    out = (ctypes.c_uint64 * 2)()
    _check(lib().gevo_spin_counters(ctypes.cast(out, ctypes.c_void_p), 1 if reset else 0))
    return out[0], out[1]


def train_seed(master: int) -> int:
    return lib().gevo_train_seed(master)


def heldout_seed(master: int) -> int:
    return lib().gevo_heldout_seed(master)


# ---- device API ------------------------------------------------------------------
class Suite:
    """Test suite resident on one GPU."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_benchmark(cls, bench: str, n_tests: int, seed: int, device: int = -1) -> "Suite":
        h = ctypes.c_void_p()
        _check(lib().gevo_suite_from_benchmark(_b(bench), n_tests, seed, device, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_spec(cls, kernel_ir: str, gen_json: str, n_tests: int, seed: int,
                  device: int = -1) -> "Suite":
        """generate_tests_for(kernel, spec, n_tests, seed): seeded inputs, oracle
        = the kernel's own outputs (computed on the device)."""
        h = ctypes.c_void_p()
        _check(lib().gevo_suite_from_spec(_b(kernel_ir), _b(gen_json), n_tests, seed, device,
                                          ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_json(cls, kernel_ir: str, tests: Iterable, device: int = -1) -> "Suite":
        docs = [t if isinstance(t, str) else json.dumps(t) for t in tests]
        arr = (ctypes.c_char_p * max(len(docs), 1))(*[_b(d) for d in docs])
        h = ctypes.c_void_p()
        _check(lib().gevo_suite_from_json(_b(kernel_ir), arr, len(docs), device, ctypes.byref(h)))
        return cls(h)

    @property
    def n_tests(self) -> int:
        return lib().gevo_suite_n_tests(self._h)

    def exec_config(self) -> ExecConfig:
        c = ExecConfig()
        _check(lib().gevo_suite_exec_config(self._h, ctypes.byref(c)))
        return c

    def kernel_ir(self) -> str:
        out = ctypes.c_void_p()
        _check(lib().gevo_suite_kernel_ir(self._h, ctypes.byref(out)))
        return _take(out)

    def batch(self) -> "Batch":
        h = ctypes.c_void_p()
        _check(lib().gevo_batch_create(self._h, ctypes.byref(h)))
        return Batch(self, h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gevo_suite_free(self._h)
            self._h = None


class Batch:
    """A population of variants encoded to device bytecode."""

    def __init__(self, suite: Suite, handle):
        self.suite = suite
        self._h = handle

    def add_ir(self, ir: str) -> "Batch":
        _check(lib().gevo_batch_add_ir(self._h, _b(ir)))
        return self

    def add_patch(self, patch) -> "Batch":
        text = patch if isinstance(patch, str) else json.dumps(patch)
        _check(lib().gevo_batch_add_patch(self._h, _b(text)))
        return self

    def __len__(self) -> int:
        return lib().gevo_batch_size(self._h)

    def blob(self) -> bytes:
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().gevo_batch_blob(self._h, ctypes.byref(p), ctypes.byref(n)))
        return ctypes.string_at(p.value, n.value)

    def eval(self, cfg: ExecConfig, tolerance: float = 0.0, early_exit: bool = False,
             tests: bool = False, sequential: bool = False):
        """Returns (variant_records, test_records | None, EvalStats).
        sequential=True forces the sequential-lane interpreter."""
        n, t = len(self), self.suite.n_tests
        vrec = np.zeros(n, VARIANT_RECORD)
        trec = np.zeros(n * t, TEST_RECORD) if tests else None
        flags = ((EVAL_EARLY_EXIT if early_exit else 0) | (EVAL_TESTS if tests else 0) |
                 (EVAL_SEQUENTIAL if sequential else 0))
        st = EvalStats()
        _check(lib().gevo_eval(self._h, ctypes.byref(cfg), tolerance, flags,
                               vrec.ctypes.data_as(ctypes.c_void_p),
                               trec.ctypes.data_as(ctypes.c_void_p) if tests else None,
                               ctypes.byref(st)))
        return vrec, (trec.reshape(n, t) if tests else None), st

    def make_resident(self):
        _check(lib().gevo_batch_make_resident(self._h))

    def eval_resident_async(self, cfg: ExecConfig, tolerance: float = 0.0,
                            early_exit: bool = True, upload: bool = False) -> None:
        """Launch on the batch's own stream and return (overlaps with other
        batches in flight); pair with wait(). upload=True copies the host
        bytecode to the device as part of the evaluation."""
        flags = (EVAL_EARLY_EXIT if early_exit else 0) | (EVAL_UPLOAD if upload else 0)
        _check(lib().gevo_eval_resident_async(self._h, ctypes.byref(cfg), tolerance, flags))

    def wait(self, records: bool = True):
        """(variant records | None, EvalStats) of the evaluation in flight."""
        vrec = np.zeros(len(self), VARIANT_RECORD) if records else None
        st = EvalStats()
        _check(lib().gevo_eval_resident_wait(
            self._h, vrec.ctypes.data_as(ctypes.c_void_p) if records else None, ctypes.byref(st)))
        return vrec, st

    def eval_resident(self, cfg: ExecConfig, tolerance: float = 0.0, early_exit: bool = True,
                      records: bool = False):
        vrec = np.zeros(len(self), VARIANT_RECORD) if records else None
        st = EvalStats()
        _check(lib().gevo_eval_resident(
            self._h, ctypes.byref(cfg), tolerance, EVAL_EARLY_EXIT if early_exit else 0,
            vrec.ctypes.data_as(ctypes.c_void_p) if records else None, ctypes.byref(st)))
        return vrec, st

    def outputs(self, cfg: ExecConfig) -> list:
        """Final global buffers per [variant][test] (None when not completed)."""
        out = ctypes.c_void_p()
        _check(lib().gevo_eval_outputs_json(self._h, ctypes.byref(cfg), ctypes.byref(out)))
        return json.loads(_take(out))

    def reason(self, variant: int, code: int, aux: int, fail_error: float = 0.0) -> str:
        out = ctypes.c_void_p()
        _check(lib().gevo_reason(self._h, variant, code, aux, fail_error, ctypes.byref(out)))
        return _take(out)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gevo_batch_free(self._h)
            self._h = None


def rank(cost, error, device: int = -1):
    """GPU rank_population: (front[n], crowding[n], fronts as lists)."""
    c = np.ascontiguousarray(cost, dtype=np.float64)
    e = np.ascontiguousarray(error, dtype=np.float64)
    n = len(c)
    front = np.zeros(n, np.int32)
    crowd = np.zeros(n, np.float64)
    members = np.zeros(max(n, 1), np.int32)
    offsets = np.zeros(n + 1, np.int32)
    nf = ctypes.c_int32()
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib().gevo_rank(vp(c), vp(e), n, device, vp(front), vp(crowd), vp(members),
                           vp(offsets), ctypes.byref(nf)))
    fronts = [members[offsets[f]:offsets[f + 1]].tolist() for f in range(nf.value)]
    return front, crowd, fronts


def execute(kernel_ir: str, test, cfg: ExecConfig) -> dict:
    """evoir::execute as a batch of one (status, reason, cost, outputs)."""
    text = test if isinstance(test, str) else json.dumps(test)
    out = ctypes.c_void_p()
    _check(lib().gevo_execute(_b(kernel_ir), _b(text), ctypes.byref(cfg), ctypes.byref(out)))
    return json.loads(_take(out))


def evaluate_fitness(kernel_ir: str, tests: Sequence, cfg: ExecConfig, tolerance: float) -> dict:
    docs = [t if isinstance(t, str) else json.dumps(t) for t in tests]
    arr = (ctypes.c_char_p * max(len(docs), 1))(*[_b(d) for d in docs])
    out = ctypes.c_void_p()
    _check(lib().gevo_evaluate_fitness(_b(kernel_ir), arr, len(docs), ctypes.byref(cfg),
                                       tolerance, ctypes.byref(out)))
    return json.loads(_take(out))


def nsga_select(cost, error, keep: int, tournament_seed: int, k: int, device: int = -1):
    c = np.ascontiguousarray(cost, dtype=np.float64)
    e = np.ascontiguousarray(error, dtype=np.float64)
    best = np.zeros(max(keep, 1), np.int32)
    tour = np.zeros(max(k, 1), np.int32)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib().gevo_nsga_select(vp(c), vp(e), len(c), device, keep, vp(best), tournament_seed,
                                  k, vp(tour)))
    return best[:keep].tolist(), tour[:k].tolist()


def debug_cta_clock(n_variants: int, n_tests: int):
    """Per-CTA timing of the last evaluation (GEVO_CTA_CLOCK=1):
    [variant, test, 4] uint64 {start ns, end ns, SM, device IR}."""
    out = np.zeros((n_variants, n_tests, 4), np.uint64)
    got = ctypes.c_size_t()
    _check(lib().gevo_debug_cta_clock(out.ctypes.data_as(ctypes.c_void_p), out.size,
                                      ctypes.byref(got)))
    return out


def select_best(cost, error, keep: int, device: int = -1):
    """rank_population + select_best(rank, keep) in one device pass:
    (keep order as int32 array, device ms of the ranking kernels)."""
    c = np.ascontiguousarray(cost, dtype=np.float64)
    e = np.ascontiguousarray(error, dtype=np.float64)
    best = np.zeros(max(keep, 1), np.int32)
    ms = ctypes.c_float()
    _check(lib().gevo_select_best(c.ctypes.data_as(ctypes.c_void_p), e.ctypes.data_as(ctypes.c_void_p),
                                  len(c), device, keep, best.ctypes.data_as(ctypes.c_void_p),
                                  ctypes.byref(ms)))
    return best[:keep], ms.value


def crowding(cost, error, device: int = -1):
    c = np.ascontiguousarray(cost, dtype=np.float64)
    e = np.ascontiguousarray(error, dtype=np.float64)
    out = np.zeros(len(c), np.float64)
    _check(lib().gevo_crowding(c.ctypes.data_as(ctypes.c_void_p),
                               e.ctypes.data_as(ctypes.c_void_p), len(c), device,
                               out.ctypes.data_as(ctypes.c_void_p)))
    return out


def run_search(bench: str, seed: int, pop: int, generations: int, mode: str = "default",
               tolerance: float = -1.0, train_tests: int = 3, heldout_tests: int = 3,
               jobs: int = 1):
    """``evoir run`` on a registry benchmark: (log_csv, report_json, RunStats)."""
    log, rep = ctypes.c_void_p(), ctypes.c_void_p()
    st = RunStats()
    _check(lib().gevo_run_search(_b(bench), seed, pop, generations, _b(mode), tolerance,
                                 train_tests, heldout_tests, jobs, ctypes.byref(log),
                                 ctypes.byref(rep), ctypes.byref(st)))
    return _take(log), _take(rep), st
