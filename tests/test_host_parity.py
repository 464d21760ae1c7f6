"""Host-side parity (CPU only): the C++ host that feeds the device must
reproduce the reference's IR text, mutation draws, patch application,
validation verdicts and seeded test inputs bit for bit, and the C ABI must
export every entry point its header declares."""
import os
import re
import struct

import pytest

from _util import fixture_test_json, kernel_hash

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_corpus_kernels_print_identically(gevo, corpus_golden):
    kernels = [j for j in corpus_golden if j["kind"] == "kernel"]
    assert sorted(j["name"] for j in kernels) == gevo.benchmark_names()
    for j in kernels:
        assert gevo.benchmark_ir(j["name"]) == j["ir"]
        improved, n = gevo.apply_patch(j["ir"], j["reach_patch"])
        assert n == len(j["reach_patch"]) and improved == j["improved"]
        assert gevo.canonical(j["ir"]) == j["ir"]
        assert gevo.validate(j["ir"]) == []


def test_vmcase_kernels_round_trip(gevo, vmcases_golden):
    for case in vmcases_golden:
        assert gevo.canonical(case["ir"]) == case["ir"], case["label"]
        assert (gevo.validate(case["ir"]) == []) == case["valid"], case["label"]


@pytest.mark.parametrize("fixture", ["mutants_golden", "mutants_budget_golden"])
def test_mutation_draws_apply_and_validate(gevo, request, fixture):
    """random_mutation (RNG draw order included), apply_edit, validate."""
    records = request.getfixturevalue(fixture)
    names = gevo.benchmark_names()
    orig = {n: gevo.benchmark_ir(n) for n in names}
    n_edits = 0
    for m in records:
        k = names.index(m["name"])
        parent, n = gevo.apply_patch(orig[m["name"]], m["parent_patch"])
        assert n == len(m["parent_patch"])
        edit, probe = gevo.random_mutation(parent, 0x5EED, k, m["i"], 77)
        assert edit == m["edit"], (m["name"], m["i"])
        assert "%016x" % probe == m["probe"], (m["name"], m["i"])
        if edit is None:
            continue
        child, n = gevo.apply_patch(orig[m["name"]], m["parent_patch"] + [edit])
        assert (n == len(m["parent_patch"]) + 1) == m["applied"], (m["name"], m["i"])
        if not m["applied"]:
            continue
        assert kernel_hash(child) == m["kernel_hash"], (m["name"], m["i"])
        assert gevo.validate(child) == m["rules"], (m["name"], m["i"])
        n_edits += 1
    assert n_edits > 800


def test_seeded_inputs_bit_exact(gevo, corpus_golden):
    """generate_tests input draws (Rng::stream(seed, t, buffer, 91), float
    arithmetic without contraction) for every corpus suite."""
    seen = 0
    cache = {}
    for j in corpus_golden:
        if j["kind"] != "test":
            continue
        n = {"train3_seed1": 3, "heldout3_seed1": 3, "train16_seed1": 16}[j["suite"]]
        key = (j["name"], n, j["seed"])
        if key not in cache:
            cache[key] = gevo.benchmark_inputs(j["name"], n, j["seed"])
        mine = cache[key][j["index"]]
        ref = fixture_test_json(j["test"])
        assert sorted(mine["inputs"]) == sorted(ref["inputs"])
        for name, b in ref["inputs"].items():
            fmt = "<i" if b["type"] == "i32" else "<f"
            got = "".join("%08x" % struct.unpack("<I", struct.pack(fmt, x))[0]
                          for x in mine["inputs"][name]["data"])
            assert got == b["hex"], (j["name"], j["suite"], name)
        seen += 1
    assert seen == 6 * 22


def test_suite_seed_derivation(gevo, corpus_golden):
    seeds = {j["suite"]: j["seed"] for j in corpus_golden if j["kind"] == "test"}
    assert gevo.train_seed(1) == seeds["train3_seed1"] == seeds["train16_seed1"]
    assert gevo.heldout_seed(1) == seeds["heldout3_seed1"]


def test_abi_exports_every_declared_symbol(gevo):
    header = open(os.path.join(ROOT, "include", "gevo_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(gevo_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    lib = gevo.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(gevo.exported_symbols())
    assert gevo.lib().gevo_abi_version() == 1


def test_record_layouts_match_header(gevo):
    h = open(os.path.join(ROOT, "paper_2004_08140_b200", "csrc", "device", "bytecode.h")).read()
    assert "int64_t cost;" in h and "double error;" in h
    assert gevo.TEST_RECORD.itemsize == 32 and gevo.VARIANT_RECORD.itemsize == 48


def test_device_calls_fail_loudly_without_gpu(gevo):
    """No CPU fallback: on a GPU-less host every evaluation entry point raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gevo.DeviceError):
        gevo.Suite.from_benchmark("nw-sync", 3, 1)
    with pytest.raises(gevo.DeviceError):
        gevo.rank([1.0, 2.0], [0.0, 0.0])
    with pytest.raises(gevo.DeviceError):
        gevo.run_search("nw-sync", 1, 8, 1)
