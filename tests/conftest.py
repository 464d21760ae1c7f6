"""Shared fixtures. `gpu`-marked tests need a CUDA device (run under gpurun);
everything else runs on the CPU-only container."""
import gzip
import json
import os

import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_jsonl(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as f:
        return [json.loads(line) for line in f if line.strip()]


@pytest.fixture(scope="session")
def corpus_golden():
    return load_jsonl("corpus.jsonl.gz")


@pytest.fixture(scope="session")
def mutants_golden():
    return load_jsonl("mutants.jsonl.gz")


@pytest.fixture(scope="session")
def mutants_budget_golden():
    return load_jsonl("mutants_budget20k.jsonl.gz")


@pytest.fixture(scope="session")
def vmcases_golden():
    return load_jsonl("vmcases.jsonl.gz")


@pytest.fixture(scope="session")
def nsga_golden():
    return load_jsonl("nsga.jsonl.gz")


@pytest.fixture(scope="session")
def gevo():
    import paper_2004_08140_b200 as g
    g.lib()
    return g


def authored_fixture(name):
    """(suite header, records) of tests/golden/authored_<name>.jsonl.gz
    (oracle/gen_golden_authored.py, compiled reference)."""
    rows = load_jsonl("authored_%s.jsonl.gz" % name)
    return rows[0], rows[1:]
