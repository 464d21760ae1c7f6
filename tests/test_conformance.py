"""The reference's own unit suites (proj/tests/test_*.cpp) compiled against
this framework's evoir headers and libgevo_b200.so (oracle/Makefile
"conformance", built where /root/reference exists; the binaries travel to the
GPU box under oracle/_ref/). Host-only suites run here; the suites that
execute kernels launch the sm_100a interpreter for every evoir::execute call
and run on the GPU."""
import os
import subprocess

import pytest

DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "conformance")
HOST_ONLY = ["ir", "genome"]
DEVICE = ["vm", "operators", "nsga", "corpus", "engine"]


def _run(name):
    exe = os.path.join(DIR, "test_" + name)
    if not os.path.exists(exe):
        pytest.skip("conformance binaries not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1800)
    summary = (r.stdout.strip().splitlines() or [""])[-1]
    assert r.returncode == 0, summary + "\n" + r.stderr[-4000:]
    assert "| 0 failed" in summary, summary


@pytest.mark.parametrize("name", HOST_ONLY)
def test_reference_suite_host(name):
    _run(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", HOST_ONLY + DEVICE)
def test_reference_suite_on_device(name):
    _run(name)
