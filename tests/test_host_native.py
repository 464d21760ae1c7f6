"""Host candidate-production code, natively: scripts/native/host_bench.cpp is
compiled against include/evoir and libgevo_b200.so and checks that the
in-place apply_patch equals the left fold of apply_edit (the reference's
definition, src/genome.cpp:216-227) on random walks and on their messy
crossover children (many edits no longer apply), for every corpus kernel, and
that the verdict-only is_valid equals validate().empty() on thousands of
unfiltered (mostly invalid) mutation and crossover children."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2004_08140_b200")


@pytest.fixture(scope="module")
def host_bench(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libgevo_b200.so")):
        pytest.skip("library not built")
    exe = str(tmp_path_factory.mktemp("native") / "host_bench")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "scripts", "native", "host_bench.cpp"), "-L" + LIBDIR,
                    "-lgevo_b200", "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("bench", ["nw-sync", "lud-store", "hot-branch", "bfs-load", "lud-unroll",
                                   "hot-memo"])
def test_in_place_apply_patch_equals_edit_fold(host_bench, bench):
    out = subprocess.run([host_bench, bench, "16"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 mismatches" in out.stdout, out.stdout
    assert " 0 validity mismatches" in out.stdout, out.stdout
