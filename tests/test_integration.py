"""The reference-side binding (integration/b200_shim.cpp):
it compiles against the UNMODIFIED reference headers and links with the
reference core + libtt_b200.so (CPU test, needs /root/reference), and on a
GPU one reference-API round through it selects exactly the schedules the
reference's own round composition selects, and train() through it matches
the reference's train() (integration/shim_round_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "shim_round_test")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/core/include"), reason="reference headers absent")
def test_shim_compiles_against_reference_headers():
    lib = os.path.join(ROOT, "paper_2402_02361_b200", "_lib", "libtt_b200.so")
    ref = os.path.join(ROOT, "oracle", "_ref", "libtiletune_ref.a")
    if not (os.path.exists(lib) and os.path.exists(ref)):
        pytest.skip("build() first (libtt_b200.so, oracle/_ref)")
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "integration")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(BIN)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build/shim_round_test not built (build())")
def test_shim_round_matches_reference_round():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
