"""The C++ drop-in surface (cpp/gridgnn/ggb.hpp): compiles against the C ABI on
CPU; its acceptance-style program (tests/cpp/test_dropin.cpp) runs on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_dropin_header_compiles_and_links():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgridgnn_ref.so")):
        pytest.skip("oracle/_ref not built")
    _build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_acceptance_on_gpu():
    if not os.path.exists(BIN):
        _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 5
