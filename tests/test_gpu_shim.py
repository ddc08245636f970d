"""The C++ drop-in (include/sale_b200.hpp) on a B200: tests/cpp/test_shim.cpp,
built against the reference headers, compares sale::b200::X with the
reference's sale::X (quant, selection_pass, block_sparse_attention,
full_attention, flop_accounting, error classes)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "test_shim")


def test_cpp_shim_against_reference():
    assert os.path.exists(BIN), "tests/cpp/_build/test_shim missing: run __graft_entry__.build()"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and "ALL OK" in r.stdout
