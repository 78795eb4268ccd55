"""GPU: the C++ drop-in adapter (include/knnj_knnjoin_adapter.hpp) against the
reference's own run_hybrid, in one C++ program (tests/adapter_check.cpp, built by
`make -C oracle adapter` where /root/reference exists; the binary travels with the
repo snapshot). Byte-identical io::tsv_string output, provenance, eps, failed
counts, for all four engine modes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")

pytestmark = pytest.mark.gpu


def test_reference_run_hybrid_equals_adapter():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "ADAPTER OK" in p.stdout
