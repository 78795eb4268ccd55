"""CPU: the drop-in C-ABI library loads and exports every symbol include/knnj_c.h declares.

No compute calls here (no GPU in the CPU tier)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "knnj_c.h")
LIB = os.path.join(ROOT, "paper_1810_04758_b200", "libknnj_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(knnj_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.dirname(LIB)], check=True)
    return ctypes.CDLL(LIB)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("knnj_create", "knnj_set_points", "knnj_reorder_by_variance", "knnj_eps_mean",
                 "knnj_histogram", "knnj_grid_build", "knnj_split", "knnj_dense_join",
                 "knnj_exact_knn", "knnj_run"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_1810_04758_b200 import _capi
    bound = {name for name, _, _ in _capi.SIGNATURES}
    assert set(declared_symbols()) <= bound


def test_abi_version_without_gpu(lib):
    lib.knnj_abi_version.restype = ctypes.c_int
    assert lib.knnj_abi_version() == 5


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_adapter_header_compiles_against_reference_headers():
    """include/knnj_knnjoin_adapter.hpp is valid C++20 against the reference's own
    knnjoin headers (the drop-in a maintainer adds)."""
    import shutil
    import subprocess
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc) or not shutil.which("g++"):
        pytest.skip("reference headers / g++ not available")
    src = '#include "knnj_knnjoin_adapter.hpp"\nint main() { return 0; }\n'
    p = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        "-I", ref_inc, "-x", "c++", "-"], input=src, capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
