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


ACCEPT = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.parametrize("criterion", list(range(1, 11)))
def test_reference_acceptance_suite_on_the_dropin(criterion):
    """The reference's own acceptance suite (proj/tests/acceptance.cpp, compiled
    unchanged) linked against the link-time drop-in
    (paper_1810_04758_b200/dropin/knnjoin_dropin.cpp): run_hybrid, estimate_eps_mean,
    build_distance_histogram, GridIndex::build, split_work and run_dense_join run on the
    B200. C1: 56 random instances x {Hybrid, SparseOnly, DenseOnly} byte-identical to
    BruteOracle; C7: eps / split monotonicity through the device phases; C8: forced
    dense failures stay exact; C9: determinism of the TSV and the run report."""
    if not os.path.exists(ACCEPT):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs /root/reference at build time)")
    p = subprocess.run([ACCEPT, str(criterion)], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert f"[PASS] criterion {criterion}" in p.stdout
