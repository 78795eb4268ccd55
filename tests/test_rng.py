"""The block-generated mt19937_64 pair draw used by knnj_run's eps_mean phase
(paper_1810_04758_b200/csrc/knnj_rng.hpp) must reproduce the reference's
std::mt19937_64 + std::uniform_int_distribution<uint64_t> stream exactly
(estimate_eps_mean, proj/src/epsilon.cpp:14-44), and the fast query sampler must return
what the reference's sample_without_replacement returns (util.hpp:70-92). CPU only."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_block_mt64_pairs_match_std(tmp_path):
    exe = str(tmp_path / "rng_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_1810_04758_b200", "csrc"),
                    os.path.join(ROOT, "tests", "rng_check.cpp"),
                    os.path.join(ROOT, "paper_1810_04758_b200", "csrc", "knnj_rng.cpp"), "-o", exe],
                   check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout
