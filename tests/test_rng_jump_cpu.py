"""The producer's xoshiro256++ jump-ahead (k1_window): the J-step bit matrix and
its two-column table equal J plain steps of the reference generator
(rng.hpp:23-33). Host-only: tools/jump_check.cu compiled with nvcc (no GPU)."""
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not installed")
def test_jump_matrix_and_table_equal_stepping(tmp_path):
    exe = tmp_path / "jump_check"
    subprocess.run(["nvcc", "-std=c++17", "-O2", "-I", os.path.join(REPO, "paper_1908_00210_b200", "csrc"),
                    os.path.join(REPO, "tools", "jump_check.cu"), "-o", str(exe)], check=True,
                   capture_output=True, timeout=300)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=120)
    assert out.stdout.strip() == "ok", out.stdout
