"""The reference's own acceptance program (proj/tests/acceptance.cpp, its 8
acceptance criteria: oracle equivalence, greedy monotonicity, counter
integrity, known-answer quality, standard-vs-GDI scaling, balance, ...),
compiled unchanged against include/ising and linked to this repository's
libising.so by oracle/Makefile (oracle/_ref/acceptance_ours): a reference
caller that keeps working without a source change. It exits with the number
of failed criteria."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "acceptance_ours")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/acceptance_ours not built (make && make -C oracle)")
def test_reference_acceptance_program_passes_on_this_library():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
