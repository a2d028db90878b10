"""Drop-in check: the reference's own Python tests
(proj/python/tests/test_smoke.py), unchanged, against this repository's
pyising. The file is copied at build time into tests/_ref/ (git-ignored;
scripts/vendor_ref_tests.sh) and run in a subprocess whose `import pyising`
resolves to paper_1908_00210_b200/pyising*.so (the reference module.cpp
names, the GPU path behind them)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
VENDORED = os.path.join(HERE, "_ref", "ref_test_smoke.py")


@pytest.mark.skipif(not os.path.exists(VENDORED), reason="reference test not vendored (scripts/vendor_ref_tests.sh)")
def test_reference_smoke_tests_unchanged():
    env = dict(os.environ, PYTHONPATH=os.path.join(REPO, "paper_1908_00210_b200"))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir",
                          os.path.dirname(VENDORED), "-c", os.devnull, VENDORED],
                         env=env, capture_output=True, text=True, timeout=600, cwd=os.path.dirname(VENDORED))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert re.search(r"\b8 passed", out.stdout), out.stdout[-2000:]
