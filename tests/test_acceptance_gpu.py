"""The reference's own acceptance test (tests/acceptance.cpp, criteria 1-10,
SURVEY 4 / 8(f)-1) built against this repo's public headers and linked to
libmdgemm_b200.so (oracle/Makefile: accept).  It calls the unchanged C++ API
-- gemm(), plan(), CaseLabel, FlopCounter, MatrixView on host Matrix
buffers -- with the reference's matrix/rng/oracle/bench code as test
infrastructure, and its criterion 10 drives this repo's bench CLI.

EXACT numerics (MDGEMM_GPU_NUMERICS=exact: bit-for-bit the reference's
rounding) must pass every criterion; FAST numerics (the default) must pass
the criteria that bound errors rather than demand the reference's bits."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
CLI = os.path.join(ROOT, "tools", "mdgemm_b200")


def run(numerics: str) -> dict:
    env = dict(os.environ, MDGEMM_GPU_NUMERICS=numerics)
    r = subprocess.run([BIN, CLI], capture_output=True, text=True, timeout=1800, env=env)
    out = {int(m.group(1)): (m.group(2) == "PASS", m.group(3))
           for m in re.finditer(r"criterion\s+(\d+): (PASS|FAIL)\s+(.*)", r.stdout)}
    assert len(out) == 10, r.stdout + r.stderr
    return out


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/acceptance_b200 not built")
def test_reference_acceptance_exact():
    res = run("exact")
    failed = {k: v[1] for k, v in res.items() if not v[0]}
    assert not failed, failed


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/acceptance_b200 not built")
def test_reference_acceptance_fast():
    res = run("fast")
    for k in (1, 2, 3, 4, 5, 6, 9, 10):
        assert res[k][0], (k, res[k][1])
