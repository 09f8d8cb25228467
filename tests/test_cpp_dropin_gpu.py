"""The C++ API as a drop-in: tests/cpp/drop_in.cpp is written against the
reference's public header names (mdgemm/dispatch.hpp) with host buffers and
linked to libmdgemm_b200.so.  EXACT results must equal the oracle bitwise,
FAST results must meet the reference's per-element bound, and the scalar
policy must throw the reference's exception type."""
import os
import subprocess

import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, frob_bound, rel_frobenius

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "drop_in")


def run(p: Problem, alpha, beta, numerics, tmp_path):
    files = {}
    for name, mat in (("A", p.A), ("B", p.B), ("C", p.C)):
        files[name] = tmp_path / f"{name}.bin"
        mat.buf.tofile(files[name])
    out = tmp_path / "out.bin"
    r = subprocess.run([BIN, p.label, str(p.m), str(p.n), str(p.k), repr(alpha.re), repr(alpha.im), repr(beta.re),
                        repr(beta.im), numerics, str(files["A"]), str(files["B"]), str(files["C"]), str(out)],
                       capture_output=True, text=True, timeout=120)
    return r, (np.fromfile(out, np.uint8) if out.exists() else None)


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/drop_in not built")
@pytest.mark.parametrize("label", ["zzzd", "dssd", "cdds", "sddd", "zczd", "szzs", "ccsd", "dzdd"])
def test_cpp_drop_in(label, tmp_path):
    p = Problem(label, 37, 29, 41, seed=3)
    cid = M.CaseLabel.parse(label).case_id()
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    beta = SCALARS["cfg2_beta"]
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    O.orc_gemm(alpha, va, vb, beta, vw)
    r, got = run(p, alpha, beta, "exact", tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    assert got.tobytes() == want.buf.tobytes()
    r, got = run(p, alpha, beta, "fast", tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    after = p.C.clone()
    after.buf[:] = got
    _, _, vc = p.views()
    _, _, va_after = p.views(C=after)
    assert O.orc_violation(alpha, va, vb, beta, vc, va_after, p.comp) <= 1.0
    assert rel_frobenius(after.values(), want.values()) <= frob_bound(label, p.k)
    if cid not in (0, 7):
        r, _ = run(p, SCALARS["c55"], beta, "fast", tmp_path)
        assert r.returncode == 3 and "ScalarPolicyError" in r.stdout
