"""Split-K (small output, long inner dimension): partial tiles summed in split
order then the shared fused epilogue.  Results must be repeatable bit for bit
and meet the reference's per-element bound; forced split factors cover the
path on every output datatype and pairing."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, config, frob_bound, rel_frobenius

pytestmark = pytest.mark.gpu


def run(p, alpha, beta):
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(alpha, da, db, beta, dc, config({"gpu.numerics": "fast"}))
    return dC.bytes()


@pytest.mark.parametrize("label", ["dddd", "zzzd", "sddd", "ssss", "cccs", "szzs", "zdzs", "cdds", "zczd"])
@pytest.mark.parametrize("splits", ["auto", "3", "7"])
def test_splitk(label, splits, monkeypatch):
    monkeypatch.setenv("MDGEMM_SPLITK", "0" if splits == "auto" else splits)
    p = Problem(label, 70, 90, 2100, seed=5)  # small grid, long k: auto picks a split
    cid = M.CaseLabel.parse(label).case_id()
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    first, second = run(p, alpha, SCALARS["cfg2_beta"]), run(p, alpha, SCALARS["cfg2_beta"])
    assert np.array_equal(first, second)
    after = p.C.clone()
    after.buf[:] = first
    va, vb, vc = p.views()
    _, _, va_after = p.views(C=after)
    assert O.orc_violation(alpha, va, vb, SCALARS["cfg2_beta"], vc, va_after, p.comp) <= 1.0
    want = p.C.clone()
    _, _, vw = p.views(C=want)
    O.orc_gemm(alpha, va, vb, SCALARS["cfg2_beta"], vw)
    assert rel_frobenius(after.values(), want.values()) <= frob_bound(label, p.k)


def test_splitk_off_is_bitwise_the_unsplit_grid(monkeypatch):
    # gpu.splitk = off: the same call as the whole-k grid, bit for bit, on a shape where auto splits
    p = Problem("dddd", 70, 90, 2100, seed=5)
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(SCALARS["p7"], da, db, SCALARS["m3"], dc, config({"gpu.numerics": "fast", "gpu.splitk": "off"}))
    off = dC.bytes()
    monkeypatch.setenv("MDGEMM_SPLITK", "1")  # forced factor 1 = the unsplit grid
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(SCALARS["p7"], da, db, SCALARS["m3"], dc, config({"gpu.numerics": "fast"}))
    assert np.array_equal(off, dC.bytes())
