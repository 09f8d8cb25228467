"""The fused epilogue moves C through 2-D TMA tensor maps in three layouts
(desc.h: MDG_CMAP_*): column-major C, row-major C (transposed plans, case
2bc and row-stored C) and the real part of an interleaved complex C (case
1c).  Only the data movement differs from the element-wise path (same
combine arithmetic), so both must give BITWISE identical C -- including the
untouched halves and edge tiles -- and meet the reference's bound."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu


def run(p, alpha, beta, tma, monkeypatch, kv=None):
    monkeypatch.setenv("MDGEMM_C_TMA", "1" if tma else "0")
    monkeypatch.setenv("MDGEMM_DMMA_WS", "-1")  # the classic kernels' epilogue
    monkeypatch.setenv("MDGEMM_FFMA_WS", "-1")
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(alpha, da, db, beta, dc, config({**(kv or {}), "gpu.numerics": "fast"}))
    return dC.bytes()


# 1c (C complex, A and B real), 2bc (flipped to row-major C), plain column
# and row-stored C; shapes with aligned strides, several tiles and edge tiles
LABELS = ["cdds", "zddd", "cssd", "zdzd", "zszs", "czds", "dddd", "ssss", "zzzd", "cccs"]
SHAPES = [(200, 160, 70), (96, 256, 33), (130, 64, 300)]


@pytest.mark.parametrize("label", LABELS)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("c_kind", ["col", "row"])
def test_tma_epilogue_bitwise_equals_elementwise(label, shape, c_kind, monkeypatch):
    m, n, k = shape
    p = Problem(label, m, n, k, seed=23, c_kind=c_kind)
    cid = M.CaseLabel.parse(label).case_id()
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    for beta in ("cfg2_beta", "zero", "one"):
        a = run(p, alpha, SCALARS[beta], True, monkeypatch)
        b = run(p, alpha, SCALARS[beta], False, monkeypatch)
        assert np.array_equal(a, b), (label, shape, c_kind, beta)


@pytest.mark.parametrize("label", ["cdds", "zdzd", "zszs"])
def test_tma_epilogue_against_oracle(label, monkeypatch):
    p = Problem(label, 200, 160, 70, seed=29)
    beta = SCALARS["cfg2_beta"]
    out = run(p, SCALARS["p7"], beta, True, monkeypatch)
    after = p.C.clone()
    after.buf[:] = out
    va, vb, vc = p.views()
    _, _, va_after = p.views(C=after)
    assert O.orc_violation(SCALARS["p7"], va, vb, beta, vc, va_after, p.comp) <= 1.0
