"""Warp-specialised persistent DMMA kernel (gemm_dmma_ws.cu): 128x128 tiles,
one CTA per SM, epilogue warps draining the previous tile.  Its per-element
accumulation order is the classic kernel's (same DMMA sequence over k), so
results must be BITWISE equal to the classic kernels -- with and without the
stream-K tail -- on every C datatype, pairing and edge shape."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu


def run(p, alpha, beta, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(alpha, da, db, beta, dc, config({"gpu.numerics": "fast"}))
    return dC.bytes()


SHAPES = [(2100, 2500, 300), (2176, 2304, 64), (1999, 2561, 517)]


@pytest.mark.parametrize("label", ["dddd", "sddd", "zzzd", "zczd", "cdzd", "dssd", "zdcd", "sscd"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("streamk", ["0", "-1"])
def test_ws_bitwise_equals_classic(label, shape, streamk, monkeypatch):
    m, n, k = shape
    cid = M.CaseLabel.parse(label).case_id()
    if cid == 7:
        m = m // 2
    p = Problem(label, m, n, k, seed=17)
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    beta = SCALARS["cfg2_beta"]
    classic = run(p, alpha, beta, {"MDGEMM_DMMA_WS": "-1", "MDGEMM_STREAMK": "-1"}, monkeypatch)
    ws = run(p, alpha, beta, {"MDGEMM_DMMA_WS": "1", "MDGEMM_STREAMK": streamk}, monkeypatch)
    assert np.array_equal(classic, ws)


@pytest.mark.parametrize("beta", ["zero", "one", "cfg2_beta"])
def test_ws_against_oracle(beta, monkeypatch):
    p = Problem("dddd", 2100, 2500, 40, seed=5)
    out = run(p, SCALARS["p7"], SCALARS[beta], {"MDGEMM_DMMA_WS": "1"}, monkeypatch)
    after = p.C.clone()
    after.buf[:] = out
    va, vb, vc = p.views()
    _, _, va_after = p.views(C=after)
    assert O.orc_violation(SCALARS["p7"], va, vb, SCALARS[beta], vc, va_after, p.comp) <= 1.0


@pytest.mark.parametrize("label", ["ssss", "dsss", "cccs", "cdzs", "zdzs", "szzs", "sdds", "csds",
                                   "cdds", "csss", "zdds"])  # 1c: the real part of a complex C
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("streamk", ["0", "-1"])
def test_ffma_ws_bitwise_equals_classic(label, shape, streamk, monkeypatch):
    m, n, k = shape
    cid = M.CaseLabel.parse(label).case_id()
    if cid == 7:
        m = m // 2
    p = Problem(label, m, n, k, seed=19)
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    beta = SCALARS["cfg2_beta"]
    classic = run(p, alpha, beta, {"MDGEMM_FFMA_WS": "-1", "MDGEMM_STREAMK": "-1"}, monkeypatch)
    ws = run(p, alpha, beta, {"MDGEMM_FFMA_WS": "1", "MDGEMM_STREAMK": streamk}, monkeypatch)
    assert np.array_equal(classic, ws)
