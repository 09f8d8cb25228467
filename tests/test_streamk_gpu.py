"""Stream-K schedule (common.cuh: make_sched): the tiles x k-blocks of a
launch are cut into one equal range per CTA slot and a tile split between
two CTAs is finished by the second one, seeded with the first one's
accumulators.  The element-wise rounding sequence is therefore the classic
grid's: results must be BITWISE equal to the classic schedule (and so to any
column shard), on both kernels, every C datatype, edge tiles and 1m."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu


def run(p, alpha, beta, mode, monkeypatch):
    monkeypatch.setenv("MDGEMM_STREAMK", mode)
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(alpha, da, db, beta, dc, config({"gpu.numerics": "fast"}))
    return dC.bytes()


# shapes with more 64x128 tiles than the 296 CTA slots and a ragged last wave
SHAPES = [(1100, 4700, 300), (2000, 2500, 517), (1088, 4480, 64)]


@pytest.mark.parametrize("label", ["dddd", "ssss", "sddd", "zzzd", "cccs", "cdds", "zdzs", "szzs", "zczd", "dssd"])
@pytest.mark.parametrize("shape", SHAPES)
def test_streamk_bitwise_equals_classic(label, shape, monkeypatch):
    m, n, k = shape
    if M.CaseLabel.parse(label).case_id() == 7:  # 1m doubles both real dims
        m, n = m // 2, n // 2
    p = Problem(label, m, n, k, seed=11)
    cid = M.CaseLabel.parse(label).case_id()
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    beta = SCALARS["cfg2_beta"]
    classic = run(p, alpha, beta, "-1", monkeypatch)
    sk = run(p, alpha, beta, "1", monkeypatch)
    assert np.array_equal(classic, sk)


@pytest.mark.parametrize("label", ["dddd", "ssss"])
def test_streamk_against_oracle(label, monkeypatch):
    p = Problem(label, 1100, 4700, 96, seed=3)
    out = run(p, SCALARS["p7"], SCALARS["cfg2_beta"], "1", monkeypatch)
    after = p.C.clone()
    after.buf[:] = out
    va, vb, vc = p.views()
    _, _, va_after = p.views(C=after)
    assert O.orc_violation(SCALARS["p7"], va, vb, SCALARS["cfg2_beta"], vc, va_after, p.comp) <= 1.0


def test_streamk_repeatable(monkeypatch):
    p = Problem("dddd", 2000, 2500, 700, seed=9)
    a = run(p, SCALARS["p7"], SCALARS["cfg2_beta"], "1", monkeypatch)
    b = run(p, SCALARS["p7"], SCALARS["cfg2_beta"], "1", monkeypatch)
    assert np.array_equal(a, b)
