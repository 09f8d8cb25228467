"""Every CTA tile configuration of both fast kernels, forced through the
tuning overrides (MDGEMM_DMMA_TILE / MDGEMM_FFMA_TILE), on a problem whose
inner dimension wraps the 4-stage TMA ring many times: results must be
repeatable bit for bit and meet the reference's per-element bound on
sampled sub-blocks.  (This is the test that caught a cross-proxy race in one
configuration that the size heuristics rarely select.)"""
import os

import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tile", ["64", "128", "64128"])
@pytest.mark.parametrize("label", ["dddd", "zzzd", "sddd", "ssss", "cccs", "szzs", "zdzs", "cdds"])
def test_forced_tile(label, tile, monkeypatch):
    import torch
    monkeypatch.setenv("MDGEMM_DMMA_TILE", tile)
    monkeypatch.setenv("MDGEMM_FFMA_TILE", tile)
    p = Problem(label, 300, 260, 700, seed=11)
    cid = M.CaseLabel.parse(label).case_id()
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    outs = []
    for _ in range(2):
        dA, dB, dC = p.device()
        da, db, dc = p.views(A=dA, B=dB, C=dC)
        M.gemm(alpha, da, db, SCALARS["cfg2_beta"], dc, config({"gpu.numerics": "fast"}))
        outs.append(dC.bytes())
    assert np.array_equal(outs[0], outs[1]), "not repeatable"
    after = p.C.clone()
    after.buf[:] = outs[0]
    va, vb, vc = p.views()
    _, _, va_after = p.views(C=after)
    assert O.orc_violation(alpha, va, vb, SCALARS["cfg2_beta"], vc, va_after, p.comp) <= 1.0
