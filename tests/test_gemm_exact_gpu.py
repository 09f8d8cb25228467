"""EXACT numerics on the GPU vs the oracle (pinned bitwise to the reference
engine): bitwise-identical C (including never-touched gap bytes of general
storage) and identical FlopCounter values, over all 128 labels and the
conformance harness's variants (conformance.cpp:131-203)."""
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_LABELS, Problem, SCALARS, config

pytestmark = pytest.mark.gpu


def run_both(p: Problem, alpha, beta, kv):
    cfg_exact = config({**kv, "gpu.numerics": "exact"})
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    f_ref = O.orc_gemm(alpha, va, vb, beta, vw, config(kv))
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    f_gpu = M.gemm(alpha, da, db, beta, dc, cfg_exact)
    return dC.bytes(), want.buf, f_gpu, f_ref


@pytest.mark.parametrize("label", ALL_LABELS)
def test_exact_sizes(label):
    for s in (7, 16, 17, 64):
        p = Problem(label, s, s, s)
        got, want, fg, fr = run_both(p, SCALARS["p7"], SCALARS["m3"], {})
        assert got.tobytes() == want.tobytes(), (label, s)
        assert fg == fr
    p = Problem(label, 13, 7, 19, variant="rectangular")
    got, want, fg, fr = run_both(p, SCALARS["cfg2_alpha_real"], SCALARS["cfg2_beta"], {})
    assert got.tobytes() == want.tobytes()
    assert fg == fr


VARIANTS = [
    dict(c_kind="row"), dict(c_kind="gen"), dict(trans_a=True), dict(trans_b=True),
    dict(conj_a=True), dict(conj_b=True), dict(c_kind="row", trans_a=True, trans_b=True),
    dict(c_kind="gen", trans_a=True, conj_a=True, conj_b=True),
]
CONFIGS = [{}, {"ctemp.enable": "off", "gemm.kc": "8"}, {"ukr.preference": "row"},
           {"ctemp.enable": "on", "gemm.threads": "3"}, {"gemm.kc": "6", "gemm.mc": "16", "gemm.nc": "16"}]


@pytest.mark.parametrize("label", ALL_LABELS[::2])
def test_exact_variants_and_configs(label):
    for i, var in enumerate(VARIANTS):
        kv = CONFIGS[i % len(CONFIGS)]
        p = Problem(label, 17, 17, 17, variant=f"v{i}", **var)
        for al, be in (("one", "one"), ("p7", "c34"), ("minus_one", "zero")):
            got, want, fg, fr = run_both(p, SCALARS[al], SCALARS[be], kv)
            assert got.tobytes() == want.tobytes(), (label, var, kv, al, be)
            assert fg == fr


@pytest.mark.parametrize("label", ["zzzd", "cccs", "zczd", "czzs", "zdzd", "dzzd", "sddd", "cdds"])
def test_exact_multi_kc_blocks(label):
    # several KC blocks: per-block combine, 1m first-block temp + direct continuation
    for kv in ({"gemm.kc": "16", "ctemp.enable": "off"}, {"gemm.kc": "16"}, {"gemm.kc": "16", "ukr.preference": "row"}):
        for be in ("cfg2_beta", "p3", "one", "zero"):
            p = Problem(label, 12, 8, 40)
            got, want, fg, fr = run_both(p, SCALARS["cfg2_alpha_real"], SCALARS[be], kv)
            assert got.tobytes() == want.tobytes(), (label, kv, be)
            assert fg == fr


def test_exact_empty_dimensions():
    for label in ("zzzd", "dssd", "cdds", "szzs"):
        for (m, n, k) in ((3, 2, 0), (0, 4, 3), (4, 0, 2)):
            p = Problem(label, m, n, k)
            beta = M.Scalar.complex_value(0.0, 1.0) if label[0] in "cz" else M.Scalar.real_value(-2.0)
            got, want, fg, fr = run_both(p, SCALARS["p7"], beta, {})
            assert got.tobytes() == want.tobytes()
            assert fg == fr == 0


def test_exact_host_pointer_staging():
    # views over host memory are staged through HBM by gemm()
    p = Problem("zczd", 20, 30, 25)
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    O.orc_gemm(SCALARS["cfg3_alpha"], va, vb, SCALARS["cfg2_beta"], vw)
    got = p.C.clone()
    _, _, vg = p.views(C=got)
    M.gemm(SCALARS["cfg3_alpha"], va, vb, SCALARS["cfg2_beta"], vg, config({"gpu.numerics": "exact"}))
    assert got.buf.tobytes() == want.buf.tobytes()
