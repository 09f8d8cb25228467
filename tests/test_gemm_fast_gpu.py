"""FAST numerics (DMMA fp64 / FFMA fp32 mainloops) vs the oracle.

Bar (BASELINE.json north_star): relative Frobenius error of C against the
reference result <= 4*k*eps_comp.  For labels whose computation precision is
wider than C's storage precision, a reordered fp64 sum legitimately flips
some roundings of the single-precision store, so the bound there is
4*k*eps_comp + eps_out and no element may differ by more than one storage
ulp.  Every run must also satisfy the reference's own
per-element criterion max_violation <= 1 (oracle.cpp:169-206)."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import (ALL_LABELS, HostMatrix, Problem, SCALARS, config, frob_bound, label_dtypes,
                           rel_frobenius)

pytestmark = pytest.mark.gpu


def run_fast(p: Problem, alpha, beta, kv=None):
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    flops = M.gemm(alpha, da, db, beta, dc, config({**(kv or {}), "gpu.numerics": "fast"}))
    out = p.C.clone()
    out.buf[:] = dC.bytes()
    return out, flops


def check(p: Problem, alpha, beta, kv=None):
    got, flops = run_fast(p, alpha, beta, kv)
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    f_ref = O.orc_gemm(alpha, va, vb, beta, vw, config(kv or {}))
    assert flops == f_ref
    _, _, vc = p.views()
    _, _, vg = p.views(C=got)
    viol = O.orc_violation(alpha, va, vb, beta, vc, vg, p.comp)
    assert viol <= 1.0, (p.label, viol)
    err = rel_frobenius(got.values(), want.values())
    assert err <= frob_bound(p.label, p.k), (p.label, err, frob_bound(p.label, p.k))
    return err


@pytest.mark.parametrize("label", ALL_LABELS)
def test_fast_all_labels(label):
    for s in (7, 16, 17, 64, 129):
        check(Problem(label, s, s, s), SCALARS["p7"], SCALARS["m3"])
    check(Problem(label, 13, 7, 19, variant="rectangular"), SCALARS["cfg2_alpha_real"], SCALARS["cfg2_beta"])


@pytest.mark.parametrize("label", ALL_LABELS[1::3])
def test_fast_variants(label):
    variants = [dict(c_kind="row"), dict(c_kind="gen"), dict(trans_a=True, conj_a=True),
                dict(trans_b=True, conj_b=True), dict(c_kind="gen", trans_a=True, trans_b=True)]
    for i, var in enumerate(variants):
        for al, be in (("one", "one"), ("minus_one", "c34"), ("p7", "zero")):
            check(Problem(label, 33, 21, 45, variant=f"f{i}", **var), SCALARS[al], SCALARS[be],
                  [{}, {"ukr.preference": "row"}, {"ctemp.enable": "off"}][i % 3])


@pytest.mark.parametrize("label", ["dssd", "zzzd", "cdds", "szzs", "zczd", "sddd", "cccs", "ddds"])
def test_fast_larger_shapes(label):
    # several CTA tiles, partial edge tiles, k not a multiple of the 16-deep stage
    for (m, n, k) in ((300, 257, 333), (128, 128, 16), (1, 513, 7), (515, 3, 129)):
        check(Problem(label, m, n, k), SCALARS["one"], SCALARS["cfg2_beta"] if label[0] in "cz" else SCALARS["p3"])


def test_beta_zero_never_reads_c():
    # acceptance.cpp:241-262: a C of all-ones bytes (NaN payloads) must not leak
    for label in ("dddd", "zzzd", "sssd", "sddd", "cccs"):
        p = Problem(label, 16, 16, 16)
        p.C.buf[:] = 0xFF
        got, _ = run_fast(p, SCALARS["one"], SCALARS["zero"])
        assert np.all(np.isfinite(got.values()))
    # case 1c updates Re(C) only: the poisoned Im(C) bits must come through untouched
    p = Problem("cdds", 16, 16, 16)
    p.C.buf[:] = 0xFF
    got, _ = run_fast(p, SCALARS["one"], SCALARS["zero"])
    assert np.all(np.isfinite(got.values().real))
    assert np.all(got.values().imag.view(np.uint32) == 0xFFFFFFFF)


def test_unread_imaginary_parts():
    # acceptance.cpp:196-239: Im(A) (1a), Im(B) (1b) never read; Im(C) (1c) bitwise untouched
    for label, which in (("dzdd", "A"), ("ddzd", "B"), ("zddd", "C")):
        p = Problem(label, 16, 16, 48)
        mat = {"A": p.A, "B": p.B, "C": p.C}[which]
        vals = mat.values()
        vals.imag = np.nan
        before = p.C.clone()
        got, _ = run_fast(p, SCALARS["one"], SCALARS["p7"], {"gemm.kc": "16", "ctemp.enable": "on"})
        if which == "C":
            assert np.array_equal(got.values().imag.view(np.int64), before.values().imag.view(np.int64))
            assert np.all(np.isfinite(got.values().real))
        else:
            assert np.all(np.isfinite(got.values()))


def test_scalar_policy_rejection_before_device_work():
    p = Problem("zdzd", 4, 4, 4)
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    before = dC.bytes().copy()
    with pytest.raises(M.ScalarPolicyError):
        M.gemm(SCALARS["c55"], da, db, SCALARS["one"], dc)
    assert np.array_equal(before, dC.bytes())


def test_stream_ordered_entry_points_refuse_host_operands():
    p = Problem("dddd", 8, 8, 8)
    va, vb, vc = p.views()  # host memory
    with pytest.raises(M.Error, match="device memory"):
        M.gemm_async(SCALARS["one"], va, vb, SCALARS["one"], vc)
    pl = M.plan(SCALARS["one"], va, vb, SCALARS["one"], vc)
    with pytest.raises(M.Error, match="device memory"):
        M.execute(pl)
    # the context is still healthy afterwards
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(SCALARS["one"], da, db, SCALARS["one"], dc)


def test_alias_rejected():
    h = HostMatrix(M.DT_D, 4, 4).fill(3).to_device()
    with pytest.raises(M.Error):
        M.gemm(SCALARS["one"], h.view(), h.view(), SCALARS["one"], h.view())
