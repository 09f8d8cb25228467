"""The reference conformance harness's scalar sweep, replayed against the GPU
path for all 128 labels (conformance.cpp:178-203): alpha in {0, 1, -1, 0.7}
x beta in {0, 1, 0.3, 0.3+0.4i} at m=n=k=16, then a complex alpha 0.5+0.5i
that cases 0 and 3 honour and the six others reject with ScalarPolicyError
before any device work (dispatch.cpp:56-85).

Each point runs in both numerics: EXACT must reproduce the oracle (pinned
bitwise to the reference engine) byte for byte with the same FlopCounter
value; FAST must meet the reference's per-element criterion
max_violation <= 1 (oracle.cpp:169-206, what run_one asserts,
conformance.cpp:120-126) and the north-star relative Frobenius bound.
alpha = 0 is the case the earlier suites never ran: the product must still
apply beta (and only beta) to C."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_LABELS, Problem, config, frob_bound, rel_frobenius

pytestmark = pytest.mark.gpu

ALPHAS = [M.Scalar.real_value(0.0), M.Scalar.real_value(1.0), M.Scalar.real_value(-1.0), M.Scalar.real_value(0.7)]
BETAS = [M.Scalar.real_value(0.0), M.Scalar.real_value(1.0), M.Scalar.real_value(0.3),
         M.Scalar.complex_value(0.3, 0.4)]
COMPLEX_ALPHA = M.Scalar.complex_value(0.5, 0.5)
S = 16


def _oracle(p: Problem, alpha, beta):
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    flops = O.orc_gemm(alpha, va, vb, beta, vw)
    return want, flops


def _gpu(p: Problem, alpha, beta, numerics):
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    flops = M.gemm(alpha, da, db, beta, dc, config({"gpu.numerics": numerics}))
    got = p.C.clone()
    got.buf[:] = dC.bytes()
    return got, flops


@pytest.mark.parametrize("label", ALL_LABELS)
def test_scalar_grid(label):
    for ai, alpha in enumerate(ALPHAS):
        for bi, beta in enumerate(BETAS):
            p = Problem(label, S, S, S, variant=f"scalars{ai}{bi}")
            want, f_ref = _oracle(p, alpha, beta)
            got, f_gpu = _gpu(p, alpha, beta, "exact")
            assert got.buf.tobytes() == want.buf.tobytes(), (label, ai, bi, "exact")
            assert f_gpu == f_ref
            got, f_gpu = _gpu(p, alpha, beta, "fast")
            assert f_gpu == f_ref
            va, vb, vc = p.views()
            _, _, vg = p.views(C=got)
            viol = O.orc_violation(alpha, va, vb, beta, vc, vg, p.comp)
            assert viol <= 1.0, (label, ai, bi, viol)
            err = rel_frobenius(got.values(), want.values())
            assert err <= frob_bound(label, S), (label, ai, bi, err)
            if ai == 0:
                # alpha = 0: every product is a zero, so FAST gives the reference's
                # beta*C values exactly (signed zeros aside: +0 and -0 compare equal)
                assert np.array_equal(got.values(), want.values()), (label, bi, "alpha=0 fast")


@pytest.mark.parametrize("label", ALL_LABELS)
def test_complex_alpha_policy(label):
    p = Problem(label, S, S, S, variant="complex_alpha")
    rejects = label_case(label) not in (0, 7)
    for numerics in ("exact", "fast"):
        dA, dB, dC = p.device()
        before = dC.bytes().copy()
        da, db, dc = p.views(A=dA, B=dB, C=dC)
        if rejects:
            with pytest.raises(M.ScalarPolicyError):
                M.gemm(COMPLEX_ALPHA, da, db, M.Scalar.real_value(1.0), dc, config({"gpu.numerics": numerics}))
            assert np.array_equal(dC.bytes(), before), "C changed although the call was rejected"
        else:
            want, f_ref = _oracle(p, COMPLEX_ALPHA, M.Scalar.real_value(1.0))
            got, f_gpu = _gpu(p, COMPLEX_ALPHA, M.Scalar.real_value(1.0), numerics)
            assert f_gpu == f_ref
            if numerics == "exact":
                assert got.buf.tobytes() == want.buf.tobytes()
            else:
                assert rel_frobenius(got.values(), want.values()) <= frob_bound(label, S)


def label_case(label: str) -> int:
    """Case id (0, 1a, 1b, 1c, 2ab, 2ac, 2bc, 3 -> 0..7) from the domains of C, A, B (case_label.cpp:11-26)."""
    cx = [ch in "cz" for ch in label[:3]]
    return M.classify_case(*cx)
