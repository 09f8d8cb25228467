"""Seeded random sweep over the whole input space of gemm(): label, shape
(empty, 1, odd, around the 16-step k-block and the 64/128 tiles), storage of
A, B and C (column, row, general with gaps), transposes, conjugation, the
scalars (including alpha = 0, complex beta, complex alpha where the case
allows it) and the Config keys plan() reads (ctemp, kc, row preference,
split-K off).  Each draw runs in both numerics against the oracle (pinned
bitwise to the reference engine): EXACT bitwise with the same FlopCounter,
FAST within the reference's per-element criterion and the north-star
relative Frobenius bound; never-addressed bytes of general storage must come
back untouched in both."""
import random

import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_LABELS, Problem, config, frob_bound, rel_frobenius

pytestmark = pytest.mark.gpu

DIMS = [0, 1, 2, 3, 7, 15, 16, 17, 31, 33, 63, 64, 65, 127, 128, 129, 200]
KINDS = ["col", "row", "gen"]
ALPHAS = [M.Scalar.real_value(0.0), M.Scalar.real_value(1.0), M.Scalar.real_value(-0.75),
          M.Scalar.real_value(1.2), M.Scalar.complex_value(0.5, 1.5), M.Scalar.complex_value(1.2, -0.7)]
BETAS = [M.Scalar.real_value(0.0), M.Scalar.real_value(1.0), M.Scalar.real_value(-0.3),
         M.Scalar.complex_value(0.9, 0.3), M.Scalar.complex_value(0.0, 1.0)]
CONFIGS = [{}, {"ctemp.enable": "off", "gemm.kc": "24"}, {"ctemp.enable": "on"}, {"ukr.preference": "row"},
           {"gemm.kc": "16", "gemm.threads": "4"}, {"gpu.splitk": "off"}]


def case_of(label: str) -> int:
    return M.classify_case(*[ch in "cz" for ch in label[:3]])


def draw(rng: random.Random, i: int):
    label = rng.choice(ALL_LABELS)
    m, n, k = (rng.choice(DIMS) for _ in range(3))
    alpha = rng.choice(ALPHAS)
    if case_of(label) not in (0, 7) and alpha.im != 0.0:
        alpha = M.Scalar.real_value(alpha.re)  # the six restricted cases reject it (tested elsewhere)
    p = Problem(label, m, n, k, seed=1000 + i, variant=f"fuzz{i}", c_kind=rng.choice(KINDS),
                a_kind=rng.choice(KINDS), b_kind=rng.choice(KINDS), trans_a=rng.random() < 0.3,
                trans_b=rng.random() < 0.3, conj_a=rng.random() < 0.3, conj_b=rng.random() < 0.3)
    return p, alpha, rng.choice(BETAS), rng.choice(CONFIGS)


@pytest.mark.parametrize("chunk", range(8))
def test_random_calls_against_the_oracle(chunk):
    rng = random.Random(20261020 + chunk)
    for i in range(40):
        p, alpha, beta, kv = draw(rng, chunk * 1000 + i)
        want = p.C.clone()
        va, vb, vw = p.views(C=want)
        f_ref = O.orc_gemm(alpha, va, vb, beta, vw, config(kv))
        for numerics in ("exact", "fast"):
            dA, dB, dC = p.device()
            da, db, dc = p.views(A=dA, B=dB, C=dC)
            f_gpu = M.gemm(alpha, da, db, beta, dc, config({**kv, "gpu.numerics": numerics}))
            got = p.C.clone()
            got.buf[:] = dC.bytes()
            what = (p.label, p.m, p.n, p.k, numerics, kv, p.C.kind, p.A.kind, p.B.kind)
            assert f_gpu == f_ref, what
            if numerics == "exact":
                assert got.buf.tobytes() == want.buf.tobytes(), what
                continue
            # bytes outside C's addressed elements (general storage gaps) are never written
            mask = np.zeros(p.C.buf.size, bool)
            es = M.dtype_size(p.C.dtype)
            for j in range(p.n):
                for r in range(p.m):
                    o = (r * p.C.rs + j * p.C.cs) * es
                    mask[o:o + es] = True
            assert np.array_equal(got.buf[~mask], p.C.buf[~mask]), what
            if p.m and p.n:
                _, _, vc = p.views()
                _, _, vg = p.views(C=got)
                assert O.orc_violation(alpha, va, vb, beta, vc, vg, p.comp) <= 1.0, what
                if p.k:
                    assert rel_frobenius(got.values(), want.values()) <= frob_bound(p.label, p.k), what
