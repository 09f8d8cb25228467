"""Pins the C restatement (oracle/mdg_oracle.c) to the reference engine
itself (oracle/_ref, built from /root/reference/proj/src) -- bitwise -- so
the GPU parity tests can trust it.  CPU only."""
import itertools

import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_DT, ALL_LABELS, HostMatrix, Problem, SCALARS, config

needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("dtype", ALL_DT)
@pytest.mark.parametrize("kind", ["col", "row", "gen"])
def test_rng_fill_matches_reference(dtype, kind):
    path = ["zcsd", "bench", 12345, "a"]
    mine, theirs = HostMatrix(dtype, 7, 5, kind), HostMatrix(dtype, 7, 5, kind)
    O.orc_fill_uniform(mine.view(), O.orc_rng_state(99, path))
    O.ref_fill_uniform_path(theirs.view(), 99, path)
    assert mine.buf.tobytes() == theirs.buf.tobytes()


def _plan_variants():
    for label in ALL_LABELS:
        yield label, "col", False, False, False, False, {}
    for label in ALL_LABELS[::3]:
        yield label, "row", False, False, False, False, {}
        yield label, "gen", True, False, True, True, {}
        yield label, "col", False, True, False, True, {"ukr.preference": "row"}
        yield label, "row", True, True, True, False, {"ctemp.enable": "off"}
        yield label, "col", False, False, False, False, {"ctemp.enable": "on", "gemm.threads": "4"}
        yield label, "col", False, False, False, False, {"gemm.threads": "4"}
        yield label, "col", False, False, False, False, {"gemm.kc": "8"}


@needs_ref
def test_plan_matches_reference_on_all_labels():
    n = 0
    for label, kind, ta, tb, ca, cb, kv in _plan_variants():
        p = Problem(label, 9, 10, 11, c_kind=kind, trans_a=ta, trans_b=tb, conj_a=ca, conj_b=cb)
        va, vb, vc = p.views()
        cfgv = config(kv)
        for alpha, beta in [("p7", "m3"), ("cfg2_alpha_real", "cfg2_beta"), ("one", "zero")]:
            got = O.orc_plan(SCALARS[alpha], va, vb, SCALARS[beta], vc, cfgv).as_dict(with_pointers=True)
            want = O.ref_plan(SCALARS[alpha], va, vb, SCALARS[beta], vc, cfgv).as_dict(with_pointers=True)
            assert got == want, (label, kind, kv)
            n += 1
    assert n > 400


@needs_ref
def test_scalar_policy_rejections_match_reference():
    for label in ALL_LABELS:
        p = Problem(label, 3, 3, 3)
        va, vb, vc = p.views()
        outcomes = []
        for fn in (O.orc_plan, O.ref_plan):
            try:
                fn(SCALARS["c55"], va, vb, SCALARS["one"], vc)
                outcomes.append("ok")
            except O.ScalarPolicyError:
                outcomes.append("policy")
        assert outcomes[0] == outcomes[1], label
        cid = M.CaseLabel.parse(label).case_id()
        assert outcomes[0] == ("ok" if cid in (0, 7) else "policy"), label


def _pack_cases():
    for dt, side, fmt, conj in itertools.product(ALL_DT, (M.LEFT, M.RIGHT), (M.STANDARD, M.ONE_E, M.ONE_R), (0, 1)):
        if fmt != M.STANDARD and not M.is_complex(dt):
            continue
        for target_prec in (M.SINGLE, M.DOUBLE):
            target = (2 if M.is_complex(dt) and fmt == M.STANDARD else 0) + target_prec
            for scale in ("one", "p7", "minus_one", "cfg3_alpha"):
                if scale == "cfg3_alpha" and fmt == M.STANDARD:
                    continue
                for rb in ((2, 4) if fmt == M.ONE_E else (1, 3, 4)):
                    yield dt, side, fmt, conj, target, scale, rb


@needs_ref
def test_pack_matches_reference_bitwise():
    count = 0
    for dt, side, fmt, conj, target, scale, rb in _pack_cases():
        for kind, src_conj in (("col", False), ("gen", True), ("row", False)):
            src = HostMatrix(dt, 5, 7, kind).fill(O.orc_rng_state(3, ["pack", dt, side, fmt, kind]))
            v = src.view(conj=src_conj and M.is_complex(dt))
            nbytes = O.orc_packed_bytes(v, side, fmt, target, rb)
            assert nbytes == O.ref_packed_bytes(v, side, fmt, target, rb)
            mine = np.full(nbytes, 0x5A, np.uint8)
            theirs = np.full(nbytes, 0xA5, np.uint8)
            O.orc_pack(v, side, fmt, conj, SCALARS[scale], target, rb, 0, mine.ctypes.data)
            O.ref_pack(v, side, fmt, conj, SCALARS[scale], target, rb, theirs.ctypes.data, nbytes)
            assert mine.tobytes() == theirs.tobytes(), (dt, side, fmt, conj, target, scale, rb, kind)
            count += 1
    assert count > 300


@needs_ref
def test_pack_errors_match_reference():
    src = HostMatrix(M.DT_Z, 2, 2).fill(1)
    real = HostMatrix(M.DT_D, 2, 2).fill(1)
    bad = [
        (src.view(), M.LEFT, M.STANDARD, SCALARS["c55"], M.DT_Z, 4),   # complex scale on Standard
        (real.view(), M.LEFT, M.ONE_E, SCALARS["one"], M.DT_D, 4),     # expanding format, real source
        (real.view(), M.RIGHT, M.ONE_R, SCALARS["one"], M.DT_D, 4),
        (src.view(), M.LEFT, M.ONE_E, SCALARS["one"], M.DT_Z, 3),      # odd reg_block for 1e
        (src.view(), M.LEFT, M.STANDARD, SCALARS["one"], M.DT_D, 4),   # Standard changing domain
        (src.view(), M.LEFT, M.ONE_R, SCALARS["one"], M.DT_Z, 0),      # reg_block < 1
    ]
    buf = np.zeros(4096, np.uint8)
    for v, side, fmt, sc, tgt, rb in bad:
        with pytest.raises(O.Error):
            O.orc_pack(v, side, fmt, 0, sc, tgt, rb, 0, buf.ctypes.data)
        with pytest.raises(O.Error):
            O.ref_pack(v, side, fmt, 0, sc, tgt, rb, buf.ctypes.data, buf.size)


def _gemm_cases():
    for label in ALL_LABELS:
        for s in (7, 16, 17):
            yield label, s, s, s, {}, "col", (False, False, False, False), ("p7", "m3")
        yield label, 13, 7, 19, {}, "col", (False, False, False, False), ("cfg2_alpha_real", "cfg2_beta")
    for label in ALL_LABELS[::2]:
        yield label, 9, 10, 11, {"gemm.mc": "8", "gemm.nc": "8", "gemm.kc": "4"}, "col", (False,) * 4, ("p7", "m3")
        yield label, 17, 17, 17, {"ctemp.enable": "off"}, "gen", (True, False, True, True), ("one", "c34")
        yield label, 17, 17, 17, {"ukr.preference": "row"}, "row", (False, True, False, False), ("p3", "p3")
        yield label, 12, 8, 40, {"gemm.kc": "16", "ctemp.enable": "off"}, "col", (False,) * 4, ("cfg2_alpha_real", "cfg2_beta")


@needs_ref
def test_gemm_matches_reference_bitwise_all_labels():
    count = 0
    for label, m, n, k, kv, kind, (ta, tb, ca, cb), (al, be) in _gemm_cases():
        p = Problem(label, m, n, k, c_kind=kind, trans_a=ta, trans_b=tb, conj_a=ca, conj_b=cb)
        C1, C2 = p.C.clone(), p.C.clone()
        cfgv = config(kv)
        va, vb, vc1 = p.views(C=C1)
        _, _, vc2 = p.views(C=C2)
        f1 = O.orc_gemm(SCALARS[al], va, vb, SCALARS[be], vc1, cfgv)
        f2 = O.ref_gemm(SCALARS[al], va, vb, SCALARS[be], vc2, cfgv)
        assert C1.buf.tobytes() == C2.buf.tobytes(), (label, m, n, k, kv, kind)
        assert f1 == f2, (label, f1, f2)
        count += 1
    assert count >= 128 * 4


@needs_ref
def test_empty_dimensions_match_reference():
    for label in ("zzzd", "dssd", "cdds", "szzs", "zdzs"):
        for (m, n, k) in ((3, 2, 0), (0, 4, 3), (4, 0, 2)):
            p = Problem(label, m, n, k)
            C1, C2 = p.C.clone(), p.C.clone()
            va, vb, vc1 = p.views(C=C1)
            _, _, vc2 = p.views(C=C2)
            beta = M.Scalar.complex_value(0.0, 1.0) if label[0] in "cz" else M.Scalar.real_value(-2.0)
            f1 = O.orc_gemm(SCALARS["c55"] if label[1:3] == "zz" and label[0] in "cz" else SCALARS["p7"], va, vb,
                            beta, vc1)
            f2 = O.ref_gemm(SCALARS["c55"] if label[1:3] == "zz" and label[0] in "cz" else SCALARS["p7"], va, vb,
                            beta, vc2)
            assert C1.buf.tobytes() == C2.buf.tobytes()
            assert f1 == f2 == 0


@needs_ref
def test_violation_matches_reference():
    for label in ALL_LABELS[::5]:
        p = Problem(label, 8, 9, 10)
        after = p.C.clone()
        va, vb, vc = p.views()
        _, _, va_after = p.views(C=after)
        O.ref_gemm(SCALARS["p7"], va, vb, SCALARS["m3"], va_after)
        v1 = O.orc_violation(SCALARS["p7"], va, vb, SCALARS["m3"], vc, va_after, p.comp)
        v2 = O.ref_violation(SCALARS["p7"], va, vb, SCALARS["m3"], vc, va_after, p.comp)
        assert v1 == pytest.approx(v2, rel=1e-12, abs=1e-300)
        assert v1 <= 1.0
