"""The product's host planner (C++ plan() behind mdg_plan) against the
reference plan() and the oracle restatement: identical ExecutionPlan for all
128 labels x storage/transpose/conj variants x configs (dispatch.cpp:106-305),
identical errors.  No device work."""
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_LABELS, Problem, SCALARS, config

VARIANTS = [dict(), dict(c_kind="row"), dict(c_kind="gen"), dict(trans_a=True, conj_a=True),
            dict(trans_b=True, conj_b=True), dict(c_kind="row", trans_a=True, trans_b=True)]
CONFIGS = [{}, {"ukr.preference": "row"}, {"ctemp.enable": "off"}, {"ctemp.enable": "on", "gemm.threads": "4"},
           {"gemm.threads": "2"}, {"gemm.kc": "8"}]


@pytest.mark.parametrize("label", ALL_LABELS)
def test_plan_identical(label):
    checker = O.ref_plan if O.ref is not None else O.orc_plan
    for i, var in enumerate(VARIANTS):
        p = Problem(label, 9, 10, 11, variant=f"p{i}", **var)
        va, vb, vc = p.views()
        for kv in CONFIGS:
            for al, be in (("p7", "m3"), ("cfg2_alpha_real", "cfg2_beta"), ("one", "zero")):
                cfgv = config(kv)
                got = M.plan(SCALARS[al], va, vb, SCALARS[be], vc, cfgv).as_dict(with_pointers=True)
                want = checker(SCALARS[al], va, vb, SCALARS[be], vc, cfgv).as_dict(with_pointers=True)
                assert got == want, (label, var, kv)
                assert got == O.orc_plan(SCALARS[al], va, vb, SCALARS[be], vc, cfgv).as_dict(with_pointers=True)


def test_plan_errors():
    from tests.helpers import HostMatrix
    a, b, c = HostMatrix(M.DT_D, 4, 5), HostMatrix(M.DT_D, 6, 3), HostMatrix(M.DT_D, 4, 3)
    with pytest.raises(M.Error, match="A is 4x5, B is 6x3"):  # test_dispatch.cpp:283-293
        M.plan(SCALARS["one"], a.view(), b.view(), SCALARS["one"], c.view())
    for label in ALL_LABELS:
        q = Problem(label, 2, 2, 2)
        a, b, c = q.views()
        cid = M.CaseLabel.parse(label).case_id()
        if cid in (0, 7):
            M.plan(SCALARS["c55"], a, b, SCALARS["one"], c)
        else:
            with pytest.raises(M.ScalarPolicyError):
                M.plan(SCALARS["c55"], a, b, SCALARS["one"], c)


def test_plan_known_structure():
    # test_dispatch.cpp:118-186
    p = Problem("zzdd", 6, 8, 10)
    a, b, c = p.views()
    pl = M.plan(SCALARS["one"], a, b, SCALARS["one"], c)
    assert (pl.case_id, pl.m, pl.n, pl.k, pl.ukr_path, pl.pair_axis) == (5, 12, 8, 10, M.PATH_DIRECT, M.PAIR_NONE)
    assert pl.reg_block_a == 2 and pl.target_dtype_a == M.DT_Z
    row = M.plan(SCALARS["one"], a, b, SCALARS["one"], c, config({"ukr.preference": "row"}))
    assert row.logical_transpose and row.case_id == 6 and (row.m, row.n) == (8, 12)
    q = Problem("cccs", 5, 5, 5)
    qa, qb, qc = q.views()
    pq = M.plan(SCALARS["one"], qa, qb, SCALARS["one"], qc)
    assert pq.case_id == 7 and pq.k == 10 and pq.format_a == M.ONE_E and pq.format_b == M.ONE_R
    r = Problem("sccs", 5, 5, 5)  # C real, A, B complex -> 2ab
    ra, rb, rc = r.views()
    pr = M.plan(SCALARS["one"], ra, rb, SCALARS["one"], rc)
    assert pr.case_id == 4 and pr.conj_b and pr.k == 10
