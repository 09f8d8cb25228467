"""The dual-pipe batch schedule (csrc/host/staging.cpp: dual_schedule), on the host
without a device: every launch holds only calls whose dependencies finished in
earlier launches, every dual call's tiles are covered exactly once by its pieces
(contiguous ranges, in order), a launch holds at most DUAL_MAX_JOBS jobs per group
and never two pieces of one call, and mixed batches pair FP64 with FP32 work."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from tests.helpers import HostMatrix, Problem, SCALARS, config

MAX_JOBS = 80
LABELS = [l.str() for l in M.CaseLabel.all()]


def _alpha(label):
    return SCALARS["cfg2_alpha"] if M.CaseLabel.parse(label).case_id() in (0, 7) else SCALARS["p7"]


def _windows(v):
    es = M.dtype_size(v.dtype)
    if v.m == 0 or v.n == 0:
        return None
    lo = v.base
    hi = v.base + ((v.m - 1) * v.rs + (v.n - 1) * v.cs + 1) * es
    return lo, hi


def _overlap(a, b):
    return a is not None and b is not None and a[0] < b[1] and b[0] < a[1]


def _check_schedule(calls, pieces, tiles):
    assert pieces, "expected the dual path"
    by_call = {}
    units = {}
    for unit, call, t0, t1, grp in pieces:
        by_call.setdefault(call, []).append((unit, t0, t1, grp))
        units.setdefault(unit, []).append((call, grp))
    # each call scheduled; dual calls' tiles covered exactly once, in launch order
    assert set(by_call) == set(range(len(calls)))
    finish = {}
    start = {}
    for call, ps in by_call.items():
        ps.sort()
        start[call], finish[call] = ps[0][0], ps[-1][0]
        if ps[0][3] == 0:
            assert len(ps) == 1
            continue
        assert ps[0][1] == 0 and ps[-1][2] == tiles[call]
        for (u0, _, e0, _), (u1, b1, _, _) in zip(ps, ps[1:]):
            assert u1 > u0 and b1 == e0
    # per launch: caps, one piece per call, a classic slot alone
    for unit, members in units.items():
        calls_in = [c for c, _ in members]
        assert len(calls_in) == len(set(calls_in))
        assert sum(1 for _, g in members if g == 1) <= MAX_JOBS
        assert sum(1 for _, g in members if g == 2) <= MAX_JOBS
        if any(g == 0 for _, g in members):
            assert len(members) == 1
    # dependencies: a call that conflicts with an earlier one starts after that one finished
    wins = [(_windows(a), _windows(b), _windows(c)) for _, a, b, _, c in calls]
    for j in range(len(calls)):
        for i in range(j):
            ra, rb, wc = wins[i]
            sa, sb, tc = wins[j]
            conflict = _overlap(wc, tc) or _overlap(wc, sa) or _overlap(wc, sb) or _overlap(tc, ra) or _overlap(tc, rb)
            if conflict:
                assert start[j] > finish[i], (i, j, finish[i], start[j])


def _calls(probs, shared_c=None, beta="cfg2_beta"):
    out = []
    for p in probs:
        va, vb, vc = p.views()
        if shared_c is not None:
            vc = shared_c[p.C.dtype].view(comp=p.comp)
        out.append((_alpha(p.label), va, vb, SCALARS[beta], vc))
    return out


def test_schedule_independent_mixed_calls(monkeypatch):
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    probs = [Problem(l, 130 + 7 * (i % 5), 260, 96 + 16 * (i % 3), seed=i) for i, l in enumerate(LABELS)]
    calls = _calls(probs)
    pieces, tiles = M.dual_schedule(calls, config({"gpu.numerics": "fast"}))
    _check_schedule(calls, pieces, tiles)
    # mixed batch: some launch runs both pipes
    units = {}
    for unit, _, _, _, grp in pieces:
        units.setdefault(unit, set()).add(grp)
    assert any({1, 2} <= g for g in units.values())


@pytest.mark.parametrize("beta", ["cfg2_beta", "zero"])
def test_schedule_dependency_chains(monkeypatch, beta):
    """One shared C per C datatype: four chains of 32 calls alternating FP32 / FP64."""
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    shared = {dt: HostMatrix(dt, 300, 420) for dt in range(4)}
    probs = [Problem(l, 300, 420, 200, seed=i) for i, l in enumerate(LABELS)]
    calls = _calls(probs, shared, beta)
    pieces, tiles = M.dual_schedule(calls, config({"gpu.numerics": "fast"}))
    _check_schedule(calls, pieces, tiles)


def test_schedule_splits_long_calls(monkeypatch):
    """A long FP64 call next to short FP32 calls is split into tile ranges."""
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    probs = [Problem("dddd", 2048, 2048, 512, seed=1)] + [Problem("ssss", 256, 256, 128, seed=2 + i) for i in range(4)]
    calls = _calls(probs)
    pieces, tiles = M.dual_schedule(calls, config({"gpu.numerics": "fast"}))
    _check_schedule(calls, pieces, tiles)
    assert sum(1 for p in pieces if p[1] == 0) >= 2


def test_schedule_many_calls_respects_caps(monkeypatch):
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    labels = ["dddd", "ssss", "zzzd", "cccs"]
    probs = [Problem(labels[i % 4], 20 + i % 7, 30, 16, seed=i) for i in range(400)]
    calls = _calls(probs)
    pieces, tiles = M.dual_schedule(calls, config({"gpu.numerics": "fast"}))
    _check_schedule(calls, pieces, tiles)
    assert max(p[0] for p in pieces) >= 2


def test_schedule_not_taken(monkeypatch):
    probs = [Problem(l, 40, 40, 40, seed=3) for l in ("dddd", "ssss")]
    calls = _calls(probs)
    monkeypatch.setenv("MDGEMM_DUAL", "0")
    assert M.dual_schedule(calls, config({"gpu.numerics": "fast"}))[0] == []
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    assert M.dual_schedule(calls, config({"gpu.numerics": "exact"}))[0] == []
    assert M.dual_schedule(calls[:1], config({"gpu.numerics": "fast"}))[0] == []
