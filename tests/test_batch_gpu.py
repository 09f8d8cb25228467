"""gemm_batch(): a list of gemm() calls with host staging pipelined across
calls must equal calling gemm() on each element in order -- including calls
that update the same host C (read-after-write through the copy-out), calls
that read a previous call's C as their A, and mixed host/device operands."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import HostMatrix, Problem, SCALARS, config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_batch_equals_sequential_calls(numerics):
    cfg = config({"gpu.numerics": numerics})
    labels = ["zzzd", "dssd", "cdds", "szzs", "zczd", "sddd", "cccs", "dzdd"]
    # shared host C per C dtype: later calls depend on earlier calls' results
    shared_c = {dt: HostMatrix(dt, 40, 33).fill(O.orc_rng_state(9, ["c", dt])) for dt in range(4)}
    probs = [Problem(l, 40, 33, 50, seed=i) for i, l in enumerate(labels * 2)]
    ref_c = {dt: h.clone() for dt, h in shared_c.items()}
    # the sequential oracle replay (EXACT) / sequential device calls (FAST) as the reference
    for p in probs:
        va, vb, _ = p.views()
        vc = ref_c[p.C.dtype].view(comp=p.comp)
        if numerics == "exact":
            O.orc_gemm(SCALARS["p7"], va, vb, SCALARS["cfg2_beta"], vc, cfg)
        else:
            M.gemm(SCALARS["p7"], va, vb, SCALARS["cfg2_beta"], vc, cfg)
    calls = []
    for p in probs:
        va, vb, _ = p.views()
        calls.append((SCALARS["p7"], va, vb, SCALARS["cfg2_beta"], shared_c[p.C.dtype].view(comp=p.comp)))
    flops = M.gemm_batch(calls, cfg)
    assert flops > 0
    for dt in range(4):
        assert shared_c[dt].buf.tobytes() == ref_c[dt].buf.tobytes(), dt


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_device_batch_concurrency_keeps_order(numerics):
    """Device-resident calls: independent ones may run concurrently, but RAW
    (C feeds a later A), WAR (a later call overwrites an earlier call's B) and
    WAW (shared C) must keep the sequential result."""
    import torch
    cfg = config({"gpu.numerics": numerics})
    n = 96
    mats = {name: HostMatrix(M.DT_D, n, n).fill(O.orc_rng_state(3, [name])) for name in "PQRSTUVW"}
    seq = [("P", "Q", "R"), ("S", "T", "U"), ("R", "Q", "V"),  # RAW: R written by 0, read by 2
           ("P", "T", "Q"),                                   # WAR: Q read by 0 and 2, written here
           ("S", "P", "R"), ("U", "V", "W"), ("P", "Q", "W"), ("W", "S", "T")]
    # sequential reference with the oracle (EXACT) or one gemm per call (FAST)
    ref = {k: v.clone() for k, v in mats.items()}
    for a, b, c in seq:
        if numerics == "exact":
            O.orc_gemm(SCALARS["p7"], ref[a].view(), ref[b].view(), SCALARS["m3"], ref[c].view(), cfg)
        else:
            M.gemm(SCALARS["p7"], ref[a].view(), ref[b].view(), SCALARS["m3"], ref[c].view(), cfg)
    dev = {k: v.to_device() for k, v in mats.items()}
    M.gemm_batch([(SCALARS["p7"], dev[a].view(), dev[b].view(), SCALARS["m3"], dev[c].view()) for a, b, c in seq],
                 cfg)
    torch.cuda.synchronize()
    for k in mats:
        assert dev[k].bytes().tobytes() == ref[k].buf.tobytes(), k


def test_batch_output_feeds_next_input():
    # call 2 reads call 1's C as its A (host RAW through the copy-out)
    A1 = HostMatrix(M.DT_D, 64, 64).fill(1)
    B1 = HostMatrix(M.DT_D, 64, 64).fill(2)
    C1 = HostMatrix(M.DT_D, 64, 64).fill(3)
    B2 = HostMatrix(M.DT_D, 64, 64).fill(4)
    C2 = HostMatrix(M.DT_D, 64, 64).fill(5)
    wantC1, wantC2 = C1.clone(), C2.clone()
    cfg = config({"gpu.numerics": "exact"})
    O.orc_gemm(SCALARS["one"], A1.view(), B1.view(), SCALARS["one"], wantC1.view(), cfg)
    O.orc_gemm(SCALARS["one"], wantC1.view(), B2.view(), SCALARS["p3"], wantC2.view(), cfg)
    M.gemm_batch([(SCALARS["one"], A1.view(), B1.view(), SCALARS["one"], C1.view()),
                  (SCALARS["one"], C1.view(), B2.view(), SCALARS["p3"], C2.view())], cfg)
    assert C1.buf.tobytes() == wantC1.buf.tobytes()
    assert C2.buf.tobytes() == wantC2.buf.tobytes()


def test_batch_mixed_host_and_device_operands():
    p = Problem("zzzd", 70, 65, 80)
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    cfg = config({"gpu.numerics": "exact"})
    O.orc_gemm(SCALARS["cfg3_alpha"], va, vb, SCALARS["one"], vw, cfg)
    dA = p.A.to_device()
    got = p.C.clone()
    _, vb_h, vc_h = p.views(C=got)
    M.gemm_batch([(SCALARS["cfg3_alpha"], dA.view(), vb_h, SCALARS["one"], vc_h)], cfg)
    assert got.buf.tobytes() == want.buf.tobytes()


def test_batch_errors_before_device_work():
    p = Problem("zdzd", 8, 8, 8)
    q = Problem("dddd", 8, 8, 8)
    before = q.C.buf.copy()
    qa, qb, qc = q.views()
    pa, pb, pc = p.views()
    with pytest.raises(M.ScalarPolicyError):
        M.gemm_batch([(SCALARS["one"], qa, qb, SCALARS["one"], qc), (SCALARS["c55"], pa, pb, SCALARS["one"], pc)])
    assert np.array_equal(before, q.C.buf)  # the valid first call did not run either
