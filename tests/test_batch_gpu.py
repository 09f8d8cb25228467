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


def _sub(buf: np.ndarray, dtype: int, ld: int, i0: int, j0: int, m: int, n: int, comp=None):
    """Column-major sub-view of a host buffer with leading dimension ld."""
    es = M.dtype_size(dtype)
    v = M.MatrixView.make(buf.ctypes.data + (i0 + j0 * ld) * es, m, n, 1, ld, dtype)
    return v.with_comp_prec(comp) if comp is not None else v


def _sequential_exact(seq, bufs, cfg):
    """Run (alpha, a, b, beta, c) recipes one after another with the oracle on copies of bufs."""
    ref = {k: b.copy() for k, b in bufs.items()}
    for alpha, a, b, beta, c in seq:
        O.orc_gemm(alpha, a(ref), b(ref), beta, c(ref), cfg)
    return ref


def test_batch_shared_host_operands_cross_pcie_once():
    """Every distinct host window is copied in once per batch and a host C goes back once."""
    cfg = config({"gpu.numerics": "exact"})
    A = HostMatrix(M.DT_Z, 48, 40).fill(O.orc_rng_state(1, ["a"]))
    B = HostMatrix(M.DT_D, 40, 36).fill(O.orc_rng_state(1, ["b"]))
    C = HostMatrix(M.DT_Z, 48, 36).fill(O.orc_rng_state(1, ["c"]))
    want = C.clone()
    for _ in range(5):
        O.orc_gemm(SCALARS["p7"], A.view(), B.view(), SCALARS["cfg2_beta"], want.view(), cfg)
    h0, d0 = M.staging_bytes()
    M.gemm_batch([(SCALARS["p7"], A.view(), B.view(), SCALARS["cfg2_beta"], C.view())] * 5, cfg)
    h1, d1 = M.staging_bytes()
    assert C.buf.tobytes() == want.buf.tobytes()
    assert h1 - h0 == A.buf.nbytes + B.buf.nbytes + C.buf.nbytes
    assert d1 - d0 == C.buf.nbytes


@pytest.mark.parametrize("budget_mb", [None, "0.02"])
def test_batch_overlapping_host_windows(monkeypatch, budget_mb):
    """Host operands that are sub-views of one buffer, overlapping each other and earlier residents
    (straddling, containing, contained), with and without forced evictions: the batch equals
    sequential gemm() calls bitwise (EXACT numerics)."""
    if budget_mb:
        monkeypatch.setenv("MDGEMM_RESIDENT_MB", budget_mb)
    cfg = config({"gpu.numerics": "exact"})
    ld = 64
    X = HostMatrix(M.DT_D, ld, 96).fill(O.orc_rng_state(2, ["x"]))
    Y = HostMatrix(M.DT_D, ld, 96).fill(O.orc_rng_state(2, ["y"]))
    Z = HostMatrix(M.DT_D, ld, 96).fill(O.orc_rng_state(2, ["z"]))
    bufs = {"X": X.buf, "Y": Y.buf, "Z": Z.buf}
    D = M.DT_D

    def sv(name, i0, j0, m, n):
        return lambda b: _sub(b[name], D, ld, i0, j0, m, n)
    seq = [
        (SCALARS["one"], sv("X", 0, 0, 32, 16), sv("Y", 0, 0, 16, 24), SCALARS["one"], sv("Y", 0, 40, 32, 24)),
        # A straddles the C window of call 0 (columns 30..50 of Y)
        (SCALARS["one"], sv("Y", 3, 30, 32, 20), sv("X", 0, 20, 20, 24), SCALARS["p3"], sv("X", 0, 60, 32, 24)),
        # A and B overlap each other inside one call
        (SCALARS["p7"], sv("X", 0, 10, 24, 30), sv("X", 5, 20, 30, 16), SCALARS["m3"], sv("Y", 8, 70, 24, 16)),
        # B contains everything written so far in Y
        (SCALARS["one"], sv("X", 0, 0, 40, 64), sv("Y", 0, 0, 64, 90), SCALARS["one"], sv("Z", 20, 0, 40, 90)),
        # C inside an earlier (read) window
        (SCALARS["one"], sv("Y", 0, 0, 16, 8), sv("Y", 16, 8, 8, 12), SCALARS["p3"], sv("X", 2, 2, 16, 12)),
    ]
    ref = _sequential_exact(seq, bufs, cfg)
    M.gemm_batch([(al, a(bufs), b(bufs), be, c(bufs)) for al, a, b, be, c in seq], cfg)
    for k in bufs:
        assert bufs[k].tobytes() == ref[k].tobytes(), k


def test_batch_eviction_chain(monkeypatch):
    """A dependency chain over more host data than the resident budget: evicted results go back to
    the host and are re-read correctly."""
    monkeypatch.setenv("MDGEMM_RESIDENT_MB", "0.1")
    cfg = config({"gpu.numerics": "fast"})
    mats = [HostMatrix(M.DT_D, 64, 64).fill(O.orc_rng_state(4, [str(i)])) for i in range(8)]
    ref = [m.clone() for m in mats]
    seq = [(i % 8, (i + 3) % 8, (i + 5) % 8) for i in range(20)]
    for a, b, c in seq:
        M.gemm(SCALARS["p7"], ref[a].view(), ref[b].view(), SCALARS["m3"], ref[c].view(), cfg)
    M.gemm_batch([(SCALARS["p7"], mats[a].view(), mats[b].view(), SCALARS["m3"], mats[c].view()) for a, b, c in seq],
                 cfg)
    for i in range(8):
        assert mats[i].buf.tobytes() == ref[i].buf.tobytes(), i


@pytest.mark.parametrize("label,shape", [("dssd", (1024, 1024, 1024)), ("zzzd", (300, 257, 333)),
                                         ("cdds", (130, 700, 2100)), ("sddd", (2048, 2048, 64)),
                                         ("szzs", (64, 64, 8))])
def test_lone_device_call_equals_the_batch_runner(label, shape):
    # gemm() on device operands takes the lone-call path (plan -> execute on the legacy stream); a
    # one-call gemm_batch goes through the batch runner.  Same kernels, same bits, same flop count.
    m, n, k = shape
    p = Problem(label, m, n, k, seed=17)
    cfg = config({"gpu.numerics": "fast"})
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    f1 = M.gemm(SCALARS["p7"], da, db, SCALARS["cfg2_beta"], dc, cfg)
    eA, eB, eC = p.device()
    ea, eb, ec = p.views(A=eA, B=eB, C=eC)
    f2 = M.gemm_batch([(SCALARS["p7"], ea, eb, SCALARS["cfg2_beta"], ec)], cfg)
    assert f1 == f2
    assert dC.bytes().tobytes() == eC.bytes().tobytes()
