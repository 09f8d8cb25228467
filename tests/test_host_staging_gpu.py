"""Operands in PAGEABLE host memory (numpy buffers, what a drop-in caller of
gemm() hands over) move through the library's pinned chunk ring
(csrc/host/hostcopy.cpp): 8 MiB slots, host threads filling / draining one
slot while the copy engine moves another.  Results must be bitwise those of
the same calls on device-resident operands: windows of several chunks with a
ragged last chunk, the lone-call path, the dual-pipe batch path (its pageable
results go back after the last launch) and mid-batch evictions (a pageable
write-back that must land before a later call re-reads the bytes)."""

import pytest
import torch

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import HostMatrix, Problem, SCALARS, config

pytestmark = pytest.mark.gpu

FAST = config({"gpu.numerics": "fast"})


def device_result(p: Problem, alpha, beta, cfg=FAST):
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(alpha, da, db, beta, dc, cfg)
    return dC.bytes()


@pytest.mark.parametrize("label,shape", [("zzzd", (1300, 1100, 900)), ("sddd", (2500, 2300, 300)),
                                         ("cdds", (1700, 900, 1111))])
def test_lone_call_multi_chunk_windows(label, shape):
    m, n, k = shape
    p = Problem(label, m, n, k, seed=5)
    want = device_result(p, SCALARS["cfg2_alpha_real"] if label != "zzzd" else SCALARS["cfg3_alpha"],
                         SCALARS["cfg2_beta"])
    h2d0, d2h0 = M.staging_bytes()
    host_c = p.C.clone()
    va, vb, vc = p.views(C=host_c)
    assert host_c.buf.nbytes > 8 << 20 and host_c.buf.nbytes % (8 << 20) != 0
    M.gemm(SCALARS["cfg2_alpha_real"] if label != "zzzd" else SCALARS["cfg3_alpha"], va, vb, SCALARS["cfg2_beta"], vc,
           FAST)
    assert host_c.buf.tobytes() == want.tobytes()
    h2d1, d2h1 = M.staging_bytes()
    assert h2d1 - h2d0 == p.A.buf.nbytes + p.B.buf.nbytes + p.C.buf.nbytes
    assert d2h1 - d2h0 == p.C.buf.nbytes


def test_exact_numerics_through_the_ring():
    # EXACT through pageable staging still equals the oracle byte for byte
    p = Problem("zczd", 300, 280, 40, seed=8)  # C 1.3 MB: takes the ring
    want = p.C.clone()
    va, vb, vw = p.views(C=want)
    O.orc_gemm(SCALARS["cfg3_alpha"], va, vb, SCALARS["cfg2_beta"], vw)
    got = p.C.clone()
    va, vb, vg = p.views(C=got)
    M.gemm(SCALARS["cfg3_alpha"], va, vb, SCALARS["cfg2_beta"], vg, config({"gpu.numerics": "exact"}))
    assert got.buf.tobytes() == want.buf.tobytes()


def test_dual_batch_pageable_results():
    # FP64 and FP32 calls in one batch (the dual-pipe path), every operand pageable, two calls per C
    labels = ["dddd", "ssss", "zzzd", "cccs", "dssd", "sdds"]
    probs = [Problem(l, 700, 650, 500, seed=20 + i) for i, l in enumerate(labels)]
    shared = {}
    for p in probs:
        shared.setdefault(p.C.dtype, p.C.clone())
    # reference: the same sequence on device copies
    dev_c = {dt: h.to_device() for dt, h in shared.items()}
    for p in probs + probs:
        dA, dB, _ = p.device()
        M.gemm(SCALARS["p7"], dA.view(conj=p.conj_a), dB.view(conj=p.conj_b), SCALARS["m3"],
               dev_c[p.C.dtype].view(comp=p.comp), FAST)
    torch.cuda.synchronize()
    calls = []
    for p in probs + probs:
        va, vb, _ = p.views()
        calls.append((SCALARS["p7"], va, vb, SCALARS["m3"], shared[p.C.dtype].view(comp=p.comp)))
    M.profile_begin()
    M.gemm_batch(calls, FAST)
    stats = M.profile_end()
    assert stats["dual_d"]["launches"] > 0
    for dt, h in shared.items():
        assert h.buf.tobytes() == dev_c[dt].bytes().tobytes(), dt


def test_eviction_writes_back_before_reread(monkeypatch):
    # windows of ~2.3 MB (above the direct-copy threshold) and a resident budget of about two of
    # them: results are evicted to pageable memory mid-batch and staged in again by later calls
    monkeypatch.setenv("MDGEMM_RESIDENT_MB", "5")
    monkeypatch.setenv("MDGEMM_DUAL", "0")
    n = 380
    mats = [HostMatrix(M.DT_Z, n, n).fill(O.orc_rng_state(6, [str(i)])) for i in range(6)]
    assert mats[0].buf.nbytes > 1 << 20
    ref = [m.to_device() for m in mats]
    seq = [(i % 6, (i + 2) % 6, (i + 3) % 6) for i in range(14)]
    for a, b, c in seq:
        M.gemm(SCALARS["p7"], ref[a].view(), ref[b].view(), SCALARS["m3"], ref[c].view(), FAST)
    M.gemm_batch([(SCALARS["p7"], mats[a].view(), mats[b].view(), SCALARS["m3"], mats[c].view()) for a, b, c in seq],
                 FAST)
    for i in range(6):
        assert mats[i].buf.tobytes() == ref[i].bytes().tobytes(), i


def test_pinned_host_operands_keep_the_async_path():
    # pinned (page-locked) host memory: plain async copies, same bytes
    p = Problem("dzzd", 600, 500, 400, seed=3)
    want = device_result(p, SCALARS["p7"], SCALARS["m3"])
    pin = {name: torch.from_numpy(getattr(p, name).buf.copy()).pin_memory() for name in "ABC"}
    va = M.MatrixView.make(pin["A"].data_ptr(), p.A.m, p.A.n, p.A.rs, p.A.cs, p.A.dtype)
    vb = M.MatrixView.make(pin["B"].data_ptr(), p.B.m, p.B.n, p.B.rs, p.B.cs, p.B.dtype)
    vc = M.MatrixView.make(pin["C"].data_ptr(), p.C.m, p.C.n, p.C.rs, p.C.cs, p.C.dtype)
    vc.comp_prec = p.comp
    M.gemm(SCALARS["p7"], va, vb, SCALARS["m3"], vc, FAST)
    assert pin["C"].numpy().tobytes() == want.tobytes()

