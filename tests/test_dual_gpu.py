"""The dual-pipe kernel (gemm_dual.cu) behind gemm_batch: FP64 DMMA jobs and
FP32 FFMA2 jobs of one batch share every SM.  Its results must be BITWISE the
results of calling gemm() on each call in order (same k order, same DMMA /
FFMA2 rounding, same accumulate_element combine), for every label, C layout,
edge tile, dependency chain, host or device operands."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import HostMatrix, Problem, SCALARS, config

pytestmark = pytest.mark.gpu

LABELS = [l.str() for l in M.CaseLabel.all()]
SHAPES = [(70, 65, 80), (129, 200, 33), (64, 128, 16), (5, 3, 1), (200, 129, 257), (1, 300, 7)]


def _alpha(label):
    cid = M.CaseLabel.parse(label).case_id()
    return SCALARS["cfg2_alpha"] if cid in (0, 7) else SCALARS["p7"]


def _batch_with_profile(calls, cfg):
    M.profile_begin()
    M.gemm_batch(calls, cfg)
    return M.profile_end()


@pytest.mark.parametrize("c_kind,dynamic", [("col", "0"), ("row", "0"), ("col", "1")])
def test_dual_all_labels_equal_single_calls(monkeypatch, c_kind, dynamic):
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    monkeypatch.setenv("MDGEMM_DUAL_DYNAMIC", dynamic)  # static tile order, or the atomic-counter one
    cfg = config({"gpu.numerics": "fast"})
    probs = [Problem(l, *SHAPES[i % len(SHAPES)], c_kind=c_kind, seed=7 + i, trans_a=(i % 5 == 3))
             for i, l in enumerate(LABELS)]
    want = []
    for p in probs:
        c = p.C.clone()
        va, vb, vc = p.views(C=c)
        M.gemm(_alpha(p.label), va, vb, SCALARS["cfg2_beta"], vc, cfg)
        want.append(c)
    calls = []
    for p in probs:
        va, vb, vc = p.views()
        calls.append((_alpha(p.label), va, vb, SCALARS["cfg2_beta"], vc))
    ks = _batch_with_profile(calls, cfg)
    assert ks["dual_d"]["launches"] > 0, ks
    for p, w in zip(probs, want):
        assert p.C.buf.tobytes() == w.buf.tobytes(), p.label


@pytest.mark.parametrize("beta", ["cfg2_beta", "one", "zero"])
def test_dual_chains_equal_sequential_calls(monkeypatch, beta):
    """Calls sharing one host C per C datatype (dependency chains that alternate
    computation precisions): the list schedule must keep every chain's order."""
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = config({"gpu.numerics": "fast"})
    shared = {dt: HostMatrix(dt, 96, 140).fill(O.orc_rng_state(11, ["c", dt])) for dt in range(4)}
    ref = {dt: h.clone() for dt, h in shared.items()}
    probs = [Problem(l, 96, 140, 72, seed=i) for i, l in enumerate(LABELS)]
    for p in probs:
        va, vb, _ = p.views()
        M.gemm(_alpha(p.label), va, vb, SCALARS[beta], ref[p.C.dtype].view(comp=p.comp), cfg)
    calls = []
    for p in probs:
        va, vb, _ = p.views()
        calls.append((_alpha(p.label), va, vb, SCALARS[beta], shared[p.C.dtype].view(comp=p.comp)))
    ks = _batch_with_profile(calls, cfg)
    assert ks["dual_d"]["launches"] > 0 and ks["dual_f"]["work"] > 0, ks
    for dt in range(4):
        assert shared[dt].buf.tobytes() == ref[dt].buf.tobytes(), dt


def test_dual_device_operands_and_raw_chain(monkeypatch):
    """Device operands, a later call reading an earlier call's C as its A
    (the pack must wait for that launch), k = 0 and empty calls in between."""
    import torch
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = config({"gpu.numerics": "fast"})
    n = 136
    mats = {name: HostMatrix(M.DT_D if name < "N" else M.DT_S, n, n).fill(O.orc_rng_state(5, [name]))
            for name in ["A", "B", "C", "D", "E", "P", "Q", "R", "S"]}
    seq = [("A", "B", "C", 136), ("P", "Q", "R", 136), ("C", "B", "D", 136),  # D reads C (RAW through A)
           ("R", "Q", "S", 136), ("A", "D", "E", 0), ("P", "S", "R", 136), ("E", "B", "C", 136)]
    ref = {k: v.clone() for k, v in mats.items()}

    def view(store, name, k, role):
        h = store[name]
        v = h.view()
        if role == "a":
            v = M.MatrixView.make(v.base, n, k, 1, n, v.dtype)
        elif role == "b":
            v = M.MatrixView.make(v.base, k, n, 1, max(k, 1), v.dtype)
        return v
    for a, b, c, k in seq:
        M.gemm(SCALARS["p7"], view(ref, a, k, "a"), view(ref, b, k, "b"), SCALARS["m3"], ref[c].view(), cfg)
    dev = {k: v.to_device() for k, v in mats.items()}
    calls = [(SCALARS["p7"], view(dev, a, k, "a"), view(dev, b, k, "b"), SCALARS["m3"], dev[c].view())
             for a, b, c, k in seq]
    ks = _batch_with_profile(calls, cfg)
    torch.cuda.synchronize()
    assert ks["dual_d"]["launches"] > 0, ks
    for k in mats:
        assert dev[k].bytes().tobytes() == ref[k].buf.tobytes(), k


def test_dual_off_and_exact_take_the_stream_scheduler(monkeypatch):
    probs = [Problem(l, 40, 40, 40, seed=3) for l in ("dddd", "ssss", "zzzd", "cccs")]
    for env, numerics in (("0", "fast"), ("1", "exact")):
        monkeypatch.setenv("MDGEMM_DUAL", env)
        calls = [(SCALARS["p7"], *p.views()[:2], SCALARS["one"], p.views()[2]) for p in probs]
        ks = _batch_with_profile(calls, config({"gpu.numerics": numerics}))
        assert ks["dual_d"]["launches"] == 0, (env, numerics)


@pytest.mark.parametrize("variant", ["gen_c", "conj", "trans_b", "k_ragged"])
def test_dual_variants_equal_single_calls(monkeypatch, variant):
    """General-stride C (gaps between elements), conjugated operands, transposed B and inner
    dimensions that are not multiples of the 16-deep k-block, every label."""
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = config({"gpu.numerics": "fast"})
    kw = {"gen_c": dict(c_kind="gen"), "conj": dict(conj_a=True, conj_b=True), "trans_b": dict(trans_b=True),
          "k_ragged": {}}[variant]
    shape = (37, 41, 23) if variant == "k_ragged" else (72, 136, 48)
    probs = [Problem(l, *shape, seed=100 + i, **kw) for i, l in enumerate(LABELS)]
    want = []
    for p in probs:
        c = p.C.clone()
        va, vb, vc = p.views(C=c)
        M.gemm(_alpha(p.label), va, vb, SCALARS["m3"], vc, cfg)
        want.append(c)
    calls = [(_alpha(p.label), *p.views()[:2], SCALARS["m3"], p.views()[2]) for p in probs]
    ks = _batch_with_profile(calls, cfg)
    assert ks["dual_d"]["launches"] > 0, ks
    for p, w in zip(probs, want):
        assert p.C.buf.tobytes() == w.buf.tobytes(), p.label


def test_dual_within_fast_tolerance_of_oracle(monkeypatch):
    """Independent of the classic kernels: dual results against the CPU oracle (the reference's
    per-element criterion and the north-star relative Frobenius bound, as in test_gemm_fast_gpu)."""
    from tests.test_gemm_fast_gpu import frob_bound
    from tests.helpers import rel_frobenius
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = config({"gpu.numerics": "fast"})
    probs = [Problem(l, 33, 70, 129, seed=300 + i) for i, l in enumerate(LABELS[::3])]
    orig = [p.C.clone() for p in probs]
    want = []
    for p in probs:
        c = p.C.clone()
        va, vb, vc = p.views(C=c)
        O.orc_gemm(_alpha(p.label), va, vb, SCALARS["cfg2_beta"], vc, config({}))
        want.append(c)
    calls = [(_alpha(p.label), *p.views()[:2], SCALARS["cfg2_beta"], p.views()[2]) for p in probs]
    ks = _batch_with_profile(calls, cfg)
    assert ks["dual_d"]["launches"] > 0, ks
    for p, w, o in zip(probs, want, orig):
        va, vb, _ = p.views()
        viol = O.orc_violation(_alpha(p.label), va, vb, SCALARS["cfg2_beta"], o.view(comp=p.comp),
                               p.C.view(comp=p.comp), p.comp)
        assert viol <= 1.0, (p.label, viol)
        err = rel_frobenius(p.C.values(), w.values())
        assert err <= frob_bound(p.label, p.k), (p.label, err)


def test_dual_split_tile_ranges(monkeypatch):
    """A long FP64 call next to short FP32 calls is split into tile ranges over several launches
    (each launch packs its operands again); the pieces must assemble the single-call result, and
    calls that depend on the split one (its C read as A) must see all of it."""
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = config({"gpu.numerics": "fast"})
    big = Problem("dddd", 640, 520, 384, seed=1)
    small = [Problem("cccs" if i % 2 else "ssss", 96, 80, 64, seed=10 + i) for i in range(6)]
    # a dependent call: reads big's C (640 x 520) as its A
    dep_b = HostMatrix(M.DT_D, 520, 136).fill(O.orc_rng_state(77, ["b"]))
    dep_c = HostMatrix(M.DT_D, 640, 136).fill(O.orc_rng_state(77, ["c"]))
    ref_big, ref_dep = big.C.clone(), dep_c.clone()
    va, vb, _ = big.views()
    M.gemm(SCALARS["p7"], va, vb, SCALARS["m3"], ref_big.view(), cfg)
    M.gemm(SCALARS["one"], ref_big.view(), dep_b.view(), SCALARS["p3"], ref_dep.view(), cfg)
    ref_small = []
    for p in small:
        c = p.C.clone()
        sa, sb, sc = p.views(C=c)
        M.gemm(SCALARS["p7"], sa, sb, SCALARS["m3"], sc, cfg)
        ref_small.append(c)
    calls = [(SCALARS["p7"], *big.views()[:2], SCALARS["m3"], big.views()[2])]
    calls += [(SCALARS["p7"], *p.views()[:2], SCALARS["m3"], p.views()[2]) for p in small]
    calls.append((SCALARS["one"], big.C.view(), dep_b.view(), SCALARS["p3"], dep_c.view()))
    ks = _batch_with_profile(calls, cfg)
    assert ks["dual_d"]["launches"] >= 2, ks
    assert big.C.buf.tobytes() == ref_big.buf.tobytes()
    assert dep_c.buf.tobytes() == ref_dep.buf.tobytes()
    for p, w in zip(small, ref_small):
        assert p.C.buf.tobytes() == w.buf.tobytes(), p.label


def test_dual_many_small_calls(monkeypatch):
    """More independent calls than one launch's job lists hold (DUAL_MAX_JOBS per group): the
    schedule spreads them over several launches; every call bitwise equal to its single call."""
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = config({"gpu.numerics": "fast"})
    labels = ["dddd", "ssss", "zzzd", "cccs", "dssd", "sdds"]
    probs = [Problem(labels[i % len(labels)], 17 + i % 23, 9 + i % 31, 5 + i % 40, seed=1000 + i) for i in range(300)]
    want = []
    for p in probs:
        c = p.C.clone()
        va, vb, vc = p.views(C=c)
        M.gemm(_alpha(p.label), va, vb, SCALARS["cfg2_beta"], vc, cfg)
        want.append(c)
    calls = [(_alpha(p.label), *p.views()[:2], SCALARS["cfg2_beta"], p.views()[2]) for p in probs]
    ks = _batch_with_profile(calls, cfg)
    assert ks["dual_d"]["launches"] >= 2, ks
    for p, w in zip(probs, want):
        assert p.C.buf.tobytes() == w.buf.tobytes(), p.label


@pytest.mark.parametrize("shape", [(200, 1100, 96), (136, 1024, 40)])
def test_long_chain_split_into_column_panels_equals_sequential_calls(monkeypatch, tmp_path, shape):
    """A batch that is one long dependency chain (32 calls updating one device C, alternating
    computation precisions) next to a short one: the calls on the long path are cut into column
    panels (staging.cpp: split_long_chains) so that FP64 and FP32 panels of neighbouring calls pair
    up.  Bits and FlopCounter must be those of the calls run one by one; a row-stored C is not cut."""
    import re

    import torch
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    log = tmp_path / "dual.log"
    monkeypatch.setenv("MDGEMM_DUAL_LOG", str(log))
    cfg = config({"gpu.numerics": "fast"})
    m, n, k = shape
    long_labels = [l for l in LABELS if l[0] == "z"]
    short_labels = [l for l in LABELS if l[0] == "s"][:6]
    for c_kind, expect_split in (("col", True), ("row", False)):
        log.write_text("")
        probs = [Problem(l, m, n, k, seed=40 + i, trans_b=(i % 7 == 2), c_kind=c_kind) for i, l in enumerate(long_labels)]
        probs += [Problem(l, 70, 130, 33, seed=90 + i) for i, l in enumerate(short_labels)]
        shared = {"z": probs[0].C.clone(), "s": probs[len(long_labels)].C.clone()}
        ref = {key: h.clone() for key, h in shared.items()}
        want_flops = 0
        for p in probs:
            va, vb, _ = p.views()
            want_flops += M.gemm(_alpha(p.label), va, vb, SCALARS["cfg2_beta"], ref[p.label[0]].view(comp=p.comp), cfg)
        dev_c = {key: h.to_device() for key, h in shared.items()}
        keep, calls = [], []
        for p in probs:
            dA, dB = p.A.to_device(), p.B.to_device()
            keep += [dA, dB]
            va = dA.tview(conj=p.conj_a) if p.trans_a else dA.view(conj=p.conj_a)
            vb = dB.tview(conj=p.conj_b) if p.trans_b else dB.view(conj=p.conj_b)
            calls.append((_alpha(p.label), va, vb, SCALARS["cfg2_beta"], dev_c[p.label[0]].view(comp=p.comp)))
        got_flops = M.gemm_batch(calls, cfg)
        torch.cuda.synchronize()
        for key in shared:
            assert dev_c[key].bytes().tobytes() == ref[key].buf.tobytes(), (c_kind, key)
        assert got_flops == want_flops, c_kind
        sizes = [int(x) for x in re.findall(r"batch (\d+) calls", log.read_text())]
        assert sizes and (max(sizes) > len(calls)) == expect_split, (c_kind, sizes, len(calls))
