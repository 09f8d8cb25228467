"""Parity of the bench's own timed step: bench.py's exact gemm_batch (the
dual-pipe kernel, C buffers shared per (dtype, size) so that the calls of a
step form dependency chains of alternating FP64 / FP32 computation, the sweep's
scalars), on the sweep's largest slice (3584, 4096) and its smallest (256, 512).

Every C buffer of the step is checked on sampled rows x columns (edges
included) against the oracle replaying the buffer's chain of calls in order on
that block: for the reference a row/column block of C with the full inner
dimension is bitwise the same computation as the whole call, so
the replay is the reference's own result for those elements.

Bound: the north-star bound of every call of the chain, propagated.  With
C_t = beta C_{t-1} + alpha A_t B_t and a per-call FAST error delta_t, the error
of the final C is sum_t beta^(T-t) delta_t, so (|beta| < 1)
    ||C_gpu - C_ref||_F <= sum_t (4 k eps_comp(t) [+ eps_out]) ||C_t||_F
taking each call's bound relative to its own (reference) output."""
import numpy as np
import pytest

import bench
import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import HostMatrix, config, frob_bound, rel_frobenius
from tests.test_baseline_scale_gpu import TORCH_T

pytestmark = pytest.mark.gpu


def sweep_items(sizes):
    S = M.Scalar
    items = []
    for s in sizes:
        for lab in (l.str() for l in M.CaseLabel.all()):
            cid = M.CaseLabel.parse(lab).case_id()
            alpha = S.complex_value(1.2, -0.7) if cid in (0, 7) else S.real_value(1.2)
            items.append((lab, s, s, s, alpha, S.complex_value(0.9, 0.3)))
    return items


def block(t, dtype, m, n, rows, cols) -> HostMatrix:
    import torch
    e = t.view(getattr(torch, TORCH_T[dtype])).view(n, m)  # [j, i]
    r = torch.as_tensor(rows, device=t.device)
    c = torch.as_tensor(cols, device=t.device)
    sub = e.index_select(0, c).index_select(1, r).T.contiguous().cpu().numpy()
    h = HostMatrix(dtype, len(rows), len(cols))
    h.values()[:, :] = sub
    return h


@pytest.mark.parametrize("sizes", [(3584, 4096), (256, 512)])
def test_bench_step_batch_parity(sizes):
    import torch
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    items = sweep_items(sizes)
    ops, shard, calls, call_info, _ = bench.make_operands(M, items, "sweep", 0, "uniform", dev, stream)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    samp = {s: (sorted({0, s - 1} | set(int(x) for x in rng.integers(0, s, 6))),
                sorted({0, s - 1} | set(int(x) for x in rng.integers(0, s, 6)))) for s in sizes}
    # host copies of what every call reads on the sampled block, before the step
    a_rows, b_cols, c0 = {}, {}, {}
    for (role, dt, shape), (t, _) in ops.items():
        m, n = shape
        if role == "a":
            a_rows[(dt, shape)] = block(t, dt, m, n, samp[m][0], list(range(n)))
        elif role == "b":
            b_cols[(dt, shape)] = block(t, dt, m, n, list(range(m)), samp[n][1])
        else:
            c0[(dt, shape)] = block(t, dt, m, n, *samp[m])
    # the bench's step: one gemm_batch on the timed stream
    M.gemm_batch(calls, config({"gpu.numerics": "fast"}), stream=stream, sync=False)
    torch.cuda.synchronize()
    # oracle: replay each C buffer's chain in call order on its block
    want = {key: c.clone() for key, c in c0.items()}
    bound_abs = {key: 0.0 for key in c0}
    for lab, m, n, k, al, be in items:
        dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
        comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
        key = (dc, (m, n))
        cw = want[key]
        O.orc_gemm(al, a_rows[(da, (m, k))].view(), b_cols[(db, (k, n))].view(), be, cw.view(comp=comp))
        bound_abs[key] += frob_bound(lab, k) * float(np.linalg.norm(cw.values().astype(np.complex128)))
    checked = 0
    for (dt, (m, n)), cw in want.items():
        t = ops[("c", dt, (m, n))][0]
        got = block(t, dt, m, n, *samp[m])
        err = rel_frobenius(got.values(), cw.values())
        bound = bound_abs[(dt, (m, n))] / float(np.linalg.norm(cw.values().astype(np.complex128)))
        assert err <= bound, (M.dtype_letter(dt), m, err, bound)
        checked += 1
    assert checked == 4 * len(sizes)  # one C buffer per C dtype and size
