"""Dual-pipe batch diagnostics: one sweep step (device operands) through gemm_batch with the
per-kernel profiling hook, dual on vs off; prints step time, per-kind device time and GFLOPS.
usage: python tools/exp_dual.py [sizes lo:hi:step]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06015_b200 as M  # noqa: E402

lo, hi, st = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256:4096:256").split(":"))
comp_filter = sys.argv[2] if len(sys.argv) > 2 else ""  # "d" / "s": only labels of that computation precision
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "0"]
sizes = list(range(lo, hi + 1, st))
labels = [l.str() for l in M.CaseLabel.all()]
if comp_filter:
    labels = [l for l in labels if l[3] == comp_filter]
S = M.Scalar
dev = torch.device("cuda:0")
ops = {}


def buf(role, dt, m, n):
    key = (role, dt, m, n)
    if key not in ops:
        t = torch.empty(max(m * n, 1) * M.dtype_size(dt), dtype=torch.uint8, device=dev)
        v = M.MatrixView.make(t.data_ptr(), m, n, 1, m, dt)
        M.fill_uniform(v, M.Rng(0).split(f"{role}{dt}{m}").state, 0)
        ops[key] = (t, v)
    return ops[key][1]


calls, flops = [], 0.0
for s in sizes:
    for lab in labels:
        dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
        cid = M.CaseLabel.parse(lab).case_id()
        al = S.complex_value(1.2, -0.7) if cid in (0, 7) else S.real_value(1.2)
        comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
        calls.append((al, buf("a", da, s, s), buf("b", db, s, s), S.complex_value(0.9, 0.3),
                      buf("c", dc, s, s).with_comp_prec(comp)))
        flops += M.flops_of_case(cid, s, s, s)
torch.cuda.synchronize()
for mode in modes:
    os.environ["MDGEMM_DUAL"] = mode
    M.gemm_batch(calls, sync=True)
    torch.cuda.synchronize()
    M.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    M.gemm_batch(calls, sync=False)
    h1 = time.perf_counter()
    e1.record()
    e1.synchronize()
    ks = M.profile_end()
    ms = e0.elapsed_time(e1)
    kk = {k: (v["launches"], round(v["ms"], 1), round(v["work"] / max(v["ms"], 1e-9) / 1e9, 1)) for k, v in ks.items() if v["launches"] or v["work"]}
    print(f"dual={mode} step {ms:8.1f} ms  {flops / ms / 1e9:8.0f} GFLOPS  enqueue {1e3 * (h1 - h0):7.1f} ms  {kk}", flush=True)
