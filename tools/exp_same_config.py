"""The reference arm's sample (128 labels at m=n=k=512, or --size) on one GPU:
device-resident gemm_batch with the library's per-kind kernel times, and the
per-call pageable-host gemm() e2e rate (host wall clock).

    python tools/exp_same_config.py [--size 512] [--steps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_06015_b200 as M
from oracle import abi as A

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--labels", default="")
args = ap.parse_args()
s = args.size
labels = [l for l in args.labels.split(",") if l] or A.all_labels()
cfg = M.Config.defaults()
dev_ops, host_ops, keep = [], [], []
flops = 0
for l in labels:
    cid = A.case_id(l)
    al = M.Scalar.complex_value(1.2, -0.7) if cid in (0, 7) else M.Scalar.real_value(1.2)
    be = M.Scalar.complex_value(0.9, 0.3)
    flops += A.flops_of_case(cid, s, s, s)
    comp = M.SINGLE if l[3] == "s" else M.DOUBLE
    trip, hs = [], []
    for role, ch in zip("abc", (l[1], l[2], l[0])):
        dt = M.dtype_from_letter(ch)
        t = torch.empty(s * s * M.dtype_size(dt), dtype=torch.uint8, device="cuda")
        v = M.MatrixView.make(t.data_ptr(), s, s, 1, s, dt)
        M.fill_uniform(v, M.Rng(0).split(f"x/{l}/{role}").state)
        h = np.empty(t.numel(), np.uint8)
        torch.cuda.synchronize()
        h[:] = t.cpu().numpy()
        hv = M.MatrixView.from_buffer_copy(v)
        hv.base = h.ctypes.data
        trip.append(v)
        hs.append(hv)
        keep += [t, h]
    dev_ops.append((al, trip[0], trip[1], be, trip[2].with_comp_prec(comp)))
    host_ops.append((al, hs[0], hs[1], be, hs[2].with_comp_prec(comp)))
torch.cuda.synchronize()
M.gemm_batch(dev_ops, cfg)
for _ in range(2):
    torch.cuda.synchronize()
    M.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    M.gemm_batch(dev_ops, cfg, sync=False)
    e1.record()
    e1.synchronize()
    st = M.profile_end()
    ms = e0.elapsed_time(e1)
print(f"device-resident batch: {ms:.3f} ms  {flops / ms / 1e6:.0f} GFLOPS")
for k, v in st.items():
    if v["launches"]:
        print(f"   {k:10s} launches {v['launches']:5d}  ms {v['ms']:.3f}")
for al, a, b, be, c in host_ops:
    M.gemm(al, a, b, be, c, cfg)
s0 = M.staging_bytes()
t0 = time.perf_counter()
for _ in range(args.steps):
    for al, a, b, be, c in host_ops:
        M.gemm(al, a, b, be, c, cfg)
el = time.perf_counter() - t0
s1 = M.staging_bytes()
mb = (s1[0] - s0[0] + s1[1] - s0[1]) / args.steps / 1e6
print(f"per-call pageable gemm(): {el / args.steps * 1e3:.1f} ms/step {flops * args.steps / el / 1e9:.0f} GFLOPS, "
      f"{mb:.0f} MB moved per step = {mb / (el / args.steps) / 1e3:.1f} GB/s")
