"""A lone device-resident gemm() (BASELINE cfg1 by default): CUDA-event time
per call and the library's per-kind kernel times.

    python tools/exp_lone.py [--label dssd] [--m 1024 --n 1024 --k 1024] [--reps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1901_06015_b200 as M
from oracle import abi as A

ap = argparse.ArgumentParser()
ap.add_argument("--label", default="dssd")
ap.add_argument("--m", type=int, default=1024)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--k", type=int, default=1024)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
l, m, n, k = args.label, args.m, args.n, args.k
views = []
keep = []
for role, ch, (r, c) in (("a", l[1], (m, k)), ("b", l[2], (k, n)), ("c", l[0], (m, n))):
    dt = M.dtype_from_letter(ch)
    t = torch.empty(r * c * M.dtype_size(dt), dtype=torch.uint8, device="cuda")
    v = M.MatrixView.make(t.data_ptr(), r, c, 1, r, dt)
    M.fill_uniform(v, M.Rng(0).split(role).state)
    views.append(v)
    keep.append(t)
comp = M.SINGLE if l[3] == "s" else M.DOUBLE
one = M.Scalar.real_value(1.0)
flops = A.flops_of_case(A.case_id(l), m, n, k)
s = torch.cuda.current_stream()
for _ in range(3):
    M.gemm_async(one, views[0], views[1], one, views[2].with_comp_prec(comp), stream=s)
torch.cuda.synchronize()
M.profile_begin()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    M.gemm_async(one, views[0], views[1], one, views[2].with_comp_prec(comp), stream=s)
e1.record()
e1.synchronize()
st = M.profile_end()
ms = e0.elapsed_time(e1) / args.reps
print(f"{l} {m}x{n}x{k}: {ms * 1e3:.1f} us/call  {flops / ms / 1e6:.0f} GFLOPS")
for kind, v in st.items():
    if v["launches"]:
        print(f"   {kind:12s} {v['launches'] / args.reps:5.1f} launches/call  {v['ms'] / args.reps * 1e3:7.1f} us/call")
