"""Pack time of every label at one size inside lone calls (per-kind kernel times of the library), with the
bytes the packs move: which operand type / format combinations run below the HBM rate.

    python tools/exp_pack_labels.py [--size 4096] [--reps 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1901_06015_b200 as M
from oracle import abi as A

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
s = args.size
bufs = {}
for ch in "sdcz":
    dt = M.dtype_from_letter(ch)
    for role in "abc":
        t = torch.empty(s * s * M.dtype_size(dt), dtype=torch.uint8, device="cuda")
        v = M.MatrixView.make(t.data_ptr(), s, s, 1, s, dt)
        M.fill_uniform(v, M.Rng(0).split(role + ch).state)
        bufs[(role, ch)] = (t, v)
one = M.Scalar.real_value(1.0)
st = torch.cuda.current_stream()
rows = []
for l in A.all_labels():
    comp = M.SINGLE if l[3] == "s" else M.DOUBLE
    a, b, c = bufs[("a", l[1])][1], bufs[("b", l[2])][1], bufs[("c", l[0])][1].with_comp_prec(comp)
    M.gemm_async(one, a, b, one, c, stream=st)
    torch.cuda.synchronize()
    M.profile_begin()
    for _ in range(args.reps):
        M.gemm_async(one, a, b, one, c, stream=st)
    torch.cuda.synchronize()
    k = M.profile_end()
    p = k["pack"]
    us = p["ms"] / args.reps * 1e3
    gbs = p.get("bytes", 0) / args.reps / (us * 1e-6) / 1e9 if us else 0
    rows.append((l, A.case_id(l), p["launches"] / args.reps, us, gbs))
for l, cid, n, us, gbs in sorted(rows, key=lambda r: r[4]):
    print(f"{l} case {cid} launches {n:.0f} pack {us:7.1f} us {gbs:7.0f} GB/s")
tot_us = sum(r[3] for r in rows)
print(f"total {tot_us / 1e3:.2f} ms")
