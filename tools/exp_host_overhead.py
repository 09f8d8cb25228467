"""Host cost of one synchronous gemm() on device operands (what a drop-in
caller looping over small problems pays per call): wall clock per call vs the
device time of the same call (CUDA events around gemm_async).

    python tools/exp_host_overhead.py [--labels dddd,zzzd,dssd] [--sizes 64,256,1024]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1901_06015_b200 as M

ap = argparse.ArgumentParser()
ap.add_argument("--labels", default="dddd,zzzd,dssd,cccs")
ap.add_argument("--sizes", default="64,256,1024")
ap.add_argument("--reps", type=int, default=200)
args = ap.parse_args()
cfg = M.Config.defaults()
for l in args.labels.split(","):
    for s in (int(x) for x in args.sizes.split(",")):
        keep, views = [], []
        for role, ch in zip("abc", (l[1], l[2], l[0])):
            dt = M.dtype_from_letter(ch)
            t = torch.empty(s * s * M.dtype_size(dt), dtype=torch.uint8, device="cuda")
            v = M.MatrixView.make(t.data_ptr(), s, s, 1, s, dt)
            M.fill_uniform(v, M.Rng(1).split(role).state)
            keep.append(t)
            views.append(v)
        comp = M.SINGLE if l[3] == "s" else M.DOUBLE
        a, b, c = views[0], views[1], views[2].with_comp_prec(comp)
        one = M.Scalar.real_value(1.0)
        for _ in range(10):
            M.gemm(one, a, b, one, c, cfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            M.gemm(one, a, b, one, c, cfg)
        host_us = (time.perf_counter() - t0) / args.reps * 1e6
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            M.gemm_async(one, a, b, one, c, cfg, st)
        e1.record(st)
        e1.synchronize()
        dev_us = e0.elapsed_time(e1) / args.reps * 1e3
        print(f"{l} {s:5d}: gemm() {host_us:8.1f} us/call   device (async stream) {dev_us:8.1f} us/call")
