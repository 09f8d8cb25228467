#!/usr/bin/env python3
"""Predicted strong scaling of the cfg2 sweep's multi-GPU split, measured on ONE GPU.

bench.py's split of the sweep (chains: whole calls, the calls updating one C buffer stay on one
rank, no collective in the data path) gives every rank an independent batch, so rank r of a world of
N can be timed alone: this script builds rank r's operands and batch exactly as bench.py does under
torchrun (make_operands(world=N, rank=r)) and times its step, one simulated rank after another on
cuda:0.  Whole-job time at N ranks = max over ranks; efficiency = T(1) / (N * max_r T_r(N)).
No rank ever waits on another rank's kernels, so the simulation is exact up to NVLink-free effects
(there is no data-path collective in this mode).

usage: python tools/exp_chain_ranks.py [--worlds 1,2,4,8] [--steps 2] [--shard chains|columns]
"""
import argparse
import gc
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--shard", default="chains")
    ap.add_argument("--sizes", default="256:4096:256")
    ap.add_argument("--ranks", default="", help="only these simulated ranks (comma-separated)")
    a = ap.parse_args()
    import torch

    import bench
    import paper_1901_06015_b200 as M

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    args = argparse.Namespace(workload="sweep", labels="", size=0, sizes=a.sizes)
    _, items, dist_kind = bench.workload(args)
    cfg = M.Config.defaults().set("gpu.numerics", "fast")
    flush = torch.empty(bench.L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    total_flops = bench.useful_flops(items)
    out = {"shard": a.shard, "flops_per_step": total_flops, "worlds": {}}
    t1 = None
    for world in [int(w) for w in a.worlds.split(",")]:
        per_rank = []
        for rank in ([int(r) for r in a.ranks.split(",")] if a.ranks else range(world)):
            ops, shard, calls, call_info, a_bufs = bench.make_operands(M, items, "sweep", 0, dist_kind, dev, stream,
                                                                       world, rank, a.shard if world > 1 else "columns")
            ms = []
            for it in range(1 + a.steps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                M.gemm_batch(calls, cfg, stream=stream, sync=False)
                e1.record(stream)
                e1.synchronize()
                if it > 0:
                    ms.append(e0.elapsed_time(e1))
            fl = sum(f for _, f, _ in call_info)
            per_rank.append({"rank": rank, "calls": len(calls), "flops_share": fl / total_flops,
                             "ms": sum(ms) / len(ms)})
            del ops, calls
            gc.collect()
            torch.cuda.synchronize()
            M.trim_workspace() if hasattr(M, "trim_workspace") else None
            torch.cuda.empty_cache()
        tmax = max(r["ms"] for r in per_rank)
        if world == 1:
            t1 = tmax
        eff = (t1 / (world * tmax)) if t1 else None
        out["worlds"][world] = {"max_ms": tmax, "GFLOPS": total_flops / tmax / 1e6, "efficiency": eff,
                                "ranks": per_rank}
        print(f"world {world}: max {tmax:.1f} ms, {total_flops / tmax / 1e6:.0f} GFLOPS, efficiency {eff}",
              file=sys.stderr)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
