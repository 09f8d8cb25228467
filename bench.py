#!/usr/bin/env python3
"""bench.py -- throughput of the B200 mixed-datatype gemm (arXiv 1901.06015).

Metric (BASELINE.json): effective GFLOPS = sum of flops_of_case(label, m, n, k)
(2/4/8 mnk, dispatch.cpp:35-54) / time, and its fraction of the measured
FP64-DMMA / FP32-FFMA peak.

Default workload = BASELINE configs[1], the full 128-label sweep m=n=k =
256, 512, ..., 4096: one step runs all 128 cabx labels at all 16 sizes (2,048
gemm calls, issued as one gemm_batch) with the sweep's scalars (alpha =
1.2-0.7i for cases 0 and 3, real 1.2 for the six cases that reject a complex
alpha; beta = 0.9+0.3i), A/B/C column-major, entries uniform[-1,1) from the
reference's splitmix64 Rng (generated on the device).  Other BASELINE configs
are available with --workload (cfg5 draws normal(0,1) entries by Box-Muller
over the same Rng, mdg_fill_normal).

Multi-GPU (torchrun): C and B are split into column panels per rank
(mdg_shard_columns), A is broadcast from rank 0 over NCCL inside every step;
no reduction.  Strong scaling (fixed total problem).

Arms:
  --impl b200       (default) this framework, device-resident operands
                    (value) and through the public gemm() with pinned host
                    buffers, H2D + D2H inside the timed region (e2e).
  --impl reference  the reference CPU engine (oracle/_ref, compiled from the
                    reference's own sources) on the host cores, rank 0 only,
                    on a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "effective GFLOPS and % of FP64/FP32 peak per mixed-datatype gemm case, 1/2/4/8 GPU"
PEAKS_FILE = os.path.join(ROOT, "profiles", "peaks_r01.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
L2_FLUSH_BYTES = 512 << 20


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="sweep",
                    choices=["sweep", "cfg1", "cfg3", "cfg4-cdds", "cfg4-szzs", "cfg4-zczd",
                             "cfg5-k64", "cfg5-k256", "cfg5-k1024"])
    ap.add_argument("--size", type=int, default=0, help="run the sweep at this single size m=n=k")
    ap.add_argument("--sizes", default="256:4096:256", help="sweep sizes lo:hi:step (BASELINE configs[1])")
    ap.add_argument("--labels", default="", help="comma-separated subset of labels (sweep)")
    ap.add_argument("--numerics", choices=["fast", "exact"], default="fast")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", choices=["auto", "columns", "chains"], default="auto",
                    help="multi-GPU split: C/B column panels of every call with A broadcast (columns), or whole "
                         "calls grouped by the C buffer they update (chains: dependency chains stay on one rank, "
                         "no collective); auto = chains for the cfg2 sweep, columns otherwise")
    ap.add_argument("--no-serial", action="store_true",
                    help="skip the serialized per-call pass (per-case rates, classic-kernel rooflines); "
                         "for ncu launch lists of the batched step alone")
    ap.add_argument("--cpu-size", type=int, default=512, help="sample size of the CPU baseline")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


# ------------------------------------------------------------------ workloads
def workload(args, S=None):
    """(description, [(label, m, n, k, alpha, beta)], distribution).  S: the Scalar struct class the
    items are built with (the product's by default; the reference arm passes oracle.abi.Scalar so that
    it never loads the product library)."""
    from oracle import abi as A
    if S is None:
        import paper_1901_06015_b200 as M
        S = M.Scalar
    if args.workload == "sweep":
        labels = A.all_labels()
        if args.labels:
            labels = [l for l in args.labels.split(",") if l]
        if args.size:
            sizes = [args.size]
        else:
            lo, hi, st = (int(x) for x in args.sizes.split(":"))
            sizes = list(range(lo, hi + 1, st))
        items = []
        for s in sizes:
            for lab in labels:
                cid = A.case_id(lab)
                alpha = S.complex_value(1.2, -0.7) if cid in (0, 7) else S.real_value(1.2)
                items.append((lab, s, s, s, alpha, S.complex_value(0.9, 0.3)))
        span = f"m=n=k={sizes[0]}" if len(sizes) == 1 else f"m=n=k={sizes[0]}..{sizes[-1]} step {sizes[1] - sizes[0]}"
        desc = (f"BASELINE configs[1]: {len(labels)}-label sweep, {span} ({len(items)} gemm calls per step), "
                "column-major, alpha=1.2-0.7i (cases 0,3; real 1.2 otherwise), beta=0.9+0.3i")
        return desc, items, "uniform"
    if args.workload == "cfg1":
        return ("BASELINE configs[0]: dssd m=n=k=1024, alpha=beta=1",
                [("dssd", 1024, 1024, 1024, S.real_value(1.0), S.real_value(1.0))], "uniform")
    if args.workload == "cfg3":
        return ("BASELINE configs[2]: zzzd 1m, m=n=k=8192, alpha=0.5+1.5i, beta=1",
                [("zzzd", 8192, 8192, 8192, S.complex_value(0.5, 1.5), S.real_value(1.0))], "uniform")
    if args.workload.startswith("cfg4"):
        lab = args.workload.split("-")[1]
        return (f"BASELINE configs[3]: {lab} m=n=k=16384, beta=0",
                [(lab, 16384, 16384, 16384, S.real_value(1.0), S.real_value(0.0))], "uniform")
    k = int(args.workload.split("-k")[1])
    return (f"BASELINE configs[4]: sddd rank-k update m=n=32768 k={k}, alpha=-1, beta=1",
            [("sddd", 32768, 32768, k, S.real_value(-1.0), S.real_value(1.0))], "normal")


def useful_flops(items):
    from oracle import abi as A
    return sum(A.flops_of_case(A.case_id(l), m, n, k) for l, m, n, k, _, _ in items)


# ------------------------------------------------------------------ operands
def make_operands(M, items, workload_name, seed, dist_kind, dev, stream, world=1, rank=0, shard_mode="columns"):
    """The step's operands and calls: one A/B/C per distinct (role, dtype, shape), so calls with the
    same C dtype and shape update one C buffer in sequence (a dependency chain), B and C column
    panels per rank.  Entries from the reference Rng on the device: uniform[-1,1) (fill_uniform) or
    normal(0,1) by Box-Muller over the same draws (fill_normal).  Shared with the parity test of the
    bench's own batch (tests/test_bench_parity_gpu.py).
    Returns (ops {key: (tensor, view)}, shard {item: (j0, nb)}, calls, call_info, a_bufs)."""
    import torch

    def alloc(dtype, m, n):
        t = torch.empty(max(m * n, 1) * M.dtype_size(dtype), dtype=torch.uint8, device=dev)
        return t, M.MatrixView.make(t.data_ptr(), m, n, 1, max(m, 1), dtype)

    ops, a_bufs, shard = {}, [], {}
    # Multi-GPU split.  chains: every call stays whole; the calls updating one C buffer (a
    # dependency chain) go to one rank, chains balanced over the ranks by their flops (longest
    # first); each rank generates the operands it reads.  columns: C and B column panels per
    # rank, A broadcast from rank 0 inside every step.
    mine = set()
    if shard_mode == "chains":
        chain_flops = {}
        for lab, m, n, k, _, _ in items:
            key = (lab[0], m, n)
            chain_flops[key] = chain_flops.get(key, 0.0) + M.flops_of_case(M.CaseLabel.parse(lab).case_id(), m, n, k)
        load = [0.0] * world
        owner = {}
        for key in sorted(chain_flops, key=lambda x: -chain_flops[x]):
            r = min(range(world), key=lambda q: load[q])
            owner[key] = r
            load[r] += chain_flops[key]
        mine = {key for key, r in owner.items() if r == rank}
    for lab, m, n, k, _, _ in items:
        if shard_mode == "chains":
            j0, nb = (0, n) if (lab[0], m, n) in mine else (0, 0)
        else:
            j0, nb = M.shard_columns(n, world, rank, 128)
        shard[(lab, m, n, k)] = (j0, nb)
        if nb == 0:
            continue
        dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
        for role, dt, shape in (("a", da, (m, k)), ("b", db, (k, nb)), ("c", dc, (m, nb))):
            key = (role, dt, shape)
            if key not in ops:
                t, v = alloc(dt, *shape)
                tag = f"{workload_name}/{role}/{M.dtype_letter(dt)}/{shape}/r{0 if role == 'a' or shard_mode == 'chains' else rank}"
                state = M.Rng(seed).split(tag).state
                if dist_kind == "normal":
                    M.fill_normal(v, state, stream)
                else:
                    M.fill_uniform(v, state, stream)
                ops[key] = (t, v)
                if role == "a" and shard_mode == "columns":
                    a_bufs.append(t)
    calls, call_info = [], []  # call_info: (case id, useful flops, computation precision) per call
    for lab, m, n, k, al, be in items:
        j0, nb = shard[(lab, m, n, k)]
        if nb == 0:
            continue
        dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
        comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
        va = ops[("a", da, (m, k))][1]
        vb = ops[("b", db, (k, nb))][1]
        vc = ops[("c", dc, (m, nb))][1].with_comp_prec(comp)
        calls.append((al, va, vb, be, vc))
        cid = M.CaseLabel.parse(lab).case_id()
        call_info.append((cid, M.flops_of_case(cid, m, nb, k), lab[3]))
    return ops, shard, calls, call_info, a_bufs



# ------------------------------------------------------------------- clocks
# nvidia-smi's NVML queries hold the driver lock: at a 200 ms period they stalled the host
# enqueue of lone calls by 15-65 ms in 2 of 10 steps (cfg3 33.1 -> 35.3 TFLOP/s at 1000 ms)
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("MDGEMM_BENCH_CLOCK_MS", "1000")], stdout=self.file, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        self.device_index = device_index
        # the first sample lands before the timed region starts (a region of a few ms -- cfg1 --
        # would otherwise end before nvidia-smi has started: no clock record at all)
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0:
            if os.path.getsize(self.file.name) > 0:
                break
            time.sleep(0.01)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        rows = []
        for line in open(self.file.name):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.file.name)
        if len(rows) < 2:  # a short region: one more sample right at its end, so two bracket it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device_index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                for line in out.stdout.splitlines():
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 8:
                        rows.append(parts)
            except (OSError, subprocess.SubprocessError):
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


# ------------------------------------------------------------- peak numbers
def peaks():
    with open(PEAKS_FILE) as f:
        p = json.load(f)
    hbm = None
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        hbm = json.load(open(mp)).get("hbm_gbs")
    return {"dmma_tflops": p["dmma_tflops"], "ffma_tflops": p["ffma_tflops"], "hbm_gbs": hbm or 6650.0,
            "hbm_source": "MEASURED_PEAKS.json" if hbm else "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------ b200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1901_06015_b200 as M

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook: MDGEMM_BENCH_BACKEND=gloo runs the multi-rank path functionally
    # with several ranks on fewer GPUs (host-staged collectives, no rank ever
    # waits on another rank's kernels).  Production runs use NCCL, one GPU each.
    backend = os.environ.get("MDGEMM_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    desc, items, dist_kind = workload(args)
    cfg = M.Config.defaults().set("gpu.numerics", args.numerics)

    shard_mode = args.shard if args.shard != "auto" else ("chains" if args.workload == "sweep" else "columns")
    if world == 1:
        shard_mode = "columns"
    ops, shard, calls, call_info, a_bufs = make_operands(M, items, args.workload, args.seed, dist_kind, dev, stream,
                                                         world, rank, shard_mode)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    # Column panels over NCCL ranks: the library's own multi-GPU entry point (mdg_gemm_sharded)
    # broadcasts A from rank 0 on a side stream while each rank packs its B panel.  (The gloo
    # test hook keeps the torch.distributed broadcast: several ranks may share one GPU there.)
    lib_comm = None
    if world > 1 and backend == "nccl" and shard_mode == "columns":
        uid = [M.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        lib_comm = M.Comm(uid[0], world, rank)

    def step():
        if lib_comm is not None:
            for al, va, vb, be, vc in calls:
                M.gemm_sharded(lib_comm, 0, al, va, vb, be, vc, cfg, stream)
            return
        if world > 1:
            for t in a_bufs:
                dist.broadcast(t, src=0)
        # the step's calls as one batch, forked from / joined into the timed stream: calls that
        # share no memory (different C buffers) run concurrently on the library's compute streams
        M.gemm_batch(calls, cfg, stream=stream, sync=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # no cyclic-GC pass in the middle of the timed steps (a full collection of a process with torch
    # loaded stalls the host enqueue for tens of ms; lone calls then leave the GPU idle)
    gc.collect()
    gc.disable()
    sampler = ClockSampler(local)
    launches0 = M.launch_count()
    step_ms, enqueue_ms = [], []
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush between timed steps (outside the events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        step()
        enqueue_ms.append((time.perf_counter() - h0) * 1e3)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = M.launch_count() - launches0
    clocks = sampler.stop()
    gc.enable()
    total_ms = sum(step_ms)

    # Kernels of the timed step itself: one more step of the same batch with the
    # library's per-launch CUDA events (each dual-pipe launch is bracketed on its
    # own stream after its packs, so its span is its own duration).
    flush.fill_(1)
    torch.cuda.synchronize()
    M.profile_begin()
    step()
    torch.cuda.synchronize()
    bstats = M.profile_end()

    # Per-kernel roofline: inside the timed steps independent calls overlap on
    # several streams, so a launch's event span is not its own duration; one
    # extra step runs the same calls serialized on the timed stream, each
    # kernel bracketed by CUDA events (mdg_profile_begin/end).
    # (an untimed serialized pass first: isolated calls may use kernel variants
    # the batched steps never launched, and CUDA loads modules lazily)
    serial_calls = [] if args.no_serial else calls
    for al, va, vb, be, vc in serial_calls:
        M.gemm_async(al, va, vb, be, vc, cfg, stream)
    flush.fill_(1)
    torch.cuda.synchronize()
    M.profile_begin()
    call_events = []
    for al, va, vb, be, vc in serial_calls:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record(stream)
        M.gemm_async(al, va, vb, be, vc, cfg, stream)
        ev[1].record(stream)
        call_events.append(ev)
    torch.cuda.synchronize()
    kstats = M.profile_end()
    serial_ms = sum(v["ms"] for v in kstats.values())
    # per mixed-datatype case (BASELINE's metric): whole calls (packs + gemm) in the serialized step
    per_case, pk0 = {}, peaks()
    for (cid, fl, comp), (e0, e1) in zip(call_info, call_events):
        c = per_case.setdefault(M.CASE_NAMES[cid], {"calls": 0, "flops": 0.0, "ms": 0.0, "ideal_ms": 0.0})
        c["calls"] += 1
        c["flops"] += fl
        c["ms"] += e0.elapsed_time(e1)
        c["ideal_ms"] += fl / ((pk0["ffma_tflops"] if comp == "s" else pk0["dmma_tflops"]) * 1e9)
    per_case = {name: {"calls": c["calls"], "GFLOPS": round(c["flops"] / c["ms"] / 1e6, 1),
                       "frac_of_peak": round(c["ideal_ms"] / c["ms"], 3)} for name, c in per_case.items()}
    # Per mixed-datatype case, batched (the way the timed step runs them): the calls of one case
    # as one gemm_batch (FP64 and FP32 labels of the case share the dual-pipe launches)
    per_case_batched = {}
    if not args.no_serial and args.workload == "sweep":
        pk1 = peaks()
        by_case = {}
        for (cid, fl, comp), call in zip(call_info, calls):
            e = by_case.setdefault(M.CASE_NAMES[cid], {"calls": [], "flops": 0.0, "ideal_ms": 0.0})
            e["calls"].append(call)
            e["flops"] += fl
            e["ideal_ms"] += fl / ((pk1["ffma_tflops"] if comp == "s" else pk1["dmma_tflops"]) * 1e9)
        for name, e in by_case.items():
            M.gemm_batch(e["calls"], cfg, stream=stream, sync=False)  # warm-up
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            M.gemm_batch(e["calls"], cfg, stream=stream, sync=False)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            per_case_batched[name] = {"calls": len(e["calls"]), "GFLOPS": round(e["flops"] / ms / 1e6, 1),
                                      "frac_of_serialized_peak": round(e["ideal_ms"] / ms, 3)}
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()

    flops = useful_flops(items) * args.steps
    value = flops / (total_ms * 1e-3) / 1e9
    pk = peaks()
    # time the whole job would take at the measured per-GPU peaks
    ideal_s = sum(M.flops_of_case(M.CaseLabel.parse(l).case_id(), m, n, k) /
                  ((pk["ffma_tflops"] if l[3] == "s" else pk["dmma_tflops"]) * 1e12 * world)
                  for l, m, n, k, _, _ in items) * args.steps
    peak_fraction = ideal_s / (total_ms * 1e-3)

    # roofline of the dominant kernel of the timed step (rank 0's launches)
    traffic_map = json.load(open(TRAFFIC_FILE)) if os.path.exists(TRAFFIC_FILE) else {}
    dual = bstats.get("dual_d", {"ms": 0.0})
    dom = max(("dmma", "ffma", "pack"), key=lambda k: kstats[k]["ms"])
    ks = kstats[dom]
    traffic = traffic_map.get(dom)
    # (pack spans on their side streams include waiting for SMs the dual launches hold, so the
    # dual kernel is the step's compute kernel whenever it ran)
    if dual.get("launches", 0) > 0:
        # Both pipes at once: the roofline is the serialized pipe mix of the same flops
        # (the time the DMMA flops take at the FP64 peak plus the FFMA flops at the FP32
        # peak); frac > 1 means the kernel beats running the pipes one after the other.
        fd, ff, ms = dual["work"], bstats["dual_f"]["work"], dual["ms"]
        achieved = (fd + ff) / (ms * 1e-3) / 1e12
        serial_peak = (fd + ff) / (fd / pk["dmma_tflops"] + ff / pk["ffma_tflops"]) if fd + ff else 0.0
        roof = {"bound": "tensor", "achieved": achieved, "peak": serial_peak, "unit": "TFLOP/s",
                "frac": achieved / serial_peak if serial_peak else 0.0, "traffic": traffic_map.get("dual"),
                "traffic_scope": "DRAM bytes of ONE captured launch of the 3584/4096 sweep slice (ncu --set full, "
                                 "12.6 ms: 0.48 TB/s, 6 % of the HBM rate -- the kernel is pipe-bound); achieved / peak are "
                                 "flops over all launches of the step",
                "kernel": "gemm_dual: FP64 DMMA.8x8x4 warps + FP32 FFMA2 warps on every SM at once",
                "pipes": {"dmma": {"achieved": fd / (ms * 1e-3) / 1e12, "peak": pk["dmma_tflops"],
                                   "frac": fd / (ms * 1e-3) / 1e12 / pk["dmma_tflops"]},
                          "ffma": {"achieved": ff / (ms * 1e-3) / 1e12, "peak": pk["ffma_tflops"],
                                   "frac": ff / (ms * 1e-3) / 1e12 / pk["ffma_tflops"]}},
                "launches": dual["launches"], "kernel_ms_per_step": ms,
                "peak_source": "serialized mix of the measured DMMA / FFMA peaks (profiles/peaks_r01.json) for "
                               "this step's flops",
                "algorithmic_work": "2*me*ne*ke real flops per job (= flops_of_case)",
                "measured": "one extra step of the same batch, CUDA events around every launch"}
    elif dom == "pack":
        achieved = ks["work"] / (ks["ms"] * 1e-3) / 1e9 if ks["ms"] else 0.0
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "kernel": "pack",
                "peak_source": pk["hbm_source"]}
    else:
        achieved = ks["work"] / (ks["ms"] * 1e-3) / 1e12 if ks["ms"] else 0.0
        peak = pk["dmma_tflops"] if dom == "dmma" else pk["ffma_tflops"]
        roof = {"bound": "tensor" if dom == "dmma" else "fp32-simt", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "kernel": "gemm_dmma (DMMA.8x8x4 fp64 tensor pipe)" if dom == "dmma" else "gemm_ffma (FFMA fp32)",
                "peak_source": "measured: tools/peaks.cu on this pool's B200 (profiles/peaks_r01.json)",
                "algorithmic_work": "2*me*ne*ke real flops per launch (= flops_of_case, the 1m reduction has no waste)"}
    roof.setdefault("measured", "one serialized step after the timed region, CUDA events around every launch")
    kernels = {}
    for kind, v in kstats.items():
        if not v["launches"] or not v["ms"]:
            continue
        rate = v["work"] / (v["ms"] * 1e-3)
        if kind in ("pack", "beta", "fill"):
            kernels[kind] = {"launches": v["launches"], "ms": round(v["ms"], 3), "GB/s": round(rate / 1e9, 1),
                             "frac_of_hbm": round(rate / 1e9 / pk["hbm_gbs"], 3)}
        else:
            peak = pk["dmma_tflops"] if kind == "dmma" else pk["ffma_tflops"]
            kernels[kind] = {"launches": v["launches"], "ms": round(v["ms"], 3), "TFLOP/s": round(rate / 1e12, 2),
                             "frac_of_peak": round(rate / 1e12 / peak, 3)}
    kernel_share = {k: round(v["ms"] / serial_ms, 4) if serial_ms else 0 for k, v in kstats.items() if v["launches"]}

    # ---- e2e: public gemm() on pinned host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        host = {}
        for key, (t, v) in ops.items():
            h = torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True)
            h.copy_(t)
            hv = M.MatrixView.from_buffer_copy(v)
            hv.base = h.data_ptr()
            host[key] = (h, hv)
        hcalls = []
        for lab, m, n, k, al, be in items:
            j0, nb = shard[(lab, m, n, k)]
            if nb == 0:
                continue
            dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
            comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
            ha, hb, hc = host[("a", da, (m, k))], host[("b", db, (k, nb))], host[("c", dc, (m, nb))]
            hcalls.append((al, ha[1], hb[1], be, hc[1].with_comp_prec(comp)))
        # One gemm_batch per step through the public batched gemm() on host MatrixViews: every
        # distinct host operand is copied into HBM once per step and every host C goes back to the
        # host after its last writer (h2d/d2h below are the bytes the library actually moved, from
        # its own counters); copies overlap neighbouring calls' kernels.
        torch.cuda.synchronize()
        M.gemm_batch(hcalls, cfg)  # one untimed step: the pool grows to the step's resident set
        if world > 1:
            dist.barrier()
        s0 = M.staging_bytes()
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            M.gemm_batch(hcalls, cfg)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        gc.enable()
        s1 = M.staging_bytes()
        h2d = (s1[0] - s0[0]) // args.steps
        d2h = (s1[1] - s0[1]) // args.steps
        if world > 1:
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": flops / el / 1e9, "unit": "GFLOPS", "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "api": "mdgemm::gemm_batch / mdg_gemm_batch on pinned host MatrixViews (synchronous, one batch per "
                      "step): each distinct host operand crosses PCIe once per step, each host C returns once",
               "timer": "host wall clock around synchronous calls"}

    # ---- the reference arm's own sample (same labels, sizes, scalars): device-resident as one batch,
    # and end to end through the unchanged per-call gemm() on pageable host buffers (one operand set
    # per label, every call stages its own A, B, C in and C out) -- a like-for-like pair for the
    # reference arm's number
    same = None
    if not args.no_e2e and world == 1:
        same = same_config_run(M, args, stream)
    if lib_comm is not None:
        torch.cuda.synchronize()
        lib_comm.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64/f32 (per label computation precision)",
        "data": "synthetic: reference splitmix64 Rng uniform[-1,1) generated on device"
                if dist_kind == "uniform" else
                "synthetic: normal(0,1) by Box-Muller over the reference splitmix64 Rng draws (mdg_fill_normal), on device",
        "config": {"workload": desc, "calls": len(items), "labels": len({it[0] for it in items}),
                   "numerics": args.numerics,
                   "parallelism": ("single GPU" if world == 1 else
                                   f"whole calls by C-buffer chain x{world}, chains balanced by flops, no collective"
                                   if shard_mode == "chains" else
                                   f"column panels x{world}, A broadcast by mdg_gemm_sharded over NCCL"
                                   if lib_comm is not None else f"column panels x{world}, A broadcast by torch.distributed"),
                   "l2": "operands > L2 per step and a 512 MiB L2 flush between timed steps"},
        "peak_fraction": peak_fraction,
        "peaks": {"dmma_tflops": pk["dmma_tflops"], "ffma_tflops": pk["ffma_tflops"]},
        "roofline": roof,
        "kernel_share": kernel_share,  # serialized pass of lone calls (classic kernels)
        "step_kernel_share": ({"dual": round(dual["ms"] / (total_ms / args.steps), 4)}
                              if dual.get("launches", 0) else None),
        "step_kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3)} for k, v in bstats.items()
                         if v["launches"] or v["ms"]},
        "kernels": kernels,
        "per_case": per_case,
        "per_case_batched": per_case_batched,
        "serialized_step_ms": serial_ms,
        "step_ms": [round(x, 3) for x in step_ms],
        "host_enqueue_ms": [round(x, 1) for x in enqueue_ms],
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "same_config_as_reference": same,
        "libraries_loaded": loaded_libraries(),
    }
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def same_config_run(M, args, stream):
    """The reference arm's sample on this GPU: device-resident (one gemm_batch, CUDA events) and
    per-call gemm() from pageable host memory (host wall clock, every call synchronous)."""
    import numpy as np
    import torch
    _, sample, text, dist_kind = reference_sample(args, M.Scalar)
    flops = useful_flops(sample)
    cfg = M.Config.defaults().set("gpu.numerics", args.numerics)
    dev_ops, host_ops, keep = [], [], []
    for i, (l, m, n, k, al, be) in enumerate(sample):
        dc, da, db = (M.dtype_from_letter(ch) for ch in l[:3])
        comp = M.SINGLE if l[3] == "s" else M.DOUBLE
        trip = []
        for role, dt, (r, c) in (("a", da, (m, k)), ("b", db, (k, n)), ("c", dc, (m, n))):
            t = torch.empty(max(r * c, 1) * M.dtype_size(dt), dtype=torch.uint8, device="cuda")
            v = M.MatrixView.make(t.data_ptr(), r, c, 1, max(r, 1), dt)
            state = M.Rng(args.seed).split(f"same/{l}/{role}").state
            (M.fill_normal if dist_kind == "normal" else M.fill_uniform)(v, state, stream)
            trip.append((t, v))
        dev_ops.append((al, trip[0][1], trip[1][1], be, trip[2][1].with_comp_prec(comp)))
        keep.extend(t for t, _ in trip)  # the views hold raw pointers: the tensors must outlive the batch
        hs = []
        for t, v in trip:
            h = np.empty(t.numel(), np.uint8)  # pageable, like the reference's Matrix storage
            h[:] = t.cpu().numpy()
            hv = M.MatrixView.from_buffer_copy(v)
            hv.base = h.ctypes.data
            hs.append((h, hv))
        host_ops.append((al, hs[0][1], hs[1][1], be, hs[2][1].with_comp_prec(comp), hs))
    torch.cuda.synchronize()
    M.gemm_batch(dev_ops, cfg, stream=stream, sync=False)  # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        M.gemm_batch(dev_ops, cfg, stream=stream, sync=False)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    device = flops * len(times) / sum(times) / 1e9
    for al, a, b, be, c, _ in host_ops:  # warm-up pass through the public per-call API
        M.gemm(al, a, b, be, c, cfg)
    s0 = M.staging_bytes()
    gc.collect()
    gc.disable()
    pass_s = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for al, a, b, be, c, _ in host_ops:
            M.gemm(al, a, b, be, c, cfg)
        pass_s.append(time.perf_counter() - t0)
    # the median pass: one host hiccup (a descheduled copy thread on a shared box) once cost a pass 1 s
    el = sorted(pass_s)[len(pass_s) // 2] * args.steps
    gc.enable()
    s1 = M.staging_bytes()
    del keep
    return {"workload": text, "calls": len(sample), "flops_per_step": flops,
            "device_resident": {"value": device, "unit": "GFLOPS", "api": "gemm_batch on device views, CUDA events"},
            "e2e_per_call": {"value": flops * args.steps / el / 1e9, "unit": "GFLOPS",
                             "h2d_bytes_per_step": (s1[0] - s0[0]) // args.steps,
                             "d2h_bytes_per_step": (s1[1] - s0[1]) // args.steps,
                             "api": "mdgemm::gemm / mdg_gemm per call on pageable host MatrixViews (synchronous, "
                                    "one operand set per label; each call stages its operands in and C out)",
                             "timer": "host wall clock, median pass", "pass_ms": [round(x * 1e3, 1) for x in pass_s]}}


# ----------------------------------------------------------- reference arm
def reference_sample(args, S=None):
    """The bounded CPU sample of the workload: every sweep label at m=n=k=--cpu-size (512), or a
    512 x 512 column/row sub-block of a single-problem config with its full inner dimension."""
    desc, items, dist_kind = workload(args, S)
    if args.workload == "sweep":
        s = args.cpu_size
        seen, sample = set(), []
        for l, _, _, _, al, be in items:
            if l not in seen:
                seen.add(l)
                sample.append((l, s, s, s, al, be))
        text = f"all {len(sample)} sweep labels at m=n=k={s}"
    else:
        sample, text = [], ""
        for l, m, n, k, al, be in items:  # a column/row sub-block with the full inner dimension
            mm, nn = min(m, 512), min(n, 512)
            sample.append((l, mm, nn, k, al, be))
            text = f"{l} sub-block {mm}x{nn} with the full k={k}"
    return desc, sample, text, dist_kind


def sample_operands(A, sample, seed, dist_kind, fill):
    """Host operands of the CPU sample, one A/B/C per label and shape: uniform entries from the
    reference Rng (the C restatement, bitwise the reference's fill_uniform), or normal(0,1) by the
    same Box-Muller definition the device generator uses.  `fill(view, state)` fills a view."""
    from oracle import oracle as O
    mats, calls = {}, []
    for l, m, n, k, al, be in sample:
        dc, da, db = (A.dtype_from_letter(ch) for ch in l[:3])
        for role, dt, shape in (("a", da, (m, k)), ("b", db, (k, n)), ("c", dc, (m, n))):
            key = (l, role, shape)
            if key not in mats:
                h = A.HostMatrix(dt, *shape)
                state = O.orc_rng_state(seed, [l, role, *shape])
                if dist_kind == "normal":
                    import numpy as np
                    real = np.float32 if dt in (A.DT_S, A.DT_C) else np.float64
                    h.buf.view(real)[:] = O.normal_values(state, np.arange(h.buf.size // np.dtype(real).itemsize))
                else:
                    fill(h.view(), state)
                mats[key] = h
        comp = A.SINGLE if l[3] == "s" else A.DOUBLE
        calls.append((al, mats[(l, "a", (m, k))], mats[(l, "b", (k, n))], be, mats[(l, "c", (m, n))], comp))
    return mats, calls


def run_reference_steps(args, steps, warmup):
    """Times the reference engine (oracle/_ref, built from the reference's own sources) through its
    public gemm() on host memory, all host threads, ctemp=on.  Loads only oracle/ libraries: the
    product package is never imported on this path."""
    from oracle import abi as A
    from oracle import oracle as O

    if O.ref is None:
        raise RuntimeError("oracle/_ref/libmdgemm_ref.so is missing")
    cores = os.cpu_count() or 1
    cfg = O.ref_config_defaults()
    cfg.threads = cores
    cfg.ctemp = A.CTEMP_ON
    desc, sample, text, dist_kind = reference_sample(args, A.Scalar)
    _, calls = sample_operands(A, sample, args.seed, dist_kind, O.orc_fill_uniform)
    views = [(al, a.view(), b.view(), be, c.view(comp=comp)) for al, a, b, be, c, comp in calls]
    flops = useful_flops(sample)
    for _ in range(warmup):
        for c in views:
            O.ref_gemm(*c, cfg)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        for c in views:
            O.ref_gemm(*c, cfg)
        times.append(time.perf_counter() - t0)
    return desc, text, flops, times, cores


def cpu_baseline(args):
    try:
        _, text, flops, times, cores = run_reference_steps(args, 1, 1)
    except Exception as e:  # noqa: BLE001 - reported, not fatal for the GPU line
        return {"value": None, "unit": "GFLOPS", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    return {"value": flops / times[0] / 1e9, "unit": "GFLOPS", "cores": cores, "kind": "reference",
            "sample": f"{text}; reference gemm() (oracle/_ref) with gemm.threads={cores}, ctemp.enable=on; "
                      f"1 warm-up + 1 timed pass ({times[0]:.1f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    desc, text, flops, times, cores = run_reference_steps(args, args.steps, args.warmup)
    total = sum(times)
    value = flops * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOPS",
        "n_gpus": int(os.environ.get("WORLD_SIZE", str(args.gpus))), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64/f32 (per label computation precision)", "data": "synthetic: reference Rng uniform[-1,1)",
        "config": {"workload": desc, "sample": text, "numerics": "reference CPU engine"},
        "cpu_baseline": {"value": value, "unit": "GFLOPS", "cores": cores, "kind": "reference",
                         "sample": f"{text}; reference gemm() with gemm.threads={cores}, ctemp.enable=on"},
        "e2e": {"value": value, "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "libraries_loaded": loaded_libraries(),
    }
    print(json.dumps(line), flush=True)


def loaded_libraries():
    """The repo's shared objects mapped into this process (evidence of which code ran)."""
    out = []
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if len(line.split()) >= 6 else ""
            rel = os.path.relpath(path, ROOT) if path.startswith(ROOT) and path.endswith(".so") else None
            if rel and rel not in out:
                out.append(rel)
    except OSError:
        pass
    return out


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
