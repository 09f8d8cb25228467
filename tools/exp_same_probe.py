"""Why bench.same_config_run's device-resident leg differs from tools/exp_same_config.py: variations."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1901_06015_b200 as M
args = bench.parse_args()
stream = torch.cuda.current_stream()
_, sample, text, dist_kind = bench.reference_sample(args, M.Scalar)
flops = bench.useful_flops(sample)
keep, dev_ops = [], []
for i, (l, m, n, k, al, be) in enumerate(sample):
    dc, da, db = (M.dtype_from_letter(ch) for ch in l[:3])
    comp = M.SINGLE if l[3] == "s" else M.DOUBLE
    trip = []
    for role, dt, (r, c) in (("a", da, (m, k)), ("b", db, (k, n)), ("c", dc, (m, n))):
        t = torch.empty(max(r * c, 1) * M.dtype_size(dt), dtype=torch.uint8, device="cuda")
        v = M.MatrixView.make(t.data_ptr(), r, c, 1, max(r, 1), dt)
        M.fill_uniform(v, M.Rng(args.seed).split(f"same/{l}/{role}").state, stream)
        trip.append(v); keep.append(t)
    dev_ops.append((al, trip[0], trip[1], be, trip[2].with_comp_prec(comp)))
torch.cuda.synchronize()
def run(tag, cfg, st, prof):
    out = []
    for _ in range(4):
        torch.cuda.synchronize()
        if prof: M.profile_begin()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        M.gemm_batch(dev_ops, cfg, stream=st, sync=False)
        h1 = time.perf_counter()
        e1.record(stream)
        e1.synchronize()
        if prof: M.profile_end()
        out.append((round(e0.elapsed_time(e1), 2), round((h1 - h0) * 1e3, 2)))
    print(tag, "(event ms, host enqueue ms):", out, f"{flops / out[-1][0] / 1e6:.0f} GFLOPS")
cfg_d = M.Config.defaults()
cfg_f = M.Config.defaults().set("gpu.numerics", args.numerics)
run("defaults cfg, stream None, profile", cfg_d, None, True)
run("defaults cfg, stream None", cfg_d, None, False)
run("defaults cfg, torch stream", cfg_d, stream, False)
run("numerics cfg, stream None", cfg_f, None, False)
run("numerics cfg, torch stream", cfg_f, stream, False)
