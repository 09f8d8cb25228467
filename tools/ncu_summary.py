"""Summarise the ncu captures of tools/profile_r01.sh into profiles/:
a markdown table of the key metrics per kernel and profiles/ncu_traffic.json
(DRAM bytes per captured launch next to the algorithmic bytes).

    python tools/ncu_summary.py gpurun_out/prof profiles/r01 [label]
"""
import csv
import json
import os
import sys

# algorithmic bytes of the captured launches (cfg2 slice at 4096, see profile_r01.sh)
ALGO = {
    # zzzd: 1e-packed A 8192x8192 f64 + 1r-packed B 8192x4096 f64 + C 4096^2 z read + written
    "dmma": 8192 * 8192 * 8 + 8192 * 4096 * 8 + 2 * 4096 * 4096 * 16,
    # cccs: same real dims in f32, C 4096^2 c read + written
    "ffma": 8192 * 8192 * 4 + 8192 * 4096 * 4 + 2 * 4096 * 4096 * 8,
    # zzzd 1e pack of A: 4096^2 z read, 8192^2 f64 written
    "pack": 4096 * 4096 * 16 + 8192 * 8192 * 8,
    # dddd 4096 on the warp-specialised kernel: A + B packed f64, C read + written
    "dmma_ws": 4 * 4096 * 4096 * 8,
    # cfg5 k=64 (sddd 32768^2 x 64) on the epilogue-warp WS kernel: A + B packed f64, C f32 read + written
    "dmma_ws_epi": 2 * 32768 * 64 * 8 + 2 * 32768 * 32768 * 4,
}
FLOPS = {"dmma": 2.0 * 8192 * 4096 * 8192, "ffma": 2.0 * 8192 * 4096 * 8192, "dmma_ws": 2.0 * 4096 ** 3,
         "dmma_ws_epi": 2.0 * 32768 * 32768 * 64}
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe % active"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "nsecond": 1e-9}


def load(path):
    rows = list(csv.reader(open(path)))
    h, units, r = rows[0], rows[1], rows[2]
    return {k: (v, u) for k, u, v in zip(h, units, r)}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else "round 1 (tools/profile_r01.sh"
    os.makedirs(dst, exist_ok=True)
    lines = [f"# ncu --set full captures, {label}, one launch each, --clock-control none)", "",
             "Launches: DMMA = `zzzd` 4096 (1m: me=8192, ne=4096, ke=8192), FFMA = `cccs` 4096 (same real dims), "
             "pack = the 1e pack of `zzzd`'s A, dmma_ws = the warp-specialised DMMA kernel on a lone `dddd` 4096 call, "
             "dmma_ws_epi = its epilogue-warp variant on cfg5 k=64 (`sddd` 32768^2 x 64), dual = one gemm_dual launch of "
             "the batched 3584/4096 sweep slice (tools/profile_dual.sh).  Per-launch times are cold-cache and serialised (ncu replays), so "
             "compare shares, not absolutes, with bench.py.", ""]
    traffic = {"what": "dram__bytes_read.sum + dram__bytes_write.sum of one captured launch (ncu --set full): "
                       "dmma = zzzd 4096, ffma = cccs 4096, pack = zzzd's 1e pack of A; algorithmic bytes alongside",
               "algorithmic_bytes_per_launch": {}}
    for k in ("dmma", "ffma", "pack", "dmma_ws", "dmma_ws_epi", "dual"):
        p = os.path.join(src, f"ncu_{k}_raw.csv")
        if not os.path.exists(p):
            continue
        m = load(p)
        lines.append(f"## {k}: `{m['Kernel Name'][0][:120]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in m:
                v, u = m[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        rd = float(m["dram__bytes_read.sum"][0]) * SCALE.get(m["dram__bytes_read.sum"][1], 1)
        wr = float(m["dram__bytes_write.sum"][0]) * SCALE.get(m["dram__bytes_write.sum"][1], 1)
        dur = float(m["gpu__time_duration.sum"][0]) * SCALE.get(m["gpu__time_duration.sum"][1], 1)
        traffic[k] = rd + wr
        if k == "dual":  # both pipes: fp64 tensor ops counted by ncu, FP32 via the FMA pipe share
            f64 = float(m["sm__ops_path_tensor_src_fp64.sum"][0])
            lines.append(f"| FP64 tensor ops in the launch | {f64:.4g} = {f64 / dur / 1e12:.2f} TFLOP/s of DMMA work |")
            lines.append("")
            continue
        traffic["algorithmic_bytes_per_launch"][k] = ALGO[k]
        lines.append(f"| DRAM bytes / algorithmic bytes | {(rd + wr) / ALGO[k]:.2f} |")
        if k in FLOPS:
            lines.append(f"| achieved (this launch) | {FLOPS[k] / dur / 1e12:.2f} TFLOP/s |")
        else:
            lines.append(f"| achieved (this launch) | {ALGO[k] / dur / 1e9:.0f} GB/s algorithmic |")
        lines.append("")
    open(os.path.join(dst, "ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
