"""Per-region warp-stall breakdown from an ncu source-page CSV (--page source
--csv --print-source sass): regions are address ranges split at the given
instruction-mnemonic markers (default: the first/last DMMA and FFMA2 of a
kernel give the D and F mainloops).

    python tools/ncu_stalls.py gpurun_out/x/ncu_source.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
src = [(int(r[ci["Address"]], 16), r[ci["Source"]].strip(), r) for r in data if r and r[0].startswith("0x")]


def span(mn):
    idx = [k for k, (_, s, _) in enumerate(src) if s.split()[0:1] and mn in s.split()[0]]
    return (idx[0], idx[-1]) if idx else None


regions = {}
d = span("DMMA")
f = span("FFMA2")
if d:
    regions["D mainloop (first..last DMMA)"] = d
if f:
    regions["F mainloop (first..last FFMA2)"] = f
tot = defaultdict(float)
for name, (a, b) in list(regions.items()) + [("whole kernel", (0, len(src) - 1))]:
    acc = defaultdict(float)
    inst = defaultdict(float)
    samples = 0.0
    for _, s, r in src[a:b + 1]:
        samples += float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        for h in stall_cols:
            acc[h] += float(r[ci[h]] or 0)
        op = s.split()[0] if s.split() else "?"
        if op.startswith("@"):
            op = s.split()[1]
        inst[op.split(".")[0]] += float(r[ci["Instructions Executed"]] or 0)
    print(f"== {name}: {samples:.0f} samples")
    for h, v in sorted(acc.items(), key=lambda x: -x[1])[:8]:
        print(f"   {h:28s} {v:10.0f}  {100 * v / max(samples, 1):5.1f}%")
    top = sorted(inst.items(), key=lambda x: -x[1])[:10]
    print("   instructions:", ", ".join(f"{k} {v:.3g}" for k, v in top))
