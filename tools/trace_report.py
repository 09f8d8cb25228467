"""Summarise an MDGEMM_TRACE file (per-CTA %globaltimer stamps of the fast
gemm kernels): per kernel, the span, waves, mean per-CTA phases (fill = start
to first stage ready, mainloop, epilogue) and how busy the CTA slots were.

    python tools/trace_report.py gpurun_out/trace.txt [--last-per-shape]
"""
import sys
from collections import OrderedDict


def parse(path):
    kernels, cur = [], None
    for line in open(path):
        f = line.split()
        if f[0] == "K":
            cur = {"kind": f[1], "m": int(f[2]), "n": int(f[3]), "k": int(f[4]), "bm": int(f[5]),
                   "bn": int(f[6]), "splits": int(f[7]), "grid": int(f[8]), "ctas": []}
            kernels.append(cur)
        else:
            cur["ctas"].append(tuple(int(x) for x in f))
    return kernels


def report(kn):
    c = kn["ctas"]
    t0 = min(r[1] for r in c)
    t1 = max(r[4] for r in c)
    span = (t1 - t0) / 1e3
    fill = sum(r[2] - r[1] for r in c) / len(c) / 1e3
    issue = sum(r[5] - r[1] for r in c if len(r) > 5 and r[5]) / len(c) / 1e3
    loop = sum(r[3] - r[2] for r in c) / len(c) / 1e3
    epi = sum(r[4] - r[3] for r in c) / len(c) / 1e3
    busy = sum(r[4] - r[1] for r in c) / 1e3
    per_sm = {}
    for r in c:
        per_sm.setdefault(r[0], []).append(r)
    sms = len(per_sm)
    conc = max(len(v) for v in per_sm.values())
    # slots: max CTAs simultaneously resident on one SM
    def max_overlap(v):
        ev = sorted([(r[1], 1) for r in v] + [(r[4], -1) for r in v])
        cur = best = 0
        for _, d in ev:
            cur += d
            best = max(best, cur)
        return best
    slots = max(max_overlap(v) for v in per_sm.values())
    # start skew of the first wave and the tail: last CTA start vs kernel end
    starts = sorted(r[1] for r in c)
    ends = sorted(r[4] for r in c)
    tail = (t1 - ends[int(len(ends) * 0.5)]) / 1e3
    flops = 2.0 * kn["m"] * kn["n"] * kn["k"]
    print(f"{kn['kind']} {kn['m']}x{kn['n']}x{kn['k']} tile {kn['bm']}x{kn['bn']} splits {kn['splits']} grid {kn['grid']}"
          f" SMs {sms} slots/SM {slots}: span {span:.1f} us ({flops / span / 1e6:.1f} TF/s) |"
          f" per CTA fill {fill:.2f} (first issue after {issue:.2f}) loop {loop:.1f} epi {epi:.2f} us |"
          f" slot occupancy {busy / (span * sms * slots):.3f} | first-wave start skew {(starts[min(len(starts)-1, sms*slots-1)] - t0)/1e3:.2f} us"
          f" | end-median->end {tail:.1f} us")


def main():
    ks = parse(sys.argv[1])
    if "--last-per-shape" in sys.argv:
        last = OrderedDict()
        for k in ks:
            last[(k["kind"], k["m"], k["n"], k["k"])] = k
        ks = list(last.values())
    for k in ks:
        report(k)


if __name__ == "__main__":
    main()
