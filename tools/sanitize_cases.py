#!/usr/bin/env python3
"""Small problems that drive every kernel family of the library, for
compute-sanitizer (racecheck / synccheck / memcheck / initcheck):

  python tools/sanitize_cases.py --family F      (one family per process)
  tools/sanitize.sh TOOL                         (all families under TOOL)

Each family sets the tuning knobs that force its kernels (read once per
process, hence one process per family) and MDGEMM_SMS, which schedules for a
few SMs so that tiny problems still run the persistent, stream-K and
multi-tile paths.  Every result is checked against the oracle (the
reference's per-element criterion), so a run also proves the kernels stayed
correct under the sanitizer's serialisation.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FAMILIES = {
    # classic grids (one tile per CTA), both tile shapes, every C route
    "classic": {"MDGEMM_DMMA_WS": "-1", "MDGEMM_FFMA_WS": "-1", "MDGEMM_STREAMK": "-1"},
    # warp-specialised persistent kernels incl. the epilogue-warp DMMA variant and the stream-K tail
    "ws": {"MDGEMM_SMS": "4", "MDGEMM_DMMA_WS": "1", "MDGEMM_FFMA_WS": "1"},
    # classic kernels with the stream-K hybrid tail (seeded partial tiles, publish flags)
    "streamk": {"MDGEMM_SMS": "2", "MDGEMM_DMMA_WS": "-1", "MDGEMM_FFMA_WS": "-1", "MDGEMM_STREAMK": "1"},
    # split-K partial tiles + the reduce pass
    "splitk": {"MDGEMM_DMMA_WS": "-1", "MDGEMM_FFMA_WS": "-1", "MDGEMM_SPLITK": "3"},
    # the dual-pipe kernel (gemm_batch of mixed computation precisions)
    "dual": {"MDGEMM_SMS": "4", "MDGEMM_DUAL": "2"},
    # EXACT replay kernel (every output route)
    "exact": {},
    # pack kernels alone (every format, side, conj, scale, reg_block)
    "pack": {},
}


def run(family: str) -> int:
    import numpy as np
    import torch

    import paper_1901_06015_b200 as M
    from oracle import oracle as O
    from tests.helpers import SCALARS, Problem, config

    torch.cuda.set_device(0)
    checked = 0

    def check(p, al, be, kv, device=None):
        nonlocal checked
        dA, dB, dC = device or p.device()
        da, db, dc = p.views(A=dA, B=dB, C=dC)
        M.gemm(SCALARS[al], da, db, SCALARS[be], dc, config(kv))
        got = p.C.clone()
        got.buf[:] = dC.bytes()
        va, vb, vc = p.views()
        _, _, vg = p.views(C=got)
        if kv.get("gpu.numerics") == "exact":
            want = p.C.clone()
            _, _, vw = p.views(C=want)
            O.orc_gemm(SCALARS[al], va, vb, SCALARS[be], vw, config(kv))
            assert got.buf.tobytes() == want.buf.tobytes(), (p.label, "EXACT differs")
        else:
            viol = O.orc_violation(SCALARS[al], va, vb, SCALARS[be], vc, vg, p.comp)
            assert viol <= 1.0, (p.label, viol)
        checked += 1

    fast = {"gpu.numerics": "fast"}
    if family == "classic":
        for label in ("dddd", "ssss", "zzzd", "cccs", "cdds", "sddd", "zczd", "dzzd", "czcs", "zdzs"):
            check(Problem(label, 150, 130, 70), "p7", "m3", fast)
            check(Problem(label, 33, 21, 45, c_kind="row", variant="r"), "one", "c34", fast)
            check(Problem(label, 17, 9, 20, c_kind="gen", variant="g"), "minus_one", "zero", fast)
    elif family == "ws":
        for label in ("dddd", "sddd", "ssss", "cdds", "sdds", "ddds"):
            check(Problem(label, 300, 280, 200), "p7", "m3", fast)   # 9 tiles on 4 CTAs, stream-K tail
            check(Problem(label, 260, 270, 40), "one", "one", fast)  # short k
    elif family == "streamk":
        for label in ("dddd", "zzzd", "ssss", "cccs", "sddd"):
            check(Problem(label, 330, 300, 300), "p7", "m3", fast)
    elif family == "splitk":
        for label in ("dddd", "ssss", "zzzd", "sddd", "cdds"):
            check(Problem(label, 100, 90, 600), "p7", "m3", fast)
    elif family == "dual":
        probs = [Problem(label, 150, 140, 90, seed=5) for label in
                 ("dddd", "ssss", "zzzd", "cccs", "sddd", "cdds", "dzzd", "zcds")]
        devs = [p.device() for p in probs]
        wants = []
        for p in probs:
            want = p.C.clone()
            va, vb, _ = p.views()
            _, _, vw = p.views(C=want)
            O.orc_gemm(SCALARS["p7"], va, vb, SCALARS["m3"], vw)
            wants.append(want)
        M.gemm_batch([(SCALARS["p7"], d[0].view(conj=p.conj_a), d[1].view(conj=p.conj_b), SCALARS["m3"],
                       d[2].view(comp=p.comp)) for p, d in zip(probs, devs)], config(fast))
        for p, (dA, dB, dC) in zip(probs, devs):
            got = p.C.clone()
            got.buf[:] = dC.bytes()
            va, vb, vc = p.views()
            _, _, vg = p.views(C=got)
            viol = O.orc_violation(SCALARS["p7"], va, vb, SCALARS["m3"], vc, vg, p.comp)
            assert viol <= 1.0, (p.label, viol)
            checked += 1
    elif family == "exact":
        ex = {"gpu.numerics": "exact"}
        for label in ("dddd", "zzzd", "cdds", "sddd", "zczd", "czcs"):
            check(Problem(label, 40, 30, 300), "cfg2_alpha_real" if label in ("cdds", "czcs") else "c55",
                  "cfg2_beta", {**ex, "ctemp.enable": "off"})
            check(Problem(label, 20, 17, 50, variant="on"), "one", "p3", {**ex, "ctemp.enable": "on"})
    elif family == "pack":
        from tests.helpers import HostMatrix
        for dt in (M.DT_S, M.DT_D, M.DT_C, M.DT_Z):
            for side in (M.LEFT, M.RIGHT):
                for fmt in ((M.STANDARD,) if not M.is_complex(dt) else (M.STANDARD, M.ONE_E, M.ONE_R)):
                    for rb in ((2, 4, 64) if fmt == M.ONE_E else (3, 4, 128)):
                        src = HostMatrix(dt, 37, 29).fill(O.orc_rng_state(1, ["san", dt, side, fmt, rb]))
                        target = (2 if M.is_complex(dt) and fmt == M.STANDARD else 0) + M.DOUBLE
                        scale = SCALARS["c55"] if fmt != M.STANDARD else SCALARS["p7"]
                        n = O.orc_packed_bytes(src.view(), side, fmt, target, rb)
                        want = np.zeros(n, np.uint8)
                        O.orc_pack(src.view(), side, fmt, 1, scale, target, rb, 0, want.ctypes.data)
                        d = src.to_device()
                        out = torch.zeros(n, dtype=torch.uint8, device="cuda")
                        M.pack_block_device(out.data_ptr(), d.view(), side, fmt, True, scale, target, rb)
                        torch.cuda.synchronize()
                        assert out.cpu().numpy().tobytes() == want.tobytes(), (dt, side, fmt, rb)
                        checked += 1
    torch.cuda.synchronize()
    print(f"sanitize_cases {family}: {checked} checks ok", flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", choices=sorted(FAMILIES), required=True)
    ap.add_argument("--print-env", action="store_true", help="print the family's environment and exit")
    a = ap.parse_args()
    if a.print_env:
        print(" ".join(f"{k}={v}" for k, v in FAMILIES[a.family].items()))
        return 0
    for k, v in FAMILIES[a.family].items():
        os.environ[k] = v
    return run(a.family)


if __name__ == "__main__":
    sys.exit(main())
