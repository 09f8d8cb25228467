"""Per-label isolated gemm rate at one size (device-resident, CUDA events):
which of the 128 labels sit furthest below their pipe's measured peak.

    python tools/exp_labels.py [size] [labels...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06015_b200 as M  # noqa: E402
from tests.test_baseline_scale_gpu import DevMat  # noqa: E402
from tests.helpers import config  # noqa: E402

PEAKS = json.load(open(os.path.join(os.path.dirname(__file__), "..", "profiles", "peaks_r01.json")))


def main():
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    labels = sys.argv[2:] or [l.str() for l in M.CaseLabel.all()]
    cfg = config({})
    alpha_c, alpha_r, beta = M.Scalar.complex_value(1.2, -0.7), M.Scalar.real_value(1.2), M.Scalar.complex_value(0.9, 0.3)
    rows = []
    cache = {}
    for lab in labels:
        dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
        comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
        for key, dt, seed in (("a", da, 1), ("b", db, 2), ("c", dc, 3)):
            if (key, dt) not in cache:
                cache[(key, dt)] = DevMat(dt, s, s, seed)
        A, B, C = cache[("a", da)], cache[("b", db)], cache[("c", dc)]
        cid = M.CaseLabel.parse(lab).case_id()
        alpha = alpha_c if cid in (0, 7) else alpha_r
        call = lambda: M.gemm_async(alpha, A.view(), B.view(), beta, C.view(comp), cfg)
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(2):
            call()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 2
        fl = M.flops_of_case(cid, s, s, s)
        peak = PEAKS["ffma_tflops"] if comp == M.SINGLE else PEAKS["dmma_tflops"]
        rows.append((fl / ms / 1e9 / peak, lab, fl / ms / 1e9, ms))
    rows.sort()
    for frac, lab, tf, ms in rows:
        print(f"{lab} {tf:6.1f} TF/s  {frac:.3f} of peak  {ms:8.2f} ms")


if __name__ == "__main__":
    main()
