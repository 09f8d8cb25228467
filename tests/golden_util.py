"""Shared loaders for the golden fixtures (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

import paper_1901_06015_b200 as M
from tests.helpers import HostMatrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FMT = {"std": M.STANDARD, "1e": M.ONE_E, "1r": M.ONE_R}
SIDE = {"left": M.LEFT, "right": M.RIGHT}


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def sha(buf: np.ndarray) -> str:
    return hashlib.sha256(buf.tobytes()).hexdigest()


def matrix_from(dtype_letter, m, n, values) -> HostMatrix:
    h = HostMatrix(M.dtype_from_letter(dtype_letter), m, n)
    vals = h.values()
    for idx, (re, im) in enumerate(values):
        vals[idx % max(m, 1), idx // max(m, 1)] = complex(re, im) if M.is_complex(h.dtype) else re
    return h


def packed_element(buf: np.ndarray, kat, i, j):
    """PackedBlock::packed_element (packing.cpp:251-260) on raw bytes."""
    tgt = M.dtype_from_letter(kat["target"])
    real_block = FMT[kat["fmt"]] != M.STANDARD
    npt = {M.DT_S: np.float32, M.DT_D: np.float64, M.DT_C: np.complex64, M.DT_Z: np.complex128}
    t = npt[(tgt & 1) if real_block else tgt]
    arr = buf.view(t)
    pd = kat["reg_block"]
    rows = {"std": kat["m"], "1e": 2 * kat["m"], "1r": kat["m"] if kat["side"] == "left" else 2 * kat["m"]}[kat["fmt"]]
    cols = {"std": kat["n"], "1e": 2 * kat["n"], "1r": 2 * kat["n"] if kat["side"] == "left" else kat["n"]}[kat["fmt"]]
    if kat["side"] == "left":
        return arr[(i // pd) * pd * cols + j * pd + i % pd]
    return arr[(j // pd) * pd * rows + i * pd + j % pd]
