"""Test fixtures: owning host/device matrices with the reference's storage
layouts (Matrix::make, matrix.hpp:17-43) and the shared problem generators.

Host operands are filled by the oracle's restatement of the reference Rng
(bit-identical to rng.hpp, pinned in test_oracle_pins.py), so every test sees
exactly the inputs the reference would draw for the same seed path."""
from __future__ import annotations

import numpy as np

import paper_1901_06015_b200 as M
from paper_1901_06015_b200 import DT_C, DT_D, DT_S, DT_Z, MatrixView, Scalar
from oracle import oracle as O

NP_TYPES = {DT_S: np.float32, DT_D: np.float64, DT_C: np.complex64, DT_Z: np.complex128}
ALL_DT = (DT_S, DT_D, DT_C, DT_Z)


def geometry(m: int, n: int, kind: str):
    if kind == "col":
        return 1, max(m, 1)
    if kind == "row":
        return max(n, 1), 1
    if kind == "gen":  # deliberate gaps between addressed elements
        return 2, 2 * max(m, 1) + 3
    raise ValueError(kind)


class HostMatrix:
    def __init__(self, dtype: int, m: int, n: int, kind: str = "col", fill_byte: int = 0):
        self.dtype, self.m, self.n, self.kind = dtype, m, n, kind
        self.rs, self.cs = geometry(m, n, kind)
        span = (m - 1) * self.rs + (n - 1) * self.cs + 1 if m > 0 and n > 0 else 0
        self.buf = np.full(max(span, 1) * M.dtype_size(dtype), fill_byte, np.uint8)

    def view(self, comp: int | None = None, conj: bool = False) -> MatrixView:
        v = MatrixView.make(self.buf.ctypes.data, self.m, self.n, self.rs, self.cs, self.dtype)
        if comp is not None:
            v.comp_prec = comp
        v.conj = int(conj)
        return v

    def tview(self, comp: int | None = None, conj: bool = False) -> MatrixView:
        """induced_transpose of view()."""
        v = self.view(comp, conj)
        v.m, v.n, v.rs, v.cs = v.n, v.m, v.cs, v.rs
        return v

    def fill(self, state: int) -> "HostMatrix":
        O.orc_fill_uniform(self.view(), state)
        return self

    def clone(self) -> "HostMatrix":
        h = HostMatrix.__new__(HostMatrix)
        h.__dict__.update(self.__dict__)
        h.buf = self.buf.copy()
        return h

    def values(self) -> np.ndarray:
        """Logical m x n elements as a (strided) numpy array."""
        t = NP_TYPES[self.dtype]
        arr = self.buf.view(t)
        es = np.dtype(t).itemsize
        return np.lib.stride_tricks.as_strided(arr, shape=(self.m, self.n), strides=(self.rs * es, self.cs * es))

    def to_device(self):
        return DeviceMatrix(self)


class DeviceMatrix:
    def __init__(self, host: HostMatrix):
        import torch
        self.dtype, self.m, self.n, self.kind, self.rs, self.cs = host.dtype, host.m, host.n, host.kind, host.rs, host.cs
        self.t = torch.from_numpy(host.buf.copy()).cuda()

    def view(self, comp: int | None = None, conj: bool = False) -> MatrixView:
        v = MatrixView.make(self.t.data_ptr(), self.m, self.n, self.rs, self.cs, self.dtype)
        if comp is not None:
            v.comp_prec = comp
        v.conj = int(conj)
        return v

    def tview(self, comp: int | None = None, conj: bool = False) -> MatrixView:
        v = self.view(comp, conj)
        v.m, v.n, v.rs, v.cs = v.n, v.m, v.cs, v.rs
        return v

    def bytes(self) -> np.ndarray:
        import torch
        torch.cuda.synchronize()
        return self.t.cpu().numpy()


def label_dtypes(label: str):
    return M.dtype_from_letter(label[0]), M.dtype_from_letter(label[1]), M.dtype_from_letter(label[2]), \
        (M.SINGLE if label[3] == "s" else M.DOUBLE)


ALL_LABELS = [l.str() for l in M.CaseLabel.all()]


class Problem:
    """One seeded gemm problem in the conformance harness's style
    (conformance.cpp:46-60): A is m x k (or k x m transposed), B k x n (or
    n x k), C m x n with the requested storage kind."""

    def __init__(self, label: str, m: int, n: int, k: int, *, c_kind="col", trans_a=False, trans_b=False,
                 conj_a=False, conj_b=False, seed=42, variant="base", a_kind="col", b_kind="col"):
        self.label = label
        dc, da, db, comp = label_dtypes(label)
        self.comp = comp
        self.m, self.n, self.k = m, n, k
        self.trans_a, self.trans_b = trans_a, trans_b
        self.conj_a = conj_a and M.is_complex(da)
        self.conj_b = conj_b and M.is_complex(db)
        root = O.orc_rng_state(seed, [label, variant, m * 1000003 + n * 1009 + k])
        self.A = HostMatrix(da, k if trans_a else m, m if trans_a else k, a_kind).fill(O.orc.orc_rng_split_tag(root, b"a"))
        self.B = HostMatrix(db, n if trans_b else k, k if trans_b else n, b_kind).fill(O.orc.orc_rng_split_tag(root, b"b"))
        self.C = HostMatrix(dc, m, n, c_kind).fill(O.orc.orc_rng_split_tag(root, b"c"))

    def views(self, A=None, B=None, C=None):
        A, B, C = A or self.A, B or self.B, C or self.C
        va = A.tview(conj=self.conj_a) if self.trans_a else A.view(conj=self.conj_a)
        vb = B.tview(conj=self.conj_b) if self.trans_b else B.view(conj=self.conj_b)
        vc = C.view(comp=self.comp)
        return va, vb, vc

    def device(self):
        return self.A.to_device(), self.B.to_device(), self.C.to_device()


def cfg(**kv) -> M.Config:
    c = M.Config.defaults()
    for key, val in kv.items():
        c.set(key.replace("_", ".", 1) if "." not in key else key, val)
    return c


def config(pairs: dict | None = None) -> M.Config:
    c = M.Config.defaults()
    for key, val in (pairs or {}).items():
        c.set(key, val)
    return c


EPS = {M.SINGLE: 2.0 ** -24, M.DOUBLE: 2.0 ** -53}


def frob_bound(label: str, k: int) -> float:
    """North-star C bound (BASELINE.json): relative Frobenius error <= 4 k eps of
    the computation precision; + eps of C's storage precision when that is
    narrower (a reordered sum legitimately flips some of its roundings,
    SURVEY 8(d))."""
    dc, _, _, comp = label_dtypes(label)
    bound = 4 * k * EPS[comp]
    if M.precision_of(dc) != comp:
        bound += EPS[M.precision_of(dc)]
    return bound


def rel_frobenius(got: np.ndarray, want: np.ndarray) -> float:
    g = got.astype(np.complex128)
    w = want.astype(np.complex128)
    den = np.linalg.norm(w)
    num = np.linalg.norm(g - w)
    return float(num / den) if den > 0 else float(num)


def ulp_distance(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Per-component distance in units of the storage precision's ulp."""
    got, want = np.ascontiguousarray(got), np.ascontiguousarray(want)
    g = got.view(np.float32 if got.dtype in (np.float32, np.complex64) else np.float64)
    w = want.view(g.dtype)
    itype = np.int32 if g.dtype == np.float32 else np.int64
    gi, wi = g.view(itype).astype(np.int64), w.view(itype).astype(np.int64)
    # map sign-magnitude to a monotone integer line
    big = np.int64(1) << (31 if itype is np.int32 else 63)
    gi = np.where(gi < 0, -(gi & (big - 1)) if itype is np.int32 else -(gi ^ np.int64(-(2**63))), gi)
    wi = np.where(wi < 0, -(wi & (big - 1)) if itype is np.int32 else -(wi ^ np.int64(-(2**63))), wi)
    return np.abs(gi - wi)


SCALARS = {
    "one": Scalar.real_value(1.0),
    "zero": Scalar.real_value(0.0),
    "minus_one": Scalar.real_value(-1.0),
    "p7": Scalar.real_value(0.7),
    "m3": Scalar.real_value(-0.3),
    "p3": Scalar.real_value(0.3),
    "c34": Scalar.complex_value(0.3, 0.4),
    "c55": Scalar.complex_value(0.5, 0.5),
    "cfg2_alpha": Scalar.complex_value(1.2, -0.7),
    "cfg2_alpha_real": Scalar.real_value(1.2),
    "cfg2_beta": Scalar.complex_value(0.9, 0.3),
    "cfg3_alpha": Scalar.complex_value(0.5, 1.5),
}
