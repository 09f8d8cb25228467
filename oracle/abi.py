"""TEST INFRASTRUCTURE ONLY: ctypes mirror of the plain-data structs and
enumerations of include/mdgemm_b200.h, for the CPU checkers.

The oracle libraries (oracle/_build/libmdg_oracle.so, oracle/_ref/
libmdgemm_ref.so) take the same structs as the product ABI.  This module
declares them without importing the product package, so that the reference
arm of bench.py and the CPU baseline load nothing of the B200 library.
Layouts must match include/mdgemm_b200.h (tests/test_abi.py checks the sizes
against the product's ctypes mirror).
"""
from __future__ import annotations

import ctypes
from ctypes import c_double, c_int32, c_int64, c_void_p

DT_S, DT_D, DT_C, DT_Z = 0, 1, 2, 3
SINGLE, DOUBLE = 0, 1
LEFT, RIGHT = 0, 1
STANDARD, ONE_E, ONE_R = 0, 1, 2
PREF_COLUMN, PREF_ROW = 0, 1
CTEMP_AUTO, CTEMP_ON, CTEMP_OFF = 0, 1, 2
OK, ERR, ERR_SCALAR_POLICY, ERR_CUDA = 0, 1, 2, 3
CASE_NAMES = ["0", "1a", "1b", "1c", "2ab", "2ac", "2bc", "3"]
_LETTERS = "sdcz"


class Error(RuntimeError):
    """mdgemm::Error raised by a checker library (dtypes.hpp:14-16)."""


class ScalarPolicyError(Error):
    """mdgemm::ScalarPolicyError raised by a checker library (dtypes.hpp:18-20)."""


def dtype_from_letter(ch: str) -> int:
    return _LETTERS.index(ch)


def dtype_size(dt: int) -> int:
    return (4 if dt in (DT_S, DT_C) else 8) * (2 if dt in (DT_C, DT_Z) else 1)


def is_complex(dt: int) -> bool:
    return dt in (DT_C, DT_Z)


def case_id(label: str) -> int:
    """classify_case on the domains of a cabx label (dispatch.cpp:11-33)."""
    c, a, b = (is_complex(dtype_from_letter(ch)) for ch in label[:3])
    if not c and not a and not b:
        return 0
    if c and a and b:
        return 7
    if not c:
        return 1 if a and not b else 2 if b and not a else 4
    return 3 if not a and not b else 5 if a else 6


def all_labels() -> list[str]:
    """CaseLabel::all() (case_label.cpp:28-39): C, A, B over s d c z, then s d."""
    return [c + a + b + p for c in _LETTERS for a in _LETTERS for b in _LETTERS for p in "sd"]


def flops_of_case(cid: int, m: int, n: int, k: int) -> int:
    """dispatch.cpp:35-54: 2mnk (0, 1a, 1b, 1c), 4mnk (2ab, 2ac, 2bc), 8mnk (3)."""
    return (2 if cid <= 3 else 4 if cid <= 6 else 8) * m * n * k


class MatrixView(ctypes.Structure):
    _fields_ = [("base", c_void_p), ("m", c_int64), ("n", c_int64), ("rs", c_int64), ("cs", c_int64),
                ("dtype", c_int32), ("conj", c_int32), ("comp_prec", c_int32), ("target_dtype", c_int32)]


class Scalar(ctypes.Structure):
    _fields_ = [("re", c_double), ("im", c_double), ("dtype", c_int32), ("reserved", c_int32)]

    @staticmethod
    def real_value(v: float) -> "Scalar":
        return Scalar(float(v), 0.0, DT_D, 0)

    @staticmethod
    def complex_value(re: float, im: float) -> "Scalar":
        return Scalar(float(re), float(im), DT_Z, 0)


class Blocking(ctypes.Structure):
    _fields_ = [("mc", c_int64), ("nc", c_int64), ("kc", c_int64), ("mr", c_int32), ("nr", c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("single_params", Blocking), ("double_params", Blocking), ("threads", c_int32),
                ("preference", c_int32), ("ctemp", c_int32), ("numerics", c_int32),
                ("splitk", c_int32), ("reserved", c_int32)]


class ExecutionPlan(ctypes.Structure):
    _fields_ = [
        ("case_id", c_int32), ("logical_transpose", c_int32), ("comp_prec", c_int32), ("reserved0", c_int32),
        ("m", c_int64), ("n", c_int64), ("k", c_int64),
        ("a", MatrixView), ("b", MatrixView), ("c", MatrixView),
        ("format_a", c_int32), ("format_b", c_int32), ("conj_a", c_int32), ("conj_b", c_int32),
        ("target_dtype_a", c_int32), ("target_dtype_b", c_int32),
        ("reg_block_a", c_int64), ("reg_block_b", c_int64),
        ("alpha", Scalar), ("beta", Scalar), ("pack_scale_a", Scalar), ("pack_scale_b", Scalar),
        ("macro_mode", c_int32), ("ukr_path", c_int32), ("pair_axis", c_int32), ("has_ctemp", c_int32),
        ("ctemp_rows", c_int64), ("ctemp_cols", c_int64), ("ctemp_precision", c_int32), ("ctemp_mode", c_int32),
        ("params", Blocking), ("threads", c_int32),
        ("ukr_precision", c_int32), ("ukr_mr", c_int32), ("ukr_nr", c_int32), ("ukr_preference", c_int32),
        ("reserved1", c_int32),
    ]

    def as_dict(self, with_pointers: bool = False) -> dict:
        """Field-by-field contents (views and scalars flattened) for comparisons."""
        out = {}
        for name, _ in self._fields_:
            if name.startswith("reserved"):
                continue
            v = getattr(self, name)
            if isinstance(v, MatrixView):
                for f, _ in MatrixView._fields_:
                    if f == "base" and not with_pointers:
                        continue
                    out[f"{name}.{f}"] = getattr(v, f)
            elif isinstance(v, Scalar):
                out[f"{name}.re"], out[f"{name}.im"], out[f"{name}.dtype"] = v.re, v.im, v.dtype
            elif isinstance(v, Blocking):
                for f, _ in Blocking._fields_:
                    out[f"{name}.{f}"] = getattr(v, f)
            else:
                out[name] = v
        if not self.has_ctemp:
            for f in ("ctemp_rows", "ctemp_cols", "ctemp_precision", "ctemp_mode"):
                out[f] = 0
        return out


def convert(T, obj):
    """obj as the checker's struct type T (a byte copy of a same-layout struct
    from the product's ctypes mirror); None stays None."""
    if obj is None or isinstance(obj, T):
        return obj
    if ctypes.sizeof(obj) != ctypes.sizeof(T):
        raise TypeError(f"{type(obj).__name__} does not have the layout of {T.__name__}")
    return T.from_buffer_copy(obj)


class HostMatrix:
    """A column-major host matrix (numpy buffer) and its view, for the CPU
    checkers and the reference arm (Matrix::make, matrix.hpp:17-43)."""

    def __init__(self, dtype: int, m: int, n: int):
        import numpy as np
        self.dtype, self.m, self.n = dtype, m, n
        self.buf = np.zeros(max(m * n, 1) * dtype_size(dtype), np.uint8)

    def view(self, comp: int | None = None) -> MatrixView:
        v = MatrixView(self.buf.ctypes.data, self.m, self.n, 1, max(self.m, 1), self.dtype, 0,
                       (SINGLE if self.dtype in (DT_S, DT_C) else DOUBLE) if comp is None else comp,
                       self.dtype)
        return v
