"""paper_1901_06015_b200 -- B200-native mixed-datatype gemm (arXiv 1901.06015).

Python mirror of the reference engine's public API (mdgemm::gemm, plan,
MatrixView, Scalar, Config; /root/reference/proj/include/mdgemm/*.hpp) over
the C ABI in include/mdgemm_b200.h.  The compute runs only in the sm_100a
library libmdgemm_b200.so built in-tree by __graft_entry__.build(); if that
library is missing, importing this package fails -- there is no CPU path.

Views hold raw pointers.  Device pointers are used in place; host pointers
(numpy buffers) are staged through HBM by gemm().
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

__all__ = [
    "Error", "ScalarPolicyError", "CudaError", "lib", "MatrixView", "Scalar", "Config", "ExecutionPlan",
    "plan", "gemm", "gemm_batch", "gemm_async", "execute", "pack_block_device", "packed_bytes", "fill_uniform", "fill_normal",
    "Rng", "Comm", "comm_unique_id", "gemm_sharded", "gemm_multi", "classify_case", "flops_of_case", "apply_scalar_policy", "shard_columns", "CaseLabel",
    "DT_S", "DT_D", "DT_C", "DT_Z", "SINGLE", "DOUBLE", "LEFT", "RIGHT", "STANDARD", "ONE_E", "ONE_R",
    "FAST", "EXACT", "dtype_from_letter", "dtype_letter", "dtype_size", "is_complex", "precision_of",
    "CASE_NAMES",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# MDGEMM_LIBRARY=checked loads the build with device-side index checks
# (make -C paper_1901_06015_b200/csrc checked; tests only)
# (or the path of another build of the library: A/B experiments)
_LIB_ENV = os.environ.get("MDGEMM_LIBRARY", "")
_LIB_PATH = (os.path.join(_HERE, "libmdgemm_b200_checked.so") if _LIB_ENV == "checked"
             else _LIB_ENV if _LIB_ENV.endswith(".so") else os.path.join(_HERE, "libmdgemm_b200.so"))

# enumerations (mdgemm_b200.h)
DT_S, DT_D, DT_C, DT_Z = 0, 1, 2, 3
SINGLE, DOUBLE = 0, 1
LEFT, RIGHT = 0, 1
STANDARD, ONE_E, ONE_R = 0, 1, 2
PREF_COLUMN, PREF_ROW = 0, 1
PAIR_NONE, PAIR_ROWS, PAIR_COLS = 0, 1, 2
PATH_DIRECT, PATH_TEMP, PATH_ONEM_COLUMN, PATH_ONEM_ROW = 0, 1, 2, 3
CTEMP_AUTO, CTEMP_ON, CTEMP_OFF = 0, 1, 2
FAST, EXACT = 0, 1
OK, ERR, ERR_SCALAR_POLICY, ERR_CUDA = 0, 1, 2, 3
CASE_NAMES = ["0", "1a", "1b", "1c", "2ab", "2ac", "2bc", "3"]

_LETTERS = "sdcz"


def dtype_from_letter(ch: str) -> int:
    if len(ch) != 1 or ch not in _LETTERS:
        raise Error(f"unknown datatype letter '{ch}'")
    return _LETTERS.index(ch)


def dtype_letter(dt: int) -> str:
    return _LETTERS[dt]


def is_complex(dt: int) -> bool:
    return dt in (DT_C, DT_Z)


def precision_of(dt: int) -> int:
    return SINGLE if dt in (DT_S, DT_C) else DOUBLE


def dtype_size(dt: int) -> int:
    return (4 if precision_of(dt) == SINGLE else 8) * (2 if is_complex(dt) else 1)


class Error(RuntimeError):
    """mdgemm::Error (dtypes.hpp:14-16)."""


class ScalarPolicyError(Error):
    """mdgemm::ScalarPolicyError (dtypes.hpp:18-20)."""


class CudaError(Error):
    """A CUDA runtime failure inside the library."""


# ---------------------------------------------------------------- structs
class MatrixView(ctypes.Structure):
    _fields_ = [("base", c_void_p), ("m", c_int64), ("n", c_int64), ("rs", c_int64), ("cs", c_int64),
                ("dtype", c_int32), ("conj", c_int32), ("comp_prec", c_int32), ("target_dtype", c_int32)]

    @staticmethod
    def make(base: int, m: int, n: int, rs: int, cs: int, dtype: int) -> "MatrixView":
        out = MatrixView()
        _check(lib.mdg_view_make(c_void_p(base), m, n, rs, cs, dtype, byref(out)))
        return out

    def with_conj(self, c: bool = True) -> "MatrixView":
        v = MatrixView.from_buffer_copy(self)
        v.conj = int(bool(c))
        return v

    def with_comp_prec(self, p: int) -> "MatrixView":
        v = MatrixView.from_buffer_copy(self)
        v.comp_prec = p
        return v

    def copy(self) -> "MatrixView":
        return MatrixView.from_buffer_copy(self)

    def __repr__(self):
        return (f"MatrixView({self.m}x{self.n} {dtype_letter(self.dtype)} rs={self.rs} cs={self.cs} "
                f"conj={self.conj} comp={'sd'[self.comp_prec]} base=0x{(self.base or 0):x})")


class Scalar(ctypes.Structure):
    _fields_ = [("re", c_double), ("im", c_double), ("dtype", c_int32), ("reserved", c_int32)]

    @staticmethod
    def real_value(v: float, prec: int = DOUBLE) -> "Scalar":
        return Scalar(_round(v, prec), 0.0, DT_S if prec == SINGLE else DT_D, 0)

    @staticmethod
    def complex_value(re: float, im: float, prec: int = DOUBLE) -> "Scalar":
        return Scalar(_round(re, prec), _round(im, prec), DT_C if prec == SINGLE else DT_Z, 0)

    def is_zero(self) -> bool:
        return self.re == 0.0 and self.im == 0.0

    def is_one(self) -> bool:
        return self.re == 1.0 and self.im == 0.0

    def value(self) -> complex:
        return complex(self.re, self.im)

    def __repr__(self):
        return f"Scalar({self.re}{self.im:+}i, {dtype_letter(self.dtype)})"


class _Blocking(ctypes.Structure):
    _fields_ = [("mc", c_int64), ("nc", c_int64), ("kc", c_int64), ("mr", c_int32), ("nr", c_int32)]


class Config(ctypes.Structure):
    """Config (config.hpp:38-72) plus gpu.numerics = fast | exact."""
    _fields_ = [("single_params", _Blocking), ("double_params", _Blocking), ("threads", c_int32),
                ("preference", c_int32), ("ctemp", c_int32), ("numerics", c_int32),
                ("splitk", c_int32), ("reserved", c_int32)]

    @staticmethod
    def defaults() -> "Config":
        out = Config()
        _check(lib.mdg_config_defaults(byref(out)))
        return out

    @staticmethod
    def load(path: str | None = None, apply_env: bool = True) -> "Config":
        out = Config()
        _check(lib.mdg_config_load(byref(out), path.encode() if path else None, int(apply_env)))
        return out

    def set(self, key: str, value) -> "Config":
        _check(lib.mdg_config_set(byref(self), str(key).encode(), str(value).encode()))
        return self

    def validate(self) -> None:
        _check(lib.mdg_config_validate(byref(self)))

    @staticmethod
    def with_(**kv) -> "Config":
        cfg = Config.defaults()
        for k, v in kv.items():
            cfg.set(k.replace("__", "."), v)
        return cfg


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
        ("params", _Blocking), ("threads", c_int32),
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
            elif isinstance(v, _Blocking):
                for f, _ in _Blocking._fields_:
                    out[f"{name}.{f}"] = getattr(v, f)
            else:
                out[name] = v
        if not self.has_ctemp:
            for f in ("ctemp_rows", "ctemp_cols", "ctemp_precision", "ctemp_mode"):
                out[f] = 0
        return out


class GemmCall(ctypes.Structure):
    """One element of gemm_batch(): C := beta*C + alpha*A*B."""
    _fields_ = [("alpha", Scalar), ("a", MatrixView), ("b", MatrixView), ("beta", Scalar), ("c", MatrixView)]


class KernelStats(ctypes.Structure):
    _fields_ = [("launches", c_uint64), ("total_ms", c_double), ("work", c_double)]


KERNEL_KINDS = ("pack", "dmma", "ffma", "exact", "beta", "fill", "dual_d", "dual_f")


def _round(v: float, prec: int) -> float:
    if prec == SINGLE:
        import struct
        return struct.unpack("f", struct.pack("f", v))[0]
    return float(v)


# ------------------------------------------------------------------ loading
def _load() -> ctypes.CDLL:
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    V, S, C, P = POINTER(MatrixView), Scalar, POINTER(Config), POINTER(ExecutionPlan)
    sig = {
        "mdg_abi_version": (c_int, []),
        "mdg_last_error": (c_char_p, []),
        "mdg_config_defaults": (c_int, [C]),
        "mdg_config_set": (c_int, [C, c_char_p, c_char_p]),
        "mdg_config_load": (c_int, [C, c_char_p, c_int]),
        "mdg_config_validate": (c_int, [C]),
        "mdg_view_make": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int32, V]),
        "mdg_classify_case": (c_int32, [c_int32, c_int32, c_int32]),
        "mdg_flops_of_case": (c_uint64, [c_int32, c_int64, c_int64, c_int64]),
        "mdg_apply_scalar_policy": (c_int, [S, S, c_int32, c_int32, c_int32, POINTER(Scalar), POINTER(Scalar)]),
        "mdg_plan": (c_int, [S, V, V, S, V, C, P]),
        "mdg_execute": (c_int, [P, c_int32, c_void_p, POINTER(c_uint64)]),
        "mdg_gemm": (c_int, [S, V, V, S, V, C, POINTER(c_uint64)]),
        "mdg_gemm_async": (c_int, [S, V, V, S, V, C, c_void_p, POINTER(c_uint64)]),
        "mdg_gemm_batch": (c_int, [c_int32, POINTER(GemmCall), C, POINTER(c_uint64)]),
        "mdg_gemm_batch_async": (c_int, [c_int32, POINTER(GemmCall), C, c_void_p, POINTER(c_uint64)]),
        "mdg_dual_schedule": (c_int, [c_int32, POINTER(GemmCall), C, c_int32, POINTER(c_int32), POINTER(c_int32),
                                      POINTER(c_int32)]),
        "mdg_packed_bytes": (c_size_t, [V, c_int32, c_int32, c_int32, c_int64, c_int64]),
        "mdg_pack_operand": (c_int, [V, c_int32, c_int32, c_int32, S, c_int32, c_int64, c_int64, c_void_p, c_void_p]),
        "mdg_fill_uniform": (c_int, [V, c_uint64, c_void_p]),
        "mdg_fill_normal": (c_int, [V, c_uint64, c_void_p]),
        "mdg_rng_split_tag": (c_uint64, [c_uint64, c_char_p]),
        "mdg_rng_split_salt": (c_uint64, [c_uint64, c_uint64]),
        "mdg_shard_columns": (c_int, [c_int64, c_int32, c_int32, c_int64, POINTER(c_int64), POINTER(c_int64)]),
        "mdg_trim_workspace": (c_int, [c_uint64]),
        "mdg_comm_unique_id": (c_int, [ctypes.c_char_p]),
        "mdg_comm_init": (c_int, [ctypes.c_char_p, c_int32, c_int32, POINTER(c_void_p)]),
        "mdg_comm_destroy": (c_int, [c_void_p]),
        "mdg_gemm_sharded": (c_int, [c_void_p, c_int32, S, V, V, S, V, C, c_void_p, POINTER(c_uint64)]),
        "mdg_gemm_multi": (c_int, [S, V, V, S, V, C, c_int32, POINTER(c_int32), POINTER(c_uint64)]),
        "mdg_launch_count": (c_uint64, []),
        "mdg_staging_bytes": (None, [POINTER(c_uint64), POINTER(c_uint64)]),
        "mdg_profile_begin": (c_int, []),
        "mdg_profile_end": (c_int, [POINTER(KernelStats)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


lib = _load()
EXPORTED_SYMBOLS = (
    "mdg_abi_version", "mdg_last_error", "mdg_config_defaults", "mdg_config_set", "mdg_config_load",
    "mdg_config_validate", "mdg_view_make", "mdg_classify_case", "mdg_flops_of_case", "mdg_apply_scalar_policy",
    "mdg_plan", "mdg_execute", "mdg_gemm", "mdg_gemm_batch", "mdg_gemm_batch_async", "mdg_gemm_async",
    "mdg_dual_schedule",
    "mdg_packed_bytes", "mdg_pack_operand",
    "mdg_fill_uniform", "mdg_fill_normal", "mdg_rng_split_tag", "mdg_rng_split_salt", "mdg_shard_columns",
    "mdg_comm_unique_id", "mdg_comm_init", "mdg_comm_destroy", "mdg_gemm_sharded", "mdg_gemm_multi",
    "mdg_trim_workspace", "mdg_launch_count", "mdg_staging_bytes", "mdg_profile_begin", "mdg_profile_end",
)


def launch_count() -> int:
    """Kernels this process has launched through the library."""
    return lib.mdg_launch_count()


def trim_workspace(keep_bytes: int = 0) -> None:
    """Synchronise the device and give the library pool's cached workspace
    above keep_bytes back to the system."""
    _check(lib.mdg_trim_workspace(keep_bytes))


def staging_bytes() -> tuple[int, int]:
    """(host->device, device->host) bytes the batch runner has copied so far."""
    h2d, d2h = c_uint64(0), c_uint64(0)
    lib.mdg_staging_bytes(byref(h2d), byref(d2h))
    return h2d.value, d2h.value


def profile_begin() -> None:
    _check(lib.mdg_profile_begin())


def profile_end() -> dict:
    """{kind: {'launches', 'ms', 'work'}} for the kernels launched on this
    thread since profile_begin(); work = flops (gemm) or bytes (pack/beta/fill)."""
    out = (KernelStats * len(KERNEL_KINDS))()
    _check(lib.mdg_profile_end(out))
    return {k: {"launches": s.launches, "ms": s.total_ms, "work": s.work} for k, s in zip(KERNEL_KINDS, out)}


def _check(rc: int) -> None:
    if rc == OK:
        return
    msg = (lib.mdg_last_error() or b"").decode(errors="replace")
    if rc == ERR_SCALAR_POLICY:
        raise ScalarPolicyError(msg)
    if rc == ERR_CUDA:
        raise CudaError(msg)
    raise Error(msg)


def _stream_ptr(stream) -> c_void_p:
    if stream is None:
        return c_void_p(None)
    if hasattr(stream, "cuda_stream"):  # torch.cuda.Stream
        return c_void_p(stream.cuda_stream)
    return c_void_p(int(stream))


# ---------------------------------------------------------------- the API
def classify_case(c_complex: bool, a_complex: bool, b_complex: bool) -> int:
    return lib.mdg_classify_case(int(c_complex), int(a_complex), int(b_complex))


def flops_of_case(case_id: int, m: int, n: int, k: int) -> int:
    return lib.mdg_flops_of_case(case_id, m, n, k)


def apply_scalar_policy(alpha: Scalar, beta: Scalar, case_id: int, comp_prec: int, c_storage_prec: int):
    a, b = Scalar(), Scalar()
    _check(lib.mdg_apply_scalar_policy(alpha, beta, case_id, comp_prec, c_storage_prec, byref(a), byref(b)))
    return a, b


def plan(alpha: Scalar, a: MatrixView, b: MatrixView, beta: Scalar, c: MatrixView,
         cfg: Config | None = None) -> ExecutionPlan:
    out = ExecutionPlan()
    _check(lib.mdg_plan(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or Config.defaults()), byref(out)))
    return out


def gemm(alpha: Scalar, a: MatrixView, b: MatrixView, beta: Scalar, c: MatrixView,
         cfg: Config | None = None) -> int:
    """C := beta*C + alpha*A*B (dispatch.hpp:89-91).  Synchronous; returns the FlopCounter value."""
    flops = c_uint64(0)
    _check(lib.mdg_gemm(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or Config.defaults()), byref(flops)))
    return flops.value


def gemm_batch(calls, cfg: Config | None = None, stream=None, sync: bool = True) -> int:
    """gemm() calls [(alpha, a, b, beta, c), ...] with the semantics of calling
    them in order; host staging is pipelined and calls that do not touch each
    other's memory run concurrently.  sync=False forks from / joins into
    `stream` without waiting.  Returns the FlopCounter total."""
    arr = (GemmCall * max(len(calls), 1))(*[GemmCall(al, a, b, be, c) for al, a, b, be, c in calls])
    flops = c_uint64(0)
    if sync:
        _check(lib.mdg_gemm_batch(len(calls), arr, byref(cfg or Config.defaults()), byref(flops)))
    else:
        _check(lib.mdg_gemm_batch_async(len(calls), arr, byref(cfg or Config.defaults()), _stream_ptr(stream),
                                        byref(flops)))
    return flops.value


def dual_schedule(calls, cfg: Config | None = None):
    """The dual-pipe launch schedule gemm_batch would use for `calls`, computed on the
    host without a device: ([(launch, call, tile_begin, tile_end, group), ...], tiles per
    call); group 1 = FP64 job, 2 = FP32 job, 0 = the call runs through execute().
    Empty when the batch would not take the dual path."""
    n = len(calls)
    arr = (GemmCall * max(n, 1))(*[GemmCall(al, a, b, be, c) for al, a, b, be, c in calls])
    cap = 4 * max(n, 1) + 64
    while True:
        pieces = (c_int32 * (5 * cap))()
        tiles = (c_int32 * max(n, 1))()
        count = c_int32(0)
        _check(lib.mdg_dual_schedule(n, arr, byref(cfg or Config.defaults()), cap, pieces, byref(count), tiles))
        if count.value <= cap:
            break
        cap = count.value
    out = [tuple(pieces[5 * x:5 * x + 5]) for x in range(count.value)]
    return out, list(tiles[:n])


def gemm_async(alpha: Scalar, a: MatrixView, b: MatrixView, beta: Scalar, c: MatrixView,
               cfg: Config | None = None, stream=None) -> int:
    """Device operands only; ordered on `stream` (torch.cuda.Stream, raw handle or None)."""
    flops = c_uint64(0)
    _check(lib.mdg_gemm_async(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or Config.defaults()),
                              _stream_ptr(stream), byref(flops)))
    return flops.value


def execute(p: ExecutionPlan, numerics: int = FAST, stream=None) -> int:
    flops = c_uint64(0)
    _check(lib.mdg_execute(byref(p), numerics, _stream_ptr(stream), byref(flops)))
    return flops.value


def packed_bytes(src: MatrixView, side: int, fmt: int, target: int, reg_block: int, panel_len: int = 0) -> int:
    n = lib.mdg_packed_bytes(byref(src), side, fmt, target, reg_block, panel_len)
    if n == 0 and src.m * src.n > 0:
        _check(ERR)
    return n


def pack_block_device(dst: int, src: MatrixView, side: int, fmt: int, conj: bool, scale: Scalar, target: int,
                      reg_block: int, panel_len: int = 0, stream=None) -> None:
    _check(lib.mdg_pack_operand(byref(src), side, fmt, int(conj), scale, target, reg_block, panel_len,
                                c_void_p(dst), _stream_ptr(stream)))


def fill_uniform(v: MatrixView, state: int, stream=None) -> None:
    _check(lib.mdg_fill_uniform(byref(v), c_uint64(state), _stream_ptr(stream)))


def fill_normal(v: MatrixView, state: int, stream=None) -> None:
    """normal(0,1) entries by Box-Muller over the reference Rng's draws (mdg_fill_normal)."""
    _check(lib.mdg_fill_normal(byref(v), c_uint64(state), _stream_ptr(stream)))


def shard_columns(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    j0, nb = c_int64(0), c_int64(0)
    _check(lib.mdg_shard_columns(n, world, rank, align, byref(j0), byref(nb)))
    return j0.value, nb.value


COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    """A fresh communicator id (on one rank; share the bytes with the others)."""
    buf = ctypes.create_string_buffer(COMM_ID_BYTES)
    _check(lib.mdg_comm_unique_id(buf))
    return buf.raw


class Comm:
    """One process per GPU: the library's NCCL communicator on the current device (mdg_comm_init).
    Collective: every rank constructs it with the same id."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        if len(uid) != COMM_ID_BYTES:
            raise Error("Comm: the id must be 128 bytes")
        self.handle = c_void_p()
        _check(lib.mdg_comm_init(uid, nranks, rank, byref(self.handle)))
        self.nranks, self.rank = nranks, rank

    def close(self) -> None:
        if self.handle:
            _check(lib.mdg_comm_destroy(self.handle))
            self.handle = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def gemm_sharded(comm: Comm, root: int, alpha: Scalar, a: MatrixView, b_panel: MatrixView, beta: Scalar,
                 c_panel: MatrixView, cfg: Config | None = None, stream=None) -> int:
    """This rank's column panel (mdg_gemm_sharded): A broadcast from `root` over the communicator
    (a.base = 0 on other ranks: the library receives it), B / C panels on this rank's device."""
    flops = c_uint64(0)
    _check(lib.mdg_gemm_sharded(comm.handle, root, alpha, byref(a), byref(b_panel), beta, byref(c_panel),
                                byref(cfg or Config.defaults()), _stream_ptr(stream), byref(flops)))
    return flops.value


def gemm_multi(alpha: Scalar, a: MatrixView, b: MatrixView, beta: Scalar, c: MatrixView, cfg: Config | None = None,
               devices=None) -> int:
    """The whole call over several GPUs of this process (mdg_gemm_multi), synchronous."""
    import torch
    devs = list(devices) if devices is not None else list(range(torch.cuda.device_count()))
    arr = (c_int32 * len(devs))(*devs)
    flops = c_uint64(0)
    _check(lib.mdg_gemm_multi(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or Config.defaults()), len(devs),
                              arr, byref(flops)))
    return flops.value


class Rng:
    """The reference's counter-based splitmix64 Rng (rng.hpp:13-45): only the
    state and the split rules; draws happen in fill_uniform."""

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFFFFFFFFFF

    def split(self, tag) -> "Rng":
        if isinstance(tag, str):
            return Rng(lib.mdg_rng_split_tag(self.state, tag.encode()))
        return Rng(lib.mdg_rng_split_salt(self.state, int(tag) & 0xFFFFFFFFFFFFFFFF))


class CaseLabel:
    """Four-letter label: C, A, B storage datatypes then computation precision (case_label.hpp)."""

    def __init__(self, c: int, a: int, b: int, comp: int):
        self.c, self.a, self.b, self.comp = c, a, b, comp

    @staticmethod
    def parse(s: str) -> "CaseLabel":
        if len(s) != 4:
            raise Error(f"case label '{s}' must have exactly four letters")
        if s[3] not in "sd":
            raise Error(f"unknown precision letter '{s[3]}'")
        return CaseLabel(dtype_from_letter(s[0]), dtype_from_letter(s[1]), dtype_from_letter(s[2]),
                         SINGLE if s[3] == "s" else DOUBLE)

    @staticmethod
    def all() -> list["CaseLabel"]:
        return [CaseLabel(c, a, b, p) for c in range(4) for a in range(4) for b in range(4) for p in (SINGLE, DOUBLE)]

    def str(self) -> str:
        return _LETTERS[self.c] + _LETTERS[self.a] + _LETTERS[self.b] + "sd"[self.comp]

    def case_id(self) -> int:
        return classify_case(is_complex(self.c), is_complex(self.a), is_complex(self.b))

    def __repr__(self):
        return f"CaseLabel({self.str()})"
