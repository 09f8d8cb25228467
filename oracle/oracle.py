"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU checkers.

  * ``orc``  -- oracle/_build/libmdg_oracle.so, the C restatement (mdg_oracle.c)
  * ``ref``  -- oracle/_ref/libmdgemm_ref.so, the reference engine compiled from
                its own sources (oracle/Makefile); absent if it was never built.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker.  Both libraries take HOST
pointers and the same plain-data structs as the product ABI; the structs are
declared in oracle/abi.py (this module never imports the product package),
and the wrappers below accept the product's same-layout ctypes structs too.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

from oracle.abi import (ERR_SCALAR_POLICY, OK, Config, Error, ExecutionPlan, MatrixView, Scalar, ScalarPolicyError,
                        convert)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmdg_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmdgemm_ref.so")

V, S, C, P = POINTER(MatrixView), Scalar, POINTER(Config), POINTER(ExecutionPlan)


def _bind(lib, sig):
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


def _load_orc():
    if not os.path.exists(ORACLE_SO):
        raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle oracle`")
    return _bind(ctypes.CDLL(ORACLE_SO), {
        "orc_last_error": (c_char_p, []),
        "orc_rng_split_tag": (c_uint64, [c_uint64, c_char_p]),
        "orc_rng_split_salt": (c_uint64, [c_uint64, c_uint64]),
        "orc_fill_uniform": (c_int, [V, c_uint64]),
        "orc_config_defaults": (c_int, [C]),
        "orc_config_validate": (c_int, [C]),
        "orc_classify_case": (c_int32, [c_int32, c_int32, c_int32]),
        "orc_flops_of_case": (c_uint64, [c_int32, c_int64, c_int64, c_int64]),
        "orc_plan": (c_int, [S, V, V, S, V, C, P]),
        "orc_packed_bytes": (c_size_t, [V, c_int32, c_int32, c_int32, c_int64, c_int64]),
        "orc_pack": (c_int, [V, c_int32, c_int32, c_int32, S, c_int32, c_int64, c_int64, c_void_p]),
        "orc_gemm": (c_int, [S, V, V, S, V, C, POINTER(c_uint64)]),
        "orc_oracle_gemm": (c_int, [S, V, V, S, V, c_int32, c_void_p]),
        "orc_violation": (c_int, [S, V, V, S, V, V, c_int32, POINTER(c_double)]),
    })


def _load_ref():
    if not os.path.exists(REF_SO):
        return None
    return _bind(ctypes.CDLL(REF_SO), {
        "ref_last_error": (c_char_p, []),
        "ref_config_defaults": (c_int, [C]),
        "ref_plan": (c_int, [S, V, V, S, V, C, P]),
        "ref_gemm": (c_int, [S, V, V, S, V, C, POINTER(c_uint64)]),
        "ref_packed_bytes": (c_size_t, [V, c_int32, c_int32, c_int32, c_int64]),
        "ref_pack": (c_int, [V, c_int32, c_int32, c_int32, S, c_int32, c_int64, c_void_p, c_size_t]),
        "ref_oracle_gemm": (c_int, [S, V, V, S, V, c_int32, c_void_p, c_size_t]),
        "ref_violation": (c_int, [S, V, V, S, V, V, c_int32, POINTER(c_double)]),
        "ref_fill_uniform_path": (c_int, [V, c_uint64, POINTER(c_char_p), POINTER(c_uint64), c_int32]),
        "ref_run_bench": (c_int, [c_char_p, c_int64, c_int64, c_int64, c_int32, C, c_uint64,
                                  POINTER(c_double), POINTER(c_double)]),
        "ref_flops_of_case": (c_uint64, [c_int32, c_int64, c_int64, c_int64]),
    })


orc = _load_orc()
ref = _load_ref()


def _raise(rc: int, msg: bytes | None):
    text = (msg or b"").decode(errors="replace")
    if rc == ERR_SCALAR_POLICY:
        raise ScalarPolicyError(text)
    raise Error(text)


def check_orc(rc: int) -> None:
    if rc != OK:
        _raise(rc, orc.orc_last_error())


def check_ref(rc: int) -> None:
    if rc != OK:
        _raise(rc, ref.ref_last_error())


# ------------------------------------------------------------ convenience
def _args(alpha, a, b, beta, c, cfg):
    return (convert(Scalar, alpha), convert(MatrixView, a), convert(MatrixView, b), convert(Scalar, beta),
            convert(MatrixView, c), convert(Config, cfg))


def ref_config_defaults() -> Config:
    out = Config()
    check_ref(ref.ref_config_defaults(byref(out)))
    return out


def orc_config_defaults() -> Config:
    out = Config()
    check_orc(orc.orc_config_defaults(byref(out)))
    return out


def orc_plan(alpha, a, b, beta, c, cfg=None) -> ExecutionPlan:
    alpha, a, b, beta, c, cfg = _args(alpha, a, b, beta, c, cfg)
    out = ExecutionPlan()
    check_orc(orc.orc_plan(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or orc_config_defaults()), byref(out)))
    return out


def ref_plan(alpha, a, b, beta, c, cfg=None) -> ExecutionPlan:
    alpha, a, b, beta, c, cfg = _args(alpha, a, b, beta, c, cfg)
    out = ExecutionPlan()
    check_ref(ref.ref_plan(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or orc_config_defaults()), byref(out)))
    return out


def orc_gemm(alpha, a, b, beta, c, cfg=None) -> int:
    alpha, a, b, beta, c, cfg = _args(alpha, a, b, beta, c, cfg)
    flops = c_uint64(0)
    check_orc(orc.orc_gemm(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or orc_config_defaults()), byref(flops)))
    return flops.value


def ref_gemm(alpha, a, b, beta, c, cfg=None) -> int:
    alpha, a, b, beta, c, cfg = _args(alpha, a, b, beta, c, cfg)
    flops = c_uint64(0)
    check_ref(ref.ref_gemm(alpha, byref(a), byref(b), beta, byref(c), byref(cfg or orc_config_defaults()), byref(flops)))
    return flops.value


def orc_pack(src, side, fmt, conj, scale, target, reg_block, panel_len, dst_ptr) -> None:
    src, scale = convert(MatrixView, src), convert(Scalar, scale)
    check_orc(orc.orc_pack(byref(src), side, fmt, int(conj), scale, target, reg_block, panel_len, c_void_p(dst_ptr)))


def ref_pack(src, side, fmt, conj, scale, target, reg_block, dst_ptr, cap) -> None:
    src, scale = convert(MatrixView, src), convert(Scalar, scale)
    check_ref(ref.ref_pack(byref(src), side, fmt, int(conj), scale, target, reg_block, c_void_p(dst_ptr), cap))


def orc_packed_bytes(src, side, fmt, target, reg_block, panel_len=0) -> int:
    src = convert(MatrixView, src)
    return orc.orc_packed_bytes(byref(src), side, fmt, target, reg_block, panel_len)


def ref_packed_bytes(src, side, fmt, target, reg_block) -> int:
    return ref.ref_packed_bytes(byref(convert(MatrixView, src)), side, fmt, target, reg_block)


def orc_violation(alpha, a, b, beta, c_before, c_after, comp_prec) -> float:
    alpha, a, b, beta, c_before, _ = _args(alpha, a, b, beta, c_before, None)
    c_after = convert(MatrixView, c_after)
    v = c_double(0.0)
    check_orc(orc.orc_violation(alpha, byref(a), byref(b), beta, byref(c_before), byref(c_after), comp_prec, byref(v)))
    return v.value


def ref_violation(alpha, a, b, beta, c_before, c_after, comp_prec) -> float:
    alpha, a, b, beta, c_before, _ = _args(alpha, a, b, beta, c_before, None)
    c_after = convert(MatrixView, c_after)
    v = c_double(0.0)
    check_ref(ref.ref_violation(alpha, byref(a), byref(b), beta, byref(c_before), byref(c_after), comp_prec, byref(v)))
    return v.value


def orc_fill_uniform(v, state: int) -> None:
    v = convert(MatrixView, v)
    check_orc(orc.orc_fill_uniform(byref(v), c_uint64(state)))


def ref_fill_uniform_path(v, seed: int, path) -> None:
    """Fill through the reference Rng: Rng(seed).split(p0).split(p1)...; str = tag, int = salt."""
    v = convert(MatrixView, v)
    n = len(path)
    tags = (c_char_p * max(n, 1))(*[p.encode() if isinstance(p, str) else None for p in path])
    salts = (c_uint64 * max(n, 1))(*[0 if isinstance(p, str) else int(p) for p in path])
    check_ref(ref.ref_fill_uniform_path(byref(v), c_uint64(seed), tags, salts, n))


def orc_rng_state(seed: int, path) -> int:
    s = seed & 0xFFFFFFFFFFFFFFFF
    for p in path:
        s = orc.orc_rng_split_tag(s, p.encode()) if isinstance(p, str) else orc.orc_rng_split_salt(s, int(p))
    return s


# ------------------------------------------------------ reference Rng draws (numpy)
_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def _mix(z):
    """Rng::mix (rng.hpp:17-22) on a uint64 array (wrapping arithmetic)."""
    z = z + _GAMMA
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform_draws(state: int, t) -> np.ndarray:
    """Draw t (0-based) of the stream with state s: next_uniform after t+1 steps
    (rng.hpp:24-31): 2 * ((mix(s + (t+1) gamma) >> 11) * 2^-53) - 1."""
    t = np.asarray(t, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = _mix(np.uint64(state) + (t + np.uint64(1)) * _GAMMA)
    return 2.0 * ((x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def normal_values(state: int, t) -> np.ndarray:
    """Box-Muller normal(0,1) of real component t (mdg_fill_normal's definition;
    the reference has no normal generator): draws 2t and 2t+1,
    u1 = (1 - d0)/2 in (0, 1], u2 = (1 + d1)/2, z = sqrt(-2 ln u1) cos(2 pi u2).
    Host libm and the device's log/cospi may differ in the last bits; parity
    tests feed the oracle the device's bytes."""
    t = np.asarray(t, dtype=np.uint64)
    u1 = 0.5 * (1.0 - uniform_draws(state, 2 * t))
    u2 = 0.5 * (1.0 + uniform_draws(state, 2 * t + np.uint64(1)))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
