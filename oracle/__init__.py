"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of oracle/liboracle.so.

The CPU oracle of the Tensor-Core Beamformer hot path (PAPER.md:78-84,
143-159, 170-172, 209-259, 282): plain fp64 / int64 triple loops with their
own fp16 rounding, sign rule and bit unpacking.  Only `tests/`,
`__graft_entry__.smoke()` and bench.py's cpu_baseline / `--impl reference`
legs may import this package; the product path (paper_2505_03269_b200) never
does.  See oracle/oracle.c for the per-function citations and DESIGN.md for
the readings and the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

LAYOUT_INTERLEAVED = 0
LAYOUT_PLANAR = 1
WEIGHTS = 0
DATA = 1

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_f32_to_f16.argtypes = [ctypes.c_float]
        L.oracle_f16_to_f64.restype = ctypes.c_double
        L.oracle_f16_to_f64.argtypes = [ctypes.c_uint16]
        L.oracle_sign_bit.restype = ctypes.c_int
        L.oracle_sign_bit.argtypes = [ctypes.c_float]
        for name in ("oracle_cgemm_f16", "oracle_cgemm_b1"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [vp, vp, ctypes.c_int, i64, i64, i64, i64, vp, i64, vp]
        L.oracle_cgemm_b1_packed.restype = ctypes.c_int
        L.oracle_cgemm_b1_packed.argtypes = [vp, vp, i64, i64, i64, i64, i64, vp, i64, vp]
        for name in ("oracle_pack_f16", "oracle_pack_b1"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [vp, ctypes.c_int, ctypes.c_int, i64, i64, i64, i64, vp]
        L.oracle_steering_weights.restype = ctypes.c_int
        L.oracle_steering_weights.argtypes = [vp, vp, vp, ctypes.c_double, i64, i64, i64, vp]
        L.oracle_useful_ops.restype = ctypes.c_double
        L.oracle_useful_ops.argtypes = [i64, i64, i64, i64]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _src(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _rows(rows, M):
    if rows is None:
        return None, M
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    return r, int(r.size)


def f32_to_f16_bits(v: np.ndarray) -> np.ndarray:
    L = lib()
    flat = np.asarray(v, dtype=np.float32).ravel()
    return np.fromiter((L.oracle_f32_to_f16(float(x)) for x in flat), dtype=np.uint16,
                       count=flat.size).reshape(np.shape(v))


def cgemm_f16(w: np.ndarray, x: np.ndarray, layout: int, M: int, N: int, K: int, B: int,
              rows=None) -> np.ndarray:
    """Returns float64 [B][2][n_rows][N] (Re, Im planes)."""
    w, x = _src(w), _src(x)
    r, nr = _rows(rows, M)
    out = np.empty((B, 2, nr, N), dtype=np.float64)
    rc = lib().oracle_cgemm_f16(_ptr(w), _ptr(x), layout, M, N, K, B,
                                None if r is None else _ptr(r), nr, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_cgemm_f16 rc={rc}")
    return out


def cgemm_b1(w: np.ndarray, x: np.ndarray, layout: int, M: int, N: int, K: int, B: int,
             rows=None) -> np.ndarray:
    """Returns int32 [B][2][n_rows][N]."""
    w, x = _src(w), _src(x)
    r, nr = _rows(rows, M)
    out = np.empty((B, 2, nr, N), dtype=np.int32)
    rc = lib().oracle_cgemm_b1(_ptr(w), _ptr(x), layout, M, N, K, B,
                               None if r is None else _ptr(r), nr, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_cgemm_b1 rc={rc}")
    return out


def cgemm_b1_packed(wp: np.ndarray, xp: np.ndarray, M: int, N: int, K: int, Kw: int, B: int,
                    rows=None) -> np.ndarray:
    wp = np.ascontiguousarray(wp, dtype=np.uint32)
    xp = np.ascontiguousarray(xp, dtype=np.uint32)
    r, nr = _rows(rows, M)
    out = np.empty((B, 2, nr, N), dtype=np.int32)
    rc = lib().oracle_cgemm_b1_packed(_ptr(wp), _ptr(xp), M, N, K, Kw, B,
                                      None if r is None else _ptr(r), nr, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_cgemm_b1_packed rc={rc}")
    return out


def pack_f16(src: np.ndarray, layout: int, operand: int, B: int, R: int, C: int,
             Cp: int) -> np.ndarray:
    """uint16 fp16 bit patterns, [B][2][R][Cp]: weights (R=M, C=K, Cp=K16) or data
    (R=K, C=N, Cp=Np) -- both keep their row order, zero column padding."""
    src = _src(src)
    out = np.empty((B, 2, R, Cp), dtype=np.uint16)
    rc = lib().oracle_pack_f16(_ptr(src), layout, operand, B, R, C, Cp, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_pack_f16 rc={rc}")
    return out


def pack_b1(src: np.ndarray, layout: int, operand: int, B: int, R: int, C: int,
            Kw: int) -> np.ndarray:
    src = _src(src)
    rows = R if operand == WEIGHTS else C
    out = np.empty((B, 2, rows, Kw), dtype=np.uint32)
    rc = lib().oracle_pack_b1(_ptr(src), layout, operand, B, R, C, Kw, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_pack_b1 rc={rc}")
    return out


def steering_weights(positions, angles, freqs, c: float) -> np.ndarray:
    """complex128 [B][M][K]: exp(+2 pi i f_b d_k sin(theta_m) / c)."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    th = np.ascontiguousarray(angles, dtype=np.float64)
    fr = np.ascontiguousarray(freqs, dtype=np.float64)
    B, M, K = fr.size, th.size, pos.size
    out = np.empty((B, M, K, 2), dtype=np.float64)
    rc = lib().oracle_steering_weights(_ptr(pos), _ptr(th), _ptr(fr), float(c), B, M, K, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_steering_weights rc={rc}")
    return out[..., 0] + 1j * out[..., 1]


def useful_ops(M: int, N: int, K: int, B: int) -> float:
    return lib().oracle_useful_ops(M, N, K, B)


def to_complex(out: np.ndarray) -> np.ndarray:
    """[B][2][R][N] planes -> complex128 [B][R][N]."""
    return out[:, 0].astype(np.float64) + 1j * out[:, 1].astype(np.float64)
