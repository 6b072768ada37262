"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO beamforming arithmetic: it only turns (seed, tensor id,
element index) into fp32 complex samples with the value distributions of the
paper's workloads.  It is the one module the oracle
(`oracle/`) and the product path may both use.

Counter-based generator
-----------------------
    base = splitmix64(seed ^ (tensor_id << 56))
    h(e) = splitmix64(base ^ e)          e = (b*R + r)*C + c   (logical element)

Everything is integer arithmetic followed by an exact int->float conversion
(or a table lookup / single fp32 multiply), so the numpy twin here and the
device twin in `gen_dev.cu` are bit-identical (checked by a gpu test).

Distributions (`DIST_*`), re from hash bits [40,64), im from bits [16,40):
  uniform    24-bit uniform in [-1, 1)                  (SPEC.md:574 range)
  adc        sum of four 6-bit signed ints, [-128,124]  (ADC-like)
  phase      unit modulus exp(i*2*pi*j/4096), j = h>>52 (steering weights)
  phase_amp  phase * amplitude in (0,1]                 (ultrasound model matrix)
  adc_scaled adc * 2^-7                                  (post-Doppler measurement)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

DIST_UNIFORM = 0
DIST_ADC = 1
DIST_PHASE = 2
DIST_PHASE_AMP = 3
DIST_ADC_SCALED = 4
DIST_NAMES = {"uniform": DIST_UNIFORM, "adc": DIST_ADC, "phase": DIST_PHASE,
              "phase_amp": DIST_PHASE_AMP, "adc_scaled": DIST_ADC_SCALED}

TENSOR_W = 0   # beam weights  [B][M][K]
TENSOR_X = 1   # sampled data  [B][K][N]

SEED_BASE = 250503269   # + config index

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream_base(seed: int, tensor_id: int) -> int:
    x = np.array([(seed ^ (tensor_id << 56)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return int(_splitmix64(x)[0])


def phase_table() -> np.ndarray:
    """4096-entry (cos, sin) table, computed in float64 and rounded to fp32.
    Shared as DATA with the device generator (passed by pointer)."""
    j = np.arange(4096, dtype=np.float64)
    ang = 2.0 * np.pi * j / 4096.0
    return np.stack([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


def _adc4(bits24: np.ndarray) -> np.ndarray:
    s = np.zeros(bits24.shape, dtype=np.int64)
    for f in range(4):
        s += ((bits24 >> np.uint64(6 * f)) & np.uint64(63)).astype(np.int64) - 32
    return s


def values_from_hash(h: np.ndarray, dist: int) -> np.ndarray:
    """Map hashes to complex64 samples (float32 re/im)."""
    hi24 = (h >> np.uint64(40)) & np.uint64(0xFFFFFF)
    lo24 = (h >> np.uint64(16)) & np.uint64(0xFFFFFF)
    if dist == DIST_UNIFORM:
        re = (hi24.astype(np.int64) - 8388608).astype(np.float32) * np.float32(2.0 ** -23)
        im = (lo24.astype(np.int64) - 8388608).astype(np.float32) * np.float32(2.0 ** -23)
    elif dist in (DIST_ADC, DIST_ADC_SCALED):
        re = _adc4(hi24).astype(np.float32)
        im = _adc4(lo24).astype(np.float32)
        if dist == DIST_ADC_SCALED:
            re = re * np.float32(2.0 ** -7)
            im = im * np.float32(2.0 ** -7)
    elif dist in (DIST_PHASE, DIST_PHASE_AMP):
        tab = phase_table()
        j = (h >> np.uint64(52)).astype(np.int64)
        re = tab[j, 0].copy()
        im = tab[j, 1].copy()
        if dist == DIST_PHASE_AMP:
            amp = (lo24.astype(np.int64) + 1).astype(np.float32) * np.float32(2.0 ** -24)
            re = (re * amp).astype(np.float32)
            im = (im * amp).astype(np.float32)
    else:
        raise ValueError(f"unknown distribution {dist}")
    out = np.empty(h.shape, dtype=np.complex64)
    out.real = re
    out.imag = im
    return out


def generate(dist, seed: int, tensor_id: int, B: int, R: int, C: int,
             b_sel=None, r_sel=None, c_sel=None) -> np.ndarray:
    """Complex64 array of logical shape [B][R][C] (or the selected sub-block:
    each *_sel is None for all, or an int array / slice of indices)."""
    if isinstance(dist, str):
        dist = DIST_NAMES[dist]
    bi = np.arange(B, dtype=np.uint64) if b_sel is None else np.arange(B, dtype=np.uint64)[b_sel]
    ri = np.arange(R, dtype=np.uint64) if r_sel is None else np.arange(R, dtype=np.uint64)[r_sel]
    ci = np.arange(C, dtype=np.uint64) if c_sel is None else np.arange(C, dtype=np.uint64)[c_sel]
    bi = np.atleast_1d(bi); ri = np.atleast_1d(ri); ci = np.atleast_1d(ci)
    e = (bi[:, None, None] * np.uint64(R) + ri[None, :, None]) * np.uint64(C) + ci[None, None, :]
    h = _splitmix64(e ^ np.uint64(stream_base(seed, tensor_id)))
    return values_from_hash(h, dist)


def to_interleaved(z: np.ndarray) -> np.ndarray:
    """complex64 [...] -> float32 [..., 2] (re, im adjacent)."""
    return np.ascontiguousarray(z).view(np.float32).reshape(z.shape + (2,))


def to_planar(z: np.ndarray) -> np.ndarray:
    """complex64 [B][R][C] -> float32 [B][2][R][C]."""
    return np.ascontiguousarray(np.stack([z.real, z.imag], axis=1).astype(np.float32))


# ---------------------------------------------------------------- device twin
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"synth device generator not built: {path} (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.synth_generate_dev.restype = ctypes.c_int
        lib.synth_generate_dev.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _LIB = lib
    return _LIB


def generate_device(dist, seed: int, tensor_id: int, B: int, R: int, C: int, device="cuda", b0: int = 0,
                    offset_elems: int = None):
    """Same values as `generate(...)[b0:b0+B]` of a larger tensor (batch entries b0..b0+B-1 of
    the global index space), produced on the GPU into a torch float32 tensor [B][R][C][2]
    (interleaved).  `offset_elems` (default b0*R*C) selects any contiguous run of the global
    element index space, e.g. a row slice of a huge matrix.  torch is plumbing here."""
    import torch
    if isinstance(dist, str):
        dist = DIST_NAMES[dist]
    out = torch.empty((B, R, C, 2), dtype=torch.float32, device=device)
    tab = torch.from_numpy(phase_table()).to(device)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = _lib().synth_generate_dev(ctypes.c_void_p(out.data_ptr()), int(dist),
                                   ctypes.c_uint64(stream_base(seed, tensor_id)),
                                   B, R, C, int(b0) * R * C if offset_elems is None else int(offset_elems),
                                   ctypes.c_void_p(tab.data_ptr()),
                                   ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_generate_dev failed with cuda error {rc}")
    return out
