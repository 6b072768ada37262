"""paper_2505_03269_b200 -- B200-native Tensor-Core Beamformer hot path.

Thin Python binding (argument marshalling only) of the C ABI in include/tcbf.h,
implemented by lib/libtcbf.so (hand-written sm_100a CUDA).  Every step of the
path -- packing, the complex GEMM, the epilogue -- runs in those kernels; torch is
used only to own device memory and streams.  There is NO CPU fallback: if the
native library is missing this module raises.

    plan = Plan(M, N, K, batch, "f16" | "b1")
    wp = plan.pack(WEIGHTS, w)            # w: cuda float32 [B,M,K,2] or [B,2,M,K]
    xp = plan.pack(DATA, x)               # x: cuda float32 [B,K,N,2] or [B,2,K,N]
    y  = plan.beamform(wp, xp)            # [B,2,M,N] float32 (f16) / int32 (b1)
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["Plan", "TcbfError", "layout_sizes", "WEIGHTS", "DATA", "INTERLEAVED", "PLANAR",
           "F16", "B1", "library_path", "lib"]

F16, B1 = 0, 1
WEIGHTS, DATA = 0, 1
INTERLEAVED, PLANAR = 0, 1
_PREC = {"f16": F16, "b1": B1, F16: F16, B1: B1}
_LAYOUT = {"interleaved": INTERLEAVED, "planar": PLANAR, INTERLEAVED: INTERLEAVED, PLANAR: PLANAR}

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "lib", "libtcbf.so")


class TcbfError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {status_string(status)}: {detail}")
        self.status = status


_LIB = None


def lib():
    """The loaded libtcbf.so (raises if it was not built -- no fallback path)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(library_path):
            raise RuntimeError(f"native library missing: {library_path}; run __graft_entry__.build()")
        L = ctypes.CDLL(library_path)
        i64, vp, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
        L.tcbf_layout_sizes.restype = ctypes.c_int
        L.tcbf_layout_sizes.argtypes = [i64, i64, i64, i64, ctypes.c_int, ctypes.POINTER(sz),
                                        ctypes.POINTER(sz), ctypes.POINTER(sz), ctypes.POINTER(i64)]
        L.tcbf_plan_create.restype = ctypes.c_int
        L.tcbf_plan_create.argtypes = [ctypes.POINTER(vp), i64, i64, i64, i64, ctypes.c_int]
        L.tcbf_plan_destroy.restype = ctypes.c_int
        L.tcbf_plan_destroy.argtypes = [vp]
        L.tcbf_packed_bytes.restype = ctypes.c_int
        L.tcbf_packed_bytes.argtypes = [vp, ctypes.c_int, ctypes.POINTER(sz)]
        L.tcbf_output_bytes.restype = ctypes.c_int
        L.tcbf_output_bytes.argtypes = [vp, ctypes.POINTER(sz)]
        L.tcbf_pack.restype = ctypes.c_int
        L.tcbf_pack.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, vp, vp]
        L.tcbf_beamform.restype = ctypes.c_int
        L.tcbf_beamform.argtypes = [vp, vp, vp, vp, vp]
        L.tcbf_beamform_raw.restype = ctypes.c_int
        L.tcbf_beamform_raw.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp]
        L.tcbf_beamform_f16i.restype = ctypes.c_int
        L.tcbf_beamform_f16i.argtypes = [vp, vp, vp, vp, vp]
        L.tcbf_steering_weights.restype = ctypes.c_int
        L.tcbf_steering_weights.argtypes = [vp, vp, vp, vp, ctypes.c_double, ctypes.c_int, vp, vp]
        L.tcbf_beamform_host.restype = ctypes.c_int
        L.tcbf_beamform_host.argtypes = [vp, vp, vp, ctypes.c_int, vp]
        L.tcbf_last_launch_count.restype = ctypes.c_int
        L.tcbf_last_launch_count.argtypes = []
        L.tcbf_plan_variant.restype = ctypes.c_char_p
        L.tcbf_plan_variant.argtypes = [vp]
        L.tcbf_plan_kernel.restype = ctypes.c_char_p
        L.tcbf_plan_kernel.argtypes = [vp, ctypes.c_int]
        L.tcbf_plan_raw_fused.restype = ctypes.c_int
        L.tcbf_plan_raw_fused.argtypes = [vp]
        L.tcbf_status_string.restype = ctypes.c_char_p
        L.tcbf_status_string.argtypes = [ctypes.c_int]
        L.tcbf_last_error.restype = ctypes.c_char_p
        L.tcbf_last_error.argtypes = []
        _LIB = L
    return _LIB


def status_string(s: int) -> str:
    return lib().tcbf_status_string(int(s)).decode()


def _check(rc: int, where: str):
    if rc != 0:
        raise TcbfError(rc, where, lib().tcbf_last_error().decode())


def layout_sizes(M, N, K, batch, precision="f16"):
    """Host-only: (w_bytes, x_bytes, out_bytes, k_packed)."""
    w, x, o, k = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_int64()
    _check(lib().tcbf_layout_sizes(M, N, K, batch, _PREC[precision], ctypes.byref(w), ctypes.byref(x),
                                   ctypes.byref(o), ctypes.byref(k)), "tcbf_layout_sizes")
    return w.value, x.value, o.value, k.value


def _dtype(name):
    import torch
    return {"f32": torch.float32, "f16": torch.float16, "i32": torch.int32}[name]


def _need(t, what, dtypes, nbytes, device=None):
    """Argument check before a raw pointer crosses the ABI (the C side cannot see tensor
    metadata): CUDA tensor, contiguous, one of `dtypes`, at least `nbytes` bytes, on `device`."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what}: expected a torch.Tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ValueError(f"{what}: must be a CUDA tensor (got device {t.device})")
    if device is not None and t.device != device:
        raise ValueError(f"{what}: on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: must be contiguous")
    if t.dtype not in tuple(_dtype(d) for d in dtypes):
        raise TypeError(f"{what}: dtype {t.dtype} not in {dtypes}")
    have = t.numel() * t.element_size()
    if have < nbytes:
        raise ValueError(f"{what}: {have} bytes < the plan's {nbytes}")


def _stream_ptr(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


class Plan:
    """Immutable beamforming plan for `batch` x (M beams, N samples, K receivers)."""

    def __init__(self, M: int, N: int, K: int, batch: int, precision="f16"):
        self.M, self.N, self.K, self.batch = int(M), int(N), int(K), int(batch)
        self.precision = _PREC[precision]
        h = ctypes.c_void_p()
        _check(lib().tcbf_plan_create(ctypes.byref(h), self.M, self.N, self.K, self.batch, self.precision),
               "tcbf_plan_create")
        self._h = h
        self.w_bytes, self.x_bytes, self.out_bytes, self.k_packed = layout_sizes(
            self.M, self.N, self.K, self.batch, self.precision)
        self.variant = lib().tcbf_plan_variant(h).decode()
        self.n_packed = (self.N + 7) // 8 * 8   # F16 data rows (MN-major packed data)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and _LIB is not None:
            try:
                _LIB.tcbf_plan_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    __del__ = close

    # ------------------------------------------------------------ buffers (torch = plumbing)
    def packed_shape(self, operand):
        if operand == WEIGHTS:
            return (self.batch, 2, self.M, self.k_packed)
        if self.precision == F16:
            return (self.batch, 2, self.K, self.n_packed)   # MN-major: [K][Np]
        return (self.batch, 2, self.N, self.k_packed)       # bits along K: [N][Kw]

    def alloc_packed(self, operand, device="cuda"):
        import torch
        dt = torch.float16 if self.precision == F16 else torch.int32
        return torch.empty(self.packed_shape(operand), dtype=dt, device=device)

    def alloc_output(self, device="cuda"):
        import torch
        dt = torch.float32 if self.precision == F16 else torch.int32
        return torch.empty((self.batch, 2, self.M, self.N), dtype=dt, device=device)

    # ------------------------------------------------------------ argument checks
    def _src_bytes(self, operand):
        rows, cols = (self.M, self.K) if operand == WEIGHTS else (self.K, self.N)
        return self.batch * rows * cols * 8

    def _packed_bytes(self, operand):
        return self.w_bytes if operand == WEIGHTS else self.x_bytes

    def _packed_dtypes(self):
        return ("f16",) if self.precision == F16 else ("i32",)

    def _out_dtype(self):
        return ("f32",) if self.precision == F16 else ("i32",)

    # ------------------------------------------------------------ the path
    def pack(self, operand, src, layout="interleaved", out=None, stream=None):
        lay = _LAYOUT[layout]
        _need(src, "pack source", ("f32",), self._src_bytes(operand))
        if out is None:
            out = self.alloc_packed(operand, src.device)
        _need(out, "packed output", self._packed_dtypes(), self._packed_bytes(operand), src.device)
        _check(lib().tcbf_pack(self._h, int(operand), ctypes.c_void_p(src.data_ptr()), lay,
                               ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream, src.device)), "tcbf_pack")
        return out

    def beamform(self, w_packed, x_packed, out=None, stream=None):
        _need(w_packed, "packed weights", self._packed_dtypes(), self.w_bytes)
        _need(x_packed, "packed data", self._packed_dtypes(), self.x_bytes, w_packed.device)
        if out is None:
            out = self.alloc_output(w_packed.device)
        _need(out, "output", self._out_dtype(), self.out_bytes, w_packed.device)
        _check(lib().tcbf_beamform(self._h, ctypes.c_void_p(w_packed.data_ptr()),
                                   ctypes.c_void_p(x_packed.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                   _stream_ptr(stream, w_packed.device)), "tcbf_beamform")
        return out

    def beamform_raw(self, w_packed, x_src, layout="interleaved", out=None, stream=None):
        """Beamform straight from the fp32 data (pack fused into the GEMM where supported)."""
        _need(w_packed, "packed weights", self._packed_dtypes(), self.w_bytes)
        _need(x_src, "data source", ("f32",), self._src_bytes(DATA), w_packed.device)
        if out is None:
            out = self.alloc_output(w_packed.device)
        _need(out, "output", self._out_dtype(), self.out_bytes, w_packed.device)
        _check(lib().tcbf_beamform_raw(self._h, ctypes.c_void_p(w_packed.data_ptr()),
                                       ctypes.c_void_p(x_src.data_ptr()), _LAYOUT[layout],
                                       ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream, w_packed.device)),
               "tcbf_beamform_raw")
        return out

    def beamform_f16i(self, w_packed, x_f16, out=None, stream=None):
        """16-bit beamform of fp16 interleaved complex data x_f16 [B][K][N][2] (torch.float16, cuda),
        no data pack (NEXT-1)."""
        _need(w_packed, "packed weights", self._packed_dtypes(), self.w_bytes)
        _need(x_f16, "fp16 interleaved data", ("f16",), self.batch * self.K * self.N * 4, w_packed.device)
        if out is None:
            out = self.alloc_output(w_packed.device)
        _need(out, "output", self._out_dtype(), self.out_bytes, w_packed.device)
        _check(lib().tcbf_beamform_f16i(self._h, ctypes.c_void_p(w_packed.data_ptr()),
                                        ctypes.c_void_p(x_f16.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                        _stream_ptr(stream, w_packed.device)), "tcbf_beamform_f16i")
        return out

    def kernel(self, entry="beamform") -> str:
        """Name of the GEMM kernel an entry point launches for this plan (chosen by the C library
        at plan creation; entry: 'beamform' | 'raw' | 'f16i')."""
        e = {"beamform": 0, "raw": 1, "f16i": 2}[entry]
        return lib().tcbf_plan_kernel(self._h, e).decode()

    @property
    def raw_fused(self) -> bool:
        """True when beamform_raw runs one kernel with the data conversion inside (no pack pass)."""
        return bool(lib().tcbf_plan_raw_fused(self._h))

    @property
    def raw_variant(self) -> str:
        return self.kernel("raw")

    def steering_weights(self, positions, angles, freqs, c, layout="interleaved", out=None, stream=None):
        """fp32 weight source w[b][m][k] = exp(+2 pi i f_b d_k sin(theta_m) / c).
        positions [K], angles [M], freqs [B]: cuda float64 tensors."""
        import torch
        for t, what, n in ((positions, "positions", self.K), (angles, "angles", self.M), (freqs, "freqs", self.batch)):
            if not isinstance(t, torch.Tensor) or t.dtype != torch.float64:
                raise TypeError(f"{what}: expected a float64 torch.Tensor")
            _need(t.view(torch.float32), what, ("f32",), 8 * n, positions.device)
        if out is None:
            shape = (self.batch, self.M, self.K, 2) if _LAYOUT[layout] == INTERLEAVED else (self.batch, 2, self.M, self.K)
            out = torch.empty(shape, dtype=torch.float32, device=positions.device)
        _need(out, "weight source", ("f32",), self._src_bytes(WEIGHTS), positions.device)
        _check(lib().tcbf_steering_weights(self._h, ctypes.c_void_p(positions.data_ptr()),
                                           ctypes.c_void_p(angles.data_ptr()), ctypes.c_void_p(freqs.data_ptr()),
                                           float(c), _LAYOUT[layout], ctypes.c_void_p(out.data_ptr()),
                                           _stream_ptr(stream, positions.device)), "tcbf_steering_weights")
        return out

    def beamform_host(self, w_packed_dev, x_host, out_host, layout="interleaved"):
        """End-to-end over host buffers (torch CPU tensors, pinned for overlap)."""
        import torch
        _need(w_packed_dev, "packed weights", self._packed_dtypes(), self.w_bytes)
        for t, what, dts, nb in ((x_host, "host data", (torch.float32,), self._src_bytes(DATA)),
                                 (out_host, "host output", (_dtype(self._out_dtype()[0]),), self.out_bytes)):
            if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_contiguous() or t.dtype not in dts:
                raise ValueError(f"{what}: must be a contiguous CPU tensor of dtype {dts[0]}")
            if t.numel() * t.element_size() < nb:
                raise ValueError(f"{what}: {t.numel() * t.element_size()} bytes < the plan's {nb}")
        _check(lib().tcbf_beamform_host(self._h, ctypes.c_void_p(w_packed_dev.data_ptr()),
                                        ctypes.c_void_p(x_host.data_ptr()), _LAYOUT[layout],
                                        ctypes.c_void_p(out_host.data_ptr())), "tcbf_beamform_host")
        return out_host

    @staticmethod
    def last_launch_count() -> int:
        return lib().tcbf_last_launch_count()
