"""Pins of the fp16-mode oracle (oracle/oracle.c) against things other than itself:
numpy's float16 conversion (library), the paper's closed forms and hand values,
np.matmul on the same rounded inputs, and exact integer arithmetic."""
import numpy as np
import pytest

import oracle
import synth
from tcbf_testutil import read_golden

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


# ----------------------------------------------------------------- rounding
def test_f16_widen_exhaustive_vs_numpy():
    """All 65536 fp16 bit patterns widen exactly like numpy's float16->float64."""
    L = oracle.lib()
    bits = np.arange(65536, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([L.oracle_f16_to_f64(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def _special_f32():
    vals = [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, 65536.0, 1e10, -1e10,
            np.inf, -np.inf, 2.0 ** -14, 2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.0000001,
            2.0 ** -26, 3 * 2.0 ** -25, 2.0 ** -15 + 2.0 ** -25, 1e-45, 1.17549435e-38]
    # exact ties between fp16 neighbours at several exponents (round-half-even both ways)
    for e in (-20, -14, -3, 0, 7, 15):
        for m in (0, 1, 2, 3, 1022, 1023):
            lo = np.float64((1024 + m) * 2.0 ** (e - 10)) if e >= -14 else np.float64(m * 2.0 ** -24)
            step = 2.0 ** (e - 10) if e >= -14 else 2.0 ** -24
            vals += [lo + step / 2, -(lo + step / 2), lo + step / 2 * 1.0001, lo + step / 2 * 0.9999]
    return np.array(vals, dtype=np.float32)


def test_f32_to_f16_rne_vs_numpy():
    """Hand-written RNE bit routine == numpy's IEEE float32->float16 (library)."""
    rng = np.random.default_rng(1)
    rand_bits = rng.integers(0, 2 ** 32, size=60000, dtype=np.uint64).astype(np.uint32)
    v = np.concatenate([_special_f32(), rand_bits.view(np.float32),
                        rng.uniform(-70000, 70000, 20000).astype(np.float32),
                        rng.standard_normal(20000).astype(np.float32) * np.float32(1e-5)])
    got = oracle.f32_to_f16_bits(v)
    ref = v.astype(np.float16).view(np.uint16)
    nan = np.isnan(v)
    assert np.all((got[nan] & 0x7C00) == 0x7C00) and np.all((got[nan] & 0x3FF) != 0)
    assert np.array_equal(got[~nan], ref[~nan])


# ----------------------------------------------------------------- GEMM pins
def _rounded(z):
    """complex64 -> complex128 of the numpy-float16-rounded parts (library RNE)."""
    return z.real.astype(np.float16).astype(np.float64) + 1j * z.imag.astype(np.float16).astype(np.float64)


def test_hand_value_1x1():
    for mode, K, ar, ai, br, bi, er, ei in read_golden("spec_examples.txt"):
        if mode != "f16":
            continue
        w = np.array([[[[float(ar), float(ai)]]]], dtype=np.float32)
        x = np.array([[[[float(br), float(bi)]]]], dtype=np.float32)
        out = oracle.cgemm_f16(w, x, oracle.LAYOUT_INTERLEAVED, 1, 1, 1, 1)
        assert out[0, 0, 0, 0] == float(er) and out[0, 1, 0, 0] == float(ei)


def test_identity_weights_return_inputs_exactly():
    """W = I (M = K): y = x exactly (Eq.3 with one-hot weights)."""
    K, N, B = 37, 29, 2
    x = synth.generate("uniform", 5, synth.TENSOR_X, B, K, N)
    w = np.zeros((B, K, K), dtype=np.complex64)
    w[:, np.arange(K), np.arange(K)] = 1.0
    out = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, K, N, K, B)
    assert np.array_equal(oracle.to_complex(out), _rounded(x))


def test_plane_wave_dirichlet_closed_form():
    """Delay-and-sum (Eqs.1-3): uniform line, d = lambda/2,
    x_k = s * exp(-i pi k sin t0), w_mk = exp(+i pi k sin t_m) ->
    |y_m| = |s| |sin(K psi/2) / sin(psi/2)|, psi = pi (sin t_m - sin t0); peak = K|s|.
    The oracle rounds inputs to fp16, so the bound is K * 2^-10 * |s| (two operands,
    relative rounding 2^-11 each)."""
    K, M, N = 64, 61, 4
    t0 = np.deg2rad(20.0)
    thetas = np.deg2rad(np.linspace(-60, 60, M))
    thetas[np.argmin(np.abs(thetas - t0))] = t0
    s = np.array([1.0, 0.5 - 0.25j, -0.75j, 0.125 + 0.5j])
    k = np.arange(K)
    x = (np.exp(-1j * np.pi * k * np.sin(t0))[:, None] * s[None, :]).astype(np.complex64)[None]
    w = np.exp(1j * np.pi * np.outer(np.sin(thetas), k)).astype(np.complex64)[None]
    out = oracle.to_complex(oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x),
                                             0, M, N, K, 1))[0]
    psi = np.pi * (np.sin(thetas) - np.sin(t0))
    with np.errstate(invalid="ignore", divide="ignore"):
        d = np.where(np.abs(psi) < 1e-12, K, np.abs(np.sin(K * psi / 2) / np.sin(psi / 2)))
    expect = d[:, None] * np.abs(s)[None, :]
    tol = K * 2.0 ** -10 * np.abs(s)[None, :] + 1e-12
    assert np.all(np.abs(np.abs(out) - expect) <= tol)
    m0 = int(np.argmin(np.abs(thetas - t0)))
    assert np.all(np.argmax(np.abs(out), axis=0) == m0)
    assert np.allclose(np.abs(out[m0]), K * np.abs(s), rtol=2.0 ** -10)


def test_integer_inputs_exact_vs_integer_matmul():
    """Integer entries in {-2..2}: every partial sum is exact, so the oracle must equal
    the integer product computed with numpy int64 matmul (library)."""
    rng = np.random.default_rng(7)
    B, M, N, K = 2, 9, 13, 50
    wr, wi = rng.integers(-2, 3, (2, B, M, K))
    xr, xi = rng.integers(-2, 3, (2, B, K, N))
    w = (wr + 1j * wi).astype(np.complex64)
    x = (xr + 1j * xi).astype(np.complex64)
    out = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
    er = np.matmul(wr, xr) - np.matmul(wi, xi)
    ei = np.matmul(wr, xi) + np.matmul(wi, xr)
    assert np.array_equal(out[:, 0], er.astype(np.float64))
    assert np.array_equal(out[:, 1], ei.astype(np.float64))


def test_random_vs_numpy_matmul_on_rounded_inputs():
    B, M, N, K = 3, 17, 23, 71
    w = synth.generate("phase", 11, 0, B, M, K)
    x = synth.generate("adc_scaled", 11, 1, B, K, N)
    out = oracle.to_complex(oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x),
                                             0, M, N, K, B))
    ref = np.matmul(_rounded(w), _rounded(x))
    assert np.max(np.abs(out - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_real_inputs_reduce_to_real_gemm():
    """Im = 0 everywhere: the complex product reduces to a real GEMM and Im(y) = 0."""
    B, M, N, K = 1, 8, 8, 40
    rng = np.random.default_rng(3)
    wr = rng.uniform(-1, 1, (B, M, K)).astype(np.float32)
    xr = rng.uniform(-1, 1, (B, K, N)).astype(np.float32)
    out = oracle.cgemm_f16(synth.to_interleaved(wr.astype(np.complex64)),
                           synth.to_interleaved(xr.astype(np.complex64)), 0, M, N, K, B)
    ref = np.matmul(wr.astype(np.float16).astype(np.float64), xr.astype(np.float16).astype(np.float64))
    assert np.allclose(out[:, 0], ref, rtol=0, atol=1e-12)
    assert np.all(out[:, 1] == 0.0)


def test_conjugate_symmetry_and_linearity():
    """y(conj W, conj X) = conj y(W, X); swapping which operand carries i changes sign as
    the complex product dictates: (iW) X = i (W X).  Catches a wrong sign in Re/Im."""
    B, M, N, K = 1, 5, 7, 33
    w = synth.generate("uniform", 2, 0, B, M, K)
    x = synth.generate("uniform", 2, 1, B, K, N)
    f = lambda a, b: oracle.to_complex(oracle.cgemm_f16(synth.to_interleaved(a), synth.to_interleaved(b),
                                                        0, M, N, K, B))
    y = f(w, x)
    assert np.array_equal(f(np.conj(w), np.conj(x)), np.conj(y))
    assert np.array_equal(f((1j * w).astype(np.complex64), x), 1j * y)


def test_planar_equals_interleaved_and_row_subset():
    B, M, N, K = 2, 12, 10, 21
    w = synth.generate("uniform", 4, 0, B, M, K)
    x = synth.generate("uniform", 4, 1, B, K, N)
    a = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
    b = oracle.cgemm_f16(synth.to_planar(w), synth.to_planar(x), 1, M, N, K, B)
    assert np.array_equal(a, b)
    rows = [11, 0, 5]
    c = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B, rows=rows)
    assert np.array_equal(c, a[:, :, rows])


def test_batch_independence():
    B, M, N, K = 3, 6, 5, 9
    w = synth.generate("uniform", 8, 0, B, M, K)
    x = synth.generate("uniform", 8, 1, B, K, N)
    full = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
    for b in range(B):
        one = oracle.cgemm_f16(synth.to_interleaved(w[b:b + 1]), synth.to_interleaved(x[b:b + 1]),
                               0, M, N, K, 1)
        assert np.array_equal(one[0], full[b])


def test_inputs_unmodified():
    w = synth.to_interleaved(synth.generate("uniform", 1, 0, 1, 4, 8))
    x = synth.to_interleaved(synth.generate("uniform", 1, 1, 1, 8, 3))
    w0, x0 = w.copy(), x.copy()
    oracle.cgemm_f16(w, x, 0, 4, 3, 8, 1)
    assert np.array_equal(w, w0) and np.array_equal(x, x0)


def test_useful_ops():
    """8 * M * N * K per complex GEMM."""
    assert oracle.useful_ops(8192, 8192, 8192, 1) == 8 * 8192 ** 3
    assert oracle.useful_ops(1024, 1024, 256, 256) == 8 * 1024 * 1024 * 256 * 256
