"""Pins of the oracle's packing routines (PAPER.md:107 packing/transpose kernels,
PAPER.md:414 re/im separation, PAPER.md:249 zero padding) against numpy library
routines: float16 astype (RNE), packbits(bitorder='little')."""
import numpy as np

import oracle
import synth


def test_pack_f16_weights_and_data_vs_numpy():
    B, M, K, N = 2, 5, 70, 9
    K16, Np = 128, 16
    w = synth.generate("uniform", 3, 0, B, M, K)
    x = synth.generate("uniform", 3, 1, B, K, N)
    for layout, conv in ((0, synth.to_interleaved), (1, synth.to_planar)):
        pw = oracle.pack_f16(conv(w), layout, oracle.WEIGHTS, B, M, K, K16)
        px = oracle.pack_f16(conv(x), layout, oracle.DATA, B, K, N, Np)
        ew = np.zeros((B, 2, M, K16), np.float16)
        ew[:, 0, :, :K] = w.real.astype(np.float16)
        ew[:, 1, :, :K] = w.imag.astype(np.float16)
        ex = np.zeros((B, 2, K, Np), np.float16)
        ex[:, 0, :, :N] = x.real.astype(np.float16)
        ex[:, 1, :, :N] = x.imag.astype(np.float16)
        assert np.array_equal(pw, ew.view(np.uint16))
        assert np.array_equal(px, ex.view(np.uint16))


def test_pack_b1_vs_numpy_packbits():
    B, M, K, N = 2, 4, 100, 6
    Kw = 8
    w = synth.generate("adc", 4, 0, B, M, K)     # adc has exact zeros -> exercises v >= 0
    x = synth.generate("adc", 4, 1, B, K, N)
    assert np.any(w.real == 0)

    def ref(bits_rows):  # [..., K] 0/1 -> [..., Kw] uint32, LSB-first
        padded = np.zeros(bits_rows.shape[:-1] + (Kw * 32,), np.uint8)
        padded[..., :K] = bits_rows
        by = np.packbits(padded, axis=-1, bitorder="little")
        return by.view("<u4")

    for layout, conv in ((0, synth.to_interleaved), (1, synth.to_planar)):
        pw = oracle.pack_b1(conv(w), layout, oracle.WEIGHTS, B, M, K, Kw)
        px = oracle.pack_b1(conv(x), layout, oracle.DATA, B, K, N, Kw)
        ew = np.stack([ref(w.real >= 0), ref(w.imag >= 0)], axis=1)
        ex = np.stack([ref((x.real >= 0).transpose(0, 2, 1)), ref((x.imag >= 0).transpose(0, 2, 1))], axis=1)
        assert np.array_equal(pw, ew) and np.array_equal(px, ex)
        # padding bits are 0 ("we set the padded region to binary 0")
        assert np.all(pw[..., K // 32] >> (K % 32) == 0) and np.all(pw[..., K // 32 + 1:] == 0)


def test_spec_pack_examples():
    """(1,-1,1,-1) -> 0b0101 (LSB = first element); 32 positives -> 0xFFFFFFFF;
    33 elements -> second word holds 1 bit."""
    w = np.array([[[[1, 0], [-1, 0], [1, 0], [-1, 0]]]], np.float32)
    assert oracle.pack_b1(w, 0, 0, 1, 1, 4, 1)[0, 0, 0, 0] == 5
    w = np.ones((1, 1, 32, 2), np.float32)
    assert oracle.pack_b1(w, 0, 0, 1, 1, 32, 1)[0, 0, 0, 0] == 0xFFFFFFFF
    w = np.ones((1, 1, 33, 2), np.float32)
    p = oracle.pack_b1(w, 0, 0, 1, 1, 33, 2)
    assert p[0, 0, 0, 0] == 0xFFFFFFFF and p[0, 0, 0, 1] == 1


def test_generator_recipes_are_deterministic_and_shaped():
    a = synth.generate("adc", 1, 1, 2, 3, 4)
    b = synth.generate("adc", 1, 1, 2, 3, 4)
    assert np.array_equal(a, b)
    sub = synth.generate("adc", 1, 1, 2, 3, 4, b_sel=[1], r_sel=[2], c_sel=slice(1, 3))
    assert np.array_equal(sub[0, 0], a[1, 2, 1:3])
    assert np.all(np.abs(a.real) <= 128) and np.all(a.real == np.round(a.real))
    p = synth.generate("phase", 1, 0, 1, 50, 50)
    assert np.allclose(np.abs(p), 1.0, atol=1e-6)
    u = synth.generate("uniform", 1, 0, 1, 100, 100)
    assert np.all(u.real >= -1) and np.all(u.real < 1)
    pa = synth.generate("phase_amp", 1, 0, 1, 50, 50)
    assert np.all(np.abs(pa) <= 1.0 + 1e-6) and np.all(np.abs(pa) > 0)
