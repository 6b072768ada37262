"""Pins of the 1-bit oracle (oracle/oracle.c) and of the paper readings it relies on:
Table II and Fig. 1 (golden fixtures), SPEC hand values, exhaustive enumeration with
the matched-beam count, invariants, numpy.packbits (library) for the packing, and the
paper's popcount equations (Eq.4-6) evaluated independently here to pin reading R1
(K in Eq.5 is the PADDED length)."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from tcbf_testutil import read_golden


def _bits_to_src(bre, bim):
    """bits (0/1 arrays) -> fp32 interleaved source with +-1 components."""
    return np.stack([np.where(bre, 1.0, -1.0), np.where(bim, 1.0, -1.0)], axis=-1).astype(np.float32)


def test_sign_rule():
    """0 is not representable; reading R4: v >= 0 -> bit 1 (-0 -> 1), NaN -> 0."""
    L = oracle.lib()
    assert L.oracle_sign_bit(0.0) == 1 and L.oracle_sign_bit(-0.0) == 1
    assert L.oracle_sign_bit(1e-45) == 1 and L.oracle_sign_bit(-1e-45) == 0
    assert L.oracle_sign_bit(float("nan")) == 0
    assert L.oracle_sign_bit(float("inf")) == 1 and L.oracle_sign_bit(float("-inf")) == 0


def test_table2_real_dot_product():
    """A=(1,-1,1,-1), B=(1,1,-1,-1): sum = 0, popc(A^B)=2, K-2popc = 0.
    Complex embedding with Im = +1 on both: Re = 0 - 4 = -4, Im = 0."""
    rows = read_golden("table2.txt")
    data = [list(map(int, r)) for r in rows if r[0] not in ("SUM", "POPC", "RESULT")]
    foot = {r[0]: int(r[1]) for r in rows if r[0] in ("SUM", "POPC", "RESULT")}
    A = np.array([d[0] for d in data]); Bv = np.array([d[1] for d in data])
    bitA = np.array([d[3] for d in data]); bitB = np.array([d[4] for d in data])
    assert np.array_equal(np.where(bitA, 1, -1), A) and np.array_equal(np.where(bitB, 1, -1), Bv)
    assert int(np.sum(bitA ^ bitB)) == foot["POPC"]
    K = len(A)
    assert K - 2 * foot["POPC"] == foot["RESULT"] == foot["SUM"]
    w = _bits_to_src(bitA, np.ones(K, int)).reshape(1, 1, K, 2)
    x = _bits_to_src(bitB, np.ones(K, int)).reshape(1, K, 1, 2)
    out = oracle.cgemm_b1(w, x, 0, 1, 1, K, 1)
    assert out[0, 0, 0, 0] == -4 and out[0, 1, 0, 0] == 0
    # the word values of Table II's vectors under LSB-first packing (reading R3)
    wp = oracle.pack_b1(w, 0, oracle.WEIGHTS, 1, 1, K, 1)
    xp = oracle.pack_b1(x, 0, oracle.DATA, 1, K, 1, 1)
    assert wp[0, 0, 0, 0] == 0b0101 and xp[0, 0, 0, 0] == 0b0011
    assert bin(int(wp[0, 0, 0, 0]) ^ int(xp[0, 0, 0, 0])).count("1") == foot["POPC"]


def test_fig1_encoding_products():
    """00=-1-i, 01=-1+i, 10=1-i, 11=1+i. All 16 K=1 products
    equal the complex products of the printed values."""
    enc = {r[0]: complex(int(r[1]), int(r[2])) for r in read_golden("fig1_encoding.txt")}
    codes = list(enc)
    w = np.array([[[[1.0 if c[0] == "1" else -1.0, 1.0 if c[1] == "1" else -1.0]] for c in codes]],
                 dtype=np.float32)                       # [1][4][1][2]  M=4, K=1
    x = np.array([[[[1.0 if c[0] == "1" else -1.0, 1.0 if c[1] == "1" else -1.0] for c in codes]]],
                 dtype=np.float32)                       # [1][1][4][2]  K=1, N=4
    out = oracle.to_complex(oracle.cgemm_b1(w, x, 0, 4, 4, 1, 1))[0]
    for i, a in enumerate(codes):
        for j, b in enumerate(codes):
            assert out[i, j] == enc[a] * enc[b]


def test_spec_hand_values():
    for mode, K, ar, ai, br, bi, er, ei in read_golden("spec_examples.txt"):
        if mode != "b1":
            continue
        K = int(K)
        w = np.tile(np.array([float(ar), float(ai)], np.float32), (1, 1, K, 1))
        x = np.tile(np.array([float(br), float(bi)], np.float32), (1, K, 1, 1))
        out = oracle.cgemm_b1(w, x, 0, 1, 1, K, 1)
        assert (out[0, 0, 0, 0], out[0, 1, 0, 0]) == (int(er), int(ei))
        # same through the packed path with a full 256-bit granule (K_pad = 256-K)
        wp = oracle.pack_b1(w, 0, oracle.WEIGHTS, 1, 1, K, 8)
        xp = oracle.pack_b1(x, 0, oracle.DATA, 1, K, 1, 8)
        outp = oracle.cgemm_b1_packed(wp, xp, 1, 1, K, 8, 1)
        assert np.array_equal(out, outp)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_exhaustive_enumeration(K):
    """All 4^K vectors as weight rows and as data columns.  Pins: y = 2K + 0i exactly
    at the matched pairs u = conj(v) (imag bits flipped) and nowhere else; the total sum
    over all pairs is 0 (each component sums to 0 over the enumeration); invariants."""
    V = 4 ** K
    codes = np.array(list(itertools.product([0, 1], repeat=2 * K)), dtype=np.int64)  # [V][2K]
    bre, bim = codes[:, :K], codes[:, K:]
    w = _bits_to_src(bre, bim).reshape(1, V, K, 2)
    x = np.ascontiguousarray(_bits_to_src(bre, bim).transpose(1, 0, 2)).reshape(1, K, V, 2)
    out = oracle.cgemm_b1(w, x, 0, V, V, K, 1)
    re, im = out[0, 0].astype(np.int64), out[0, 1].astype(np.int64)
    matched = np.zeros((V, V), bool)
    conj_index = {tuple(np.concatenate([bre[i], 1 - bim[i]])): i for i in range(V)}
    for j in range(V):
        matched[conj_index[tuple(np.concatenate([bre[j], bim[j]]))], j] = True
    hit = (re == 2 * K) & (im == 0)
    assert np.array_equal(hit, matched) and hit.sum() == V
    assert re.sum() == 0 and im.sum() == 0
    assert np.all(re % 2 == 0) and np.all(im % 2 == 0)
    assert np.all(np.abs(re) + np.abs(im) <= 2 * K)
    assert np.all(((re + im) // 2 - K) % 2 == 0)
    # the same GEMM through the packed path (K_pad = 256 - K padding bits)
    wp = oracle.pack_b1(w, 0, oracle.WEIGHTS, 1, V, K, 8)
    xp = oracle.pack_b1(x, 0, oracle.DATA, 1, K, V, 8)
    assert np.array_equal(oracle.cgemm_b1_packed(wp, xp, V, V, K, 8, 1), out)


def test_b1_equals_f16_oracle_and_numpy_on_pm1():
    """Cross-oracle: the int64 1-bit definition equals the fp64 16-bit definition and
    np.matmul (library) on the +-1 expansion (exact: integers < 2^53)."""
    rng = np.random.default_rng(5)
    B, M, N, K = 2, 7, 9, 300
    w = rng.standard_normal((B, M, K, 2)).astype(np.float32)
    x = rng.standard_normal((B, K, N, 2)).astype(np.float32)
    b1 = oracle.cgemm_b1(w, x, 0, M, N, K, B)
    pw = np.where(w >= 0, 1.0, -1.0).astype(np.float32)
    px = np.where(x >= 0, 1.0, -1.0).astype(np.float32)
    f16 = oracle.cgemm_f16(pw, px, 0, M, N, K, B)
    assert np.array_equal(b1.astype(np.float64), f16)
    ref = np.matmul(pw[..., 0] + 1j * pw[..., 1], px[..., 0] + 1j * px[..., 1])
    assert np.array_equal(oracle.to_complex(b1), ref)


def _eq5_paper(ar, ai, br, bi, Ktot, Kpad):
    """PAPER.md:252-259 verbatim (Eq.5 and the unnumbered Im form), bits as 0/1 arrays over
    the padded length; overline(B_i) = complement."""
    popc = lambda a: int(np.sum(a))
    re = 2 * (Ktot - (popc(ar ^ br) + popc(ai ^ (1 - bi))))
    im = 2 * (Ktot - Kpad - (popc(ar ^ bi) + popc(ai ^ br)))
    return re, im


def test_reading_R1_padded_K_in_eq5():
    """Reading R1: the paper's K in Eq.5 must be the padded length.  With K = K_log + K_pad
    (padding bits 0 in both operands) Eq.5 equals the definition; with the
    logical K it is off by 2*K_pad in Re whenever K_pad > 0."""
    rng = np.random.default_rng(9)
    for _ in range(200):
        K = int(rng.integers(1, 100))
        Kpad = int(rng.integers(0, 40))
        ar, ai, br, bi = (np.concatenate([rng.integers(0, 2, K), np.zeros(Kpad, int)]) for _ in range(4))
        w = _bits_to_src(ar[:K], ai[:K]).reshape(1, 1, K, 2)
        x = _bits_to_src(br[:K], bi[:K]).reshape(1, K, 1, 2)
        out = oracle.cgemm_b1(w, x, 0, 1, 1, K, 1)
        truth = (int(out[0, 0, 0, 0]), int(out[0, 1, 0, 0]))
        assert _eq5_paper(ar, ai, br, bi, K + Kpad, Kpad) == truth
        if Kpad > 0:
            assert _eq5_paper(ar, ai, br, bi, K, Kpad)[0] == truth[0] - 2 * Kpad


def test_random_corpus_invariants_and_packed_path():
    """SPEC.md:572 style corpus: M, N <= 32, K <= 2048, half with K % 32 != 0."""
    rng = np.random.default_rng(11)
    for t in range(60):
        M, N = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        K = int(rng.integers(1, 2049))
        if t % 2 == 0 and K % 32 == 0:
            K += 1
        Kw = ((K + 31) // 32 + 7) // 8 * 8
        w = rng.standard_normal((1, M, K, 2)).astype(np.float32)
        x = rng.standard_normal((1, K, N, 2)).astype(np.float32)
        out = oracle.cgemm_b1(w, x, 0, M, N, K, 1)
        re, im = out[0, 0].astype(np.int64), out[0, 1].astype(np.int64)
        assert np.all(re % 2 == 0) and np.all(im % 2 == 0)
        assert np.all(np.abs(re) + np.abs(im) <= 2 * K)
        assert np.all(((re + im) // 2 - K) % 2 == 0)
        wp = oracle.pack_b1(w, 0, oracle.WEIGHTS, 1, M, K, Kw)
        xp = oracle.pack_b1(x, 0, oracle.DATA, 1, K, N, Kw)
        assert np.array_equal(oracle.cgemm_b1_packed(wp, xp, M, N, K, Kw, 1), out)


def test_matched_beam_closed_form():
    """Closed form (iii): W[m,:] = conj(X[:, n0]) at the bit level -> y[m, n0] = 2K + 0i."""
    rng = np.random.default_rng(2)
    K, N = 777, 5
    x = rng.standard_normal((1, K, N, 2)).astype(np.float32)
    w = x[:, :, 2, :].copy().reshape(1, 1, K, 2)
    w[..., 1] = -w[..., 1]
    w[..., 1][x[:, :, 2, 1].reshape(1, 1, K) == 0] = -1.0
    out = oracle.cgemm_b1(w, x, 0, 1, N, K, 1)
    assert out[0, 0, 0, 2] == 2 * K and out[0, 1, 0, 2] == 0
