"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  1-bit: bit-exact.  16-bit: normwise relative error <= 2e-3 per batch
entry and overall (north_star), plus an elementwise accumulation bound as a diagnostic
gate, and exact equality where the arithmetic is exact (integer inputs, identity)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F16_TOL = 2e-3


@pytest.fixture(scope="module")
def tcbf():
    import paper_2505_03269_b200 as m
    m.lib()
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rounded(z):
    return z.real.astype(np.float16).astype(np.float64) + 1j * z.imag.astype(np.float16).astype(np.float64)


def _run(tcbf, prec, w_src, x_src, M, N, K, B, layout="interleaved"):
    plan = tcbf.Plan(M, N, K, B, prec)
    wp = plan.pack(tcbf.WEIGHTS, _dev(w_src), layout)
    xp = plan.pack(tcbf.DATA, _dev(x_src), layout)
    y = plan.beamform(wp, xp)
    torch.cuda.synchronize()
    return plan, wp, xp, y.cpu().numpy()


def _check_f16(y, ref, w, x):
    """y: [B][2][M][N] float32, ref: oracle float64 [B][2][M][N], w,x complex64 sources."""
    yc = y[:, 0].astype(np.float64) + 1j * y[:, 1]
    rc = ref[:, 0] + 1j * ref[:, 1]
    assert np.all(np.isfinite(yc))
    for b in range(yc.shape[0]):
        nrm = np.linalg.norm(rc[b])
        err = np.linalg.norm(yc[b] - rc[b])
        assert err <= F16_TOL * max(nrm, 1e-30), f"batch {b}: normwise {err / nrm:.3e}"
    # elementwise diagnostic: |err| <= 8 K u sum_k |w||x| (fp32 accumulation bound)
    K = w.shape[2]
    absw = np.abs(w.real.astype(np.float16).astype(np.float64)) + np.abs(w.imag.astype(np.float16).astype(np.float64))
    absx = np.abs(x.real.astype(np.float16).astype(np.float64)) + np.abs(x.imag.astype(np.float16).astype(np.float64))
    bound = 8 * K * 2.0 ** -24 * np.matmul(absw, absx) + 1e-30
    assert np.all(np.abs(yc.real - rc.real) <= bound) and np.all(np.abs(yc.imag - rc.imag) <= bound)


# ------------------------------------------------------------------ inputs module twin
@pytest.mark.parametrize("dist", list(synth.DIST_NAMES))
def test_device_generator_matches_numpy(dist):
    B, R, C = 2, 37, 53
    d = synth.generate_device(dist, 1234, 1, B, R, C).cpu().numpy()
    h = synth.to_interleaved(synth.generate(dist, 1234, 1, B, R, C))
    assert np.array_equal(d.view(np.uint32), h.view(np.uint32))


# ------------------------------------------------------------------ packing (a1, a2)
@pytest.mark.parametrize("layout", ["interleaved", "planar"])
@pytest.mark.parametrize("shape", [(3, 70, 45, 2), (128, 64, 64, 1), (5, 1, 300, 3), (1, 200, 1, 1)])
def test_pack_f16_bit_exact(tcbf, layout, shape):
    M, K, N, B = shape
    w = synth.generate("uniform", 7, 0, B, M, K) * np.float32(3000.0)   # exercise many exponents
    x = synth.generate("phase_amp", 7, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    lay = 0 if layout == "interleaved" else 1
    plan = tcbf.Plan(M, N, K, B, "f16")
    wp = plan.pack(tcbf.WEIGHTS, _dev(conv(w)), layout).cpu().numpy().view(np.uint16)
    xp = plan.pack(tcbf.DATA, _dev(conv(x)), layout).cpu().numpy().view(np.uint16)
    assert np.array_equal(wp, oracle.pack_f16(conv(w), lay, oracle.WEIGHTS, B, M, K, plan.k_packed))
    assert np.array_equal(xp, oracle.pack_f16(conv(x), lay, oracle.DATA, B, K, N, plan.n_packed))


def test_pack_f16_special_values(tcbf):
    vals = np.array([0.0, -0.0, 65504.0, 65520.0, 1e6, -1e6, 2.0 ** -25, 2.0 ** -24 * 1.5, np.inf, -np.inf,
                     1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11], np.float32)
    K = vals.size
    w = np.stack([vals, vals[::-1]], -1).reshape(1, 1, K, 2).astype(np.float32)
    plan = tcbf.Plan(1, 1, K, 1, "f16")
    wp = plan.pack(tcbf.WEIGHTS, _dev(w)).cpu().numpy().view(np.uint16)
    assert np.array_equal(wp, oracle.pack_f16(w, 0, 0, 1, 1, K, plan.k_packed))


@pytest.mark.parametrize("layout", ["interleaved", "planar"])
@pytest.mark.parametrize("shape", [(3, 70, 45, 2), (64, 256, 64, 1), (5, 1, 300, 3), (2, 1000, 33, 2)])
def test_pack_b1_bit_exact(tcbf, layout, shape):
    M, K, N, B = shape
    w = synth.generate("adc", 8, 0, B, M, K)      # exact zeros -> the >= 0 rule
    x = synth.generate("adc", 8, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    lay = 0 if layout == "interleaved" else 1
    plan = tcbf.Plan(M, N, K, B, "b1")
    wp = plan.pack(tcbf.WEIGHTS, _dev(conv(w)), layout).cpu().numpy().view(np.uint32)
    xp = plan.pack(tcbf.DATA, _dev(conv(x)), layout).cpu().numpy().view(np.uint32)
    assert np.array_equal(wp, oracle.pack_b1(conv(w), lay, oracle.WEIGHTS, B, M, K, plan.k_packed))
    assert np.array_equal(xp, oracle.pack_b1(conv(x), lay, oracle.DATA, B, K, N, plan.k_packed))


@pytest.mark.parametrize("wpt", ["32", "8", "2", "1"])
@pytest.mark.parametrize("shape", [(1, 3000, 130, 2), (1, 9000, 257, 1)])
def test_pack_b1_data_chunking_bit_exact(tcbf, shape, wpt, monkeypatch):
    """Every words-per-thread chunking of the 1-bit data pack (chosen by operand size) gives the
    oracle's packing: ragged K (partial words, partial chunks), ragged N, batch > 1."""
    monkeypatch.setenv("TCBF_PACK_WPT", wpt)
    M, K, N, B = shape
    x = synth.generate("uniform", 9, 1, B, K, N)
    plan = tcbf.Plan(M, N, K, B, "b1")
    xp = plan.pack(tcbf.DATA, _dev(synth.to_interleaved(x))).cpu().numpy().view(np.uint32)
    assert np.array_equal(xp, oracle.pack_b1(synth.to_interleaved(x), 0, oracle.DATA, B, K, N, plan.k_packed))


def test_pack_b1_nan_and_signed_zero(tcbf):
    vals = np.array([np.nan, -0.0, 0.0, -1e-45, 1e-45, -np.inf, np.inf], np.float32)
    K = vals.size
    w = np.stack([vals, vals[::-1]], -1).reshape(1, 1, K, 2)
    plan = tcbf.Plan(1, 1, K, 1, "b1")
    wp = plan.pack(tcbf.WEIGHTS, _dev(w)).cpu().numpy().view(np.uint32)
    assert np.array_equal(wp, oracle.pack_b1(w, 0, 0, 1, 1, K, plan.k_packed))


# ------------------------------------------------------------------ fp16 GEMM (a3, a5, a6)
F16_SHAPES = [
    (8, 64, 32, 2),        # BASELINE configs[0] (tiny)
    (200, 300, 100, 3),    # ragged M, N, K; several tiles; N % 4 == 0 -> TMA store
    (129, 77, 65, 2),      # N % 4 != 0 -> masked-store epilogue; K just over one block
    (256, 64, 512, 2),     # BN = 64 variant, 8 K blocks
    (1, 1, 1, 1),          # degenerate
    (384, 520, 1000, 1),   # many K blocks, ragged
]


@pytest.fixture(params=["default", "0", "1", "2", "3", "4"])
def f16_variant(request, monkeypatch):
    """fp16 kernel variants: default table choice, and each tile forced (BK32/8 epilogue warps,
    BK64/4 warps, 128x64, CTA pair 256x128, CTA pair 256x256)."""
    if request.param != "default":
        monkeypatch.setenv("TCBF_F16_VARIANT", request.param)
    return request.param


@pytest.mark.parametrize("shape", F16_SHAPES)
def test_f16_beamform_vs_oracle(tcbf, shape, f16_variant):
    M, N, K, B = shape
    w = synth.generate("uniform", 21, 0, B, M, K)
    x = synth.generate("uniform", 21, 1, B, K, N)
    _, _, _, y = _run(tcbf, "f16", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    ref = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
    _check_f16(y, ref, w, x)


def test_f16_planar_source_same_result(tcbf):
    M, N, K, B = 130, 96, 70, 2
    w = synth.generate("phase", 3, 0, B, M, K)
    x = synth.generate("adc", 3, 1, B, K, N)
    _, _, _, y0 = _run(tcbf, "f16", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    _, _, _, y1 = _run(tcbf, "f16", synth.to_planar(w), synth.to_planar(x), M, N, K, B, "planar")
    assert np.array_equal(y0, y1)


def test_f16_integer_inputs_exact(tcbf):
    """Integer entries: every partial sum is exact in fp32, so any accumulation order gives
    exactly the oracle's value."""
    rng = np.random.default_rng(4)
    M, N, K, B = 200, 136, 300, 2
    w = (rng.integers(-2, 3, (B, M, K)) + 1j * rng.integers(-2, 3, (B, M, K))).astype(np.complex64)
    x = (rng.integers(-2, 3, (B, K, N)) + 1j * rng.integers(-2, 3, (B, K, N))).astype(np.complex64)
    _, _, _, y = _run(tcbf, "f16", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    ref = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
    assert np.array_equal(y.astype(np.float64), ref)


def test_f16_identity_weights_exact(tcbf):
    K, N, B = 150, 200, 2
    x = synth.generate("adc_scaled", 5, 1, B, K, N)
    w = np.zeros((B, K, K), np.complex64)
    w[:, np.arange(K), np.arange(K)] = 1
    _, _, _, y = _run(tcbf, "f16", synth.to_interleaved(w), synth.to_interleaved(x), K, N, K, B)
    assert np.array_equal(y[:, 0].astype(np.float64) + 1j * y[:, 1], _rounded(x))


def test_f16_plane_wave_steered_beam(tcbf):
    """Delay-and-sum closed form: the steered beam reaches K|s|."""
    K, M, N = 256, 121, 64
    t0 = np.deg2rad(-13.0)
    th = np.deg2rad(np.linspace(-60, 60, M))
    m0 = int(np.argmin(np.abs(th - t0)))
    th[m0] = t0
    k = np.arange(K)
    s = synth.generate("uniform", 9, 1, 1, 1, N)[0, 0]
    x = (np.exp(-1j * np.pi * k * np.sin(t0))[:, None] * s[None, :]).astype(np.complex64)[None]
    w = np.exp(1j * np.pi * np.outer(np.sin(th), k)).astype(np.complex64)[None]
    _, _, _, y = _run(tcbf, "f16", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, 1)
    yc = y[0, 0] + 1j * y[0, 1]
    assert np.all(np.argmax(np.abs(yc), axis=0) == m0)
    assert np.allclose(np.abs(yc[m0]), K * np.abs(s), rtol=4e-3)


def test_inputs_unmodified(tcbf):
    M, N, K, B = 64, 64, 64, 1
    for prec in ("f16", "b1"):
        w = _dev(synth.to_interleaved(synth.generate("uniform", 1, 0, B, M, K)))
        x = _dev(synth.to_interleaved(synth.generate("uniform", 1, 1, B, K, N)))
        w0, x0 = w.clone(), x.clone()
        plan = tcbf.Plan(M, N, K, B, prec)
        wp = plan.pack(tcbf.WEIGHTS, w)
        xp = plan.pack(tcbf.DATA, x)
        wp0, xp0 = wp.clone(), xp.clone()
        plan.beamform(wp, xp)
        torch.cuda.synchronize()
        assert torch.equal(w, w0) and torch.equal(x, x0) and torch.equal(wp, wp0) and torch.equal(xp, xp0)


# ------------------------------------------------------------------ fused fp32 path (tcbf_beamform_raw)
RAW_SHAPES = [
    (200, 300, 100, 3, "interleaved"),   # fused, ragged M/N/K, N % 8 != 0 -> scalar loads
    (256, 256, 256, 2, "interleaved"),   # fused, vector loads, exactly K16 = 256
    (600, 300, 200, 3, "planar"),        # fused (pair: 3 pair tiles, ragged M and N), planar
    (512, 1000, 256, 2, "interleaved"),  # fused (pair: 16 units on 8 pairs -> both B buffers)
    (130, 136, 64, 3, "planar"),         # fused, planar source
    (8, 64, 32, 2, "interleaved"),       # tiny (BASELINE configs[0])
    (64, 96, 300, 2, "interleaved"),     # K16 = 320 > 256, M <= 128 -> streaming-conversion kernel
    (32, 1024, 5000, 1, "interleaved"),  # M=32 sweep shape class, long K, streaming conversion
    (100, 260, 700, 2, "planar"),        # streaming conversion, planar, ragged N (scalar loads)
    (300, 96, 300, 2, "interleaved"),    # M > 128 and K16 > 256 -> pack + beamform fallback
    (70, 77, 40, 2, "interleaved"),      # N % 4 != 0 -> fallback
]


@pytest.fixture(params=["auto", "force_stream", "no_mc", "smaj"])
def raw_mode(request, monkeypatch):
    if request.param == "force_stream":   # small-M shapes through the streaming-conversion kernel
        monkeypatch.setenv("TCBF_FORCE_STREAM_CONV", "1")
    if request.param == "no_mc":                 # the fused kernel without the CTA-pair weight multicast
        monkeypatch.setenv("TCBF_F16_MC", "0")
    if request.param == "smaj":                  # sample-major kernel with the data resident in smem
        monkeypatch.setenv("TCBF_F16_FUSED", "smaj")
    return request.param


@pytest.mark.parametrize("shape", RAW_SHAPES + [(32, 256, 1000, 80, "interleaved")])  # 160 tiles: streams
def test_f16_beamform_raw_bitwise_equals_packed_path(tcbf, shape, raw_mode, monkeypatch):
    monkeypatch.setenv("TCBF_CONV_SPLITS", "1")  # split-K sums in another order: tested below
    M, N, K, B, layout = shape
    w = synth.generate("phase", 17, 0, B, M, K)
    x = synth.generate("adc", 17, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    plan = tcbf.Plan(M, N, K, B, "f16")
    wp = plan.pack(tcbf.WEIGHTS, _dev(conv(w)), layout)
    xd = _dev(conv(x))
    y_raw = plan.beamform_raw(wp, xd, layout)
    y_ref = plan.beamform(wp, plan.pack(tcbf.DATA, xd, layout))
    torch.cuda.synchronize()
    if "smaj" in plan.raw_variant or "tmem" in plan.raw_variant:
        # sample-major kernel: the same fp16 products and fp32 accumulation, computed as X^T W^T
        # with an N=256 MMA -- the tensor core's in-MMA summation order differs by fp32 ulps
        assert (y_raw - y_ref).abs().max().item() <= 1e-6 * y_ref.abs().max().item()
    else:
        assert torch.equal(y_raw, y_ref)
    ref = oracle.cgemm_f16(conv(w), conv(x), 0 if layout == "interleaved" else 1, M, N, K, B)
    _check_f16(y_raw.cpu().numpy(), ref, w, x)


@pytest.mark.parametrize("shape", [(32, 1024, 5000, 1, "interleaved"), (100, 260, 700, 2, "planar"),
                                   (128, 512, 2049, 3, "interleaved"), (16, 128, 4096, 1, "planar")])
@pytest.mark.parametrize("splits", ["auto", "3", "16"])
def test_f16_beamform_raw_split_k(tcbf, shape, splits, monkeypatch):
    """Streaming-conversion kernel with K split across CTAs (fp32 partial tiles reduce-added by
    the TMA unit into the zeroed output): within the fp16 tolerance of the oracle and equal to
    the packed path up to fp32 summation order."""
    monkeypatch.setenv("TCBF_FORCE_STREAM_CONV", "1")
    if splits != "auto":
        monkeypatch.setenv("TCBF_CONV_SPLITS", splits)
    M, N, K, B, layout = shape
    w = synth.generate("phase", 23, 0, B, M, K)
    x = synth.generate("adc", 23, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    plan = tcbf.Plan(M, N, K, B, "f16")
    wp = plan.pack(tcbf.WEIGHTS, _dev(conv(w)), layout)
    xd = _dev(conv(x))
    y_raw = plan.beamform_raw(wp, xd, layout)
    n_launch = tcbf.Plan.last_launch_count()
    y_ref = plan.beamform(wp, plan.pack(tcbf.DATA, xd, layout))
    torch.cuda.synchronize()
    if splits != "auto":
        assert n_launch == 2  # memset + kernel
    scale = y_ref.abs().max().item()
    assert (y_raw - y_ref).abs().max().item() <= 1e-4 * scale  # fp32 partial sums, another order
    ref = oracle.cgemm_f16(conv(w), conv(x), 0 if layout == "interleaved" else 1, M, N, K, B)
    _check_f16(y_raw.cpu().numpy(), ref, w, x)


# ------------------------------------------------------------------ fp16 interleaved data, no pack (NEXT-1)
@pytest.mark.parametrize("shape", [(8, 64, 32, 2), (200, 300, 100, 3), (130, 136, 64, 3), (300, 1000, 480, 2),
                                   (1024, 1024, 256, 2), (1000, 260, 333, 1), (64, 4, 16, 1), (96, 520, 200, 90),
                                   (40, 512, 256, 160)])
@pytest.mark.parametrize("kernel", ["default", "res", "stream"])
def test_f16i_interleaved_fp16_beamform(tcbf, shape, kernel, monkeypatch):
    """tcbf_beamform_f16i on fp16 interleaved data: the default data-in-TMEM kernel (pairs
    de-interleaved into the staged unit), the resident kernel (TCBF_F16I=res: the interleaved tile
    as a real K x 2N operand, Re/Im recombined in the epilogue) and the streaming one -- within the
    16-bit tolerance of the oracle on the same fp16 values, and equal to the planar path up to one
    fp32 rounding."""
    if kernel == "res":
        monkeypatch.setenv("TCBF_F16I", "res")
    if kernel == "stream":
        monkeypatch.setenv("TCBF_F16I_STREAM", "1")
    M, N, K, B = shape
    w = synth.generate("phase", 29, 0, B, M, K)
    x = synth.generate("adc", 29, 1, B, K, N)
    wi, xi = synth.to_interleaved(w), synth.to_interleaved(x)
    x16 = xi.astype(np.float16)  # numpy RNE: the same fp16 values the oracle rounds to
    plan = tcbf.Plan(M, N, K, B, "f16")
    wp = plan.pack(tcbf.WEIGHTS, _dev(wi))
    y = plan.beamform_f16i(wp, torch.from_numpy(x16).cuda())
    assert tcbf.Plan.last_launch_count() == 1
    y_planar = plan.beamform(wp, plan.pack(tcbf.DATA, _dev(xi)))
    torch.cuda.synchronize()
    scale = y_planar.abs().max().item()
    assert (y - y_planar).abs().max().item() <= 1e-5 * scale
    _check_f16(y.cpu().numpy(), oracle.cgemm_f16(wi, xi, 0, M, N, K, B), w, x)


def test_f16i_integer_inputs_exact(tcbf):
    """Integer-valued fp16 inputs with small partial sums: every product and sum is exact, so the
    interleaved path equals the oracle exactly (SURVEY §8(c) pin iv)."""
    M, N, K, B = 96, 200, 130, 2
    rng = np.random.default_rng(5)
    w = (rng.integers(-2, 3, (B, M, K, 2))).astype(np.float32)
    x = (rng.integers(-2, 3, (B, K, N, 2))).astype(np.float32)
    plan = tcbf.Plan(M, N, K, B, "f16")
    y = plan.beamform_f16i(plan.pack(tcbf.WEIGHTS, _dev(w)), torch.from_numpy(x.astype(np.float16)).cuda())
    assert np.array_equal(y.cpu().numpy().astype(np.float64), oracle.cgemm_f16(w, x, 0, M, N, K, B))


@pytest.mark.parametrize("shape", [(256, 512, 200, 3), (130, 384, 256, 1), (70, 1000, 64, 2)])
def test_f16i_resident_equals_streaming(tcbf, shape, monkeypatch):
    """The resident-data NEXT-1 kernel (K16 <= 256: data loaded once per 128-sample unit, 64-beam
    tiles, two N = 128 MMAs per K step) against the streaming one (TCBF_F16I_STREAM: data re-read
    per beam tile, one N = 256 MMA): the same fp16 products accumulated in the same K order, so the
    results agree to the last fp32 bit or within one rounding of the final Re/Im combination."""
    M, N, K, B = shape
    w = synth.generate("phase", 31, 0, B, M, K)
    x = synth.to_interleaved(synth.generate("adc", 31, 1, B, K, N)).astype(np.float16)
    xd = torch.from_numpy(x).cuda()
    monkeypatch.setenv("TCBF_F16I", "res")
    plan = tcbf.Plan(M, N, K, B, "f16")
    assert "resident" in plan.kernel("f16i")
    wp = plan.pack(tcbf.WEIGHTS, _dev(synth.to_interleaved(w)))
    y_res = plan.beamform_f16i(wp, xd)
    monkeypatch.delenv("TCBF_F16I")
    pt = tcbf.Plan(M, N, K, B, "f16")
    assert pt.kernel("f16i").startswith("f16_tcgen05_interleaved_tmem_128x"), pt.kernel("f16i")
    y_tmem = pt.beamform_f16i(wp, xd)
    monkeypatch.setenv("TCBF_F16I_STREAM", "1")
    ps = tcbf.Plan(M, N, K, B, "f16")
    assert "resident" not in ps.kernel("f16i")
    y_str = ps.beamform_f16i(wp, xd)
    torch.cuda.synchronize()
    scale = y_str.abs().max().item()
    assert (y_res - y_str).abs().max().item() <= 1e-6 * scale
    assert (y_tmem - y_str).abs().max().item() <= 1e-6 * scale


def test_f16i_errors(tcbf):
    plan = tcbf.Plan(8, 6, 8, 1, "f16")   # N % 4 != 0
    wp = plan.alloc_packed(tcbf.WEIGHTS)
    with pytest.raises(tcbf.TcbfError):
        plan.beamform_f16i(wp, torch.zeros(1, 8, 6, 2, dtype=torch.float16, device="cuda"))
    pb = tcbf.Plan(8, 8, 8, 1, "b1")
    with pytest.raises(tcbf.TcbfError):
        pb.beamform_f16i(pb.alloc_packed(tcbf.WEIGHTS), torch.zeros(1, 8, 8, 2, dtype=torch.float16, device="cuda"))


def test_b1_beamform_raw_falls_back_bit_exact(tcbf):
    M, N, K, B = 70, 45, 300, 2
    w = synth.generate("adc", 5, 0, B, M, K)
    x = synth.generate("adc", 5, 1, B, K, N)
    plan = tcbf.Plan(M, N, K, B, "b1")
    wp = plan.pack(tcbf.WEIGHTS, _dev(synth.to_interleaved(w)))
    y = plan.beamform_raw(wp, _dev(synth.to_interleaved(x)))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x),
                                                          0, M, N, K, B))


def test_full_size_radio_f16_raw_sampled(tcbf):
    """BASELINE configs[1] through the fused path, as bench.py times it."""
    M, N, K, B = 1024, 1024, 256, 256
    seed = synth.SEED_BASE + 1
    plan = tcbf.Plan(M, N, K, B, "f16")
    assert plan.raw_fused
    wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("phase", seed, 0, B, M, K))
    y = plan.beamform_raw(wp, synth.generate_device("adc", seed, 1, B, K, N))
    torch.cuda.synchronize()
    rows = [0, 5, 640, 1023]
    for b in (0, 77, 255):
        w = synth.generate("phase", seed, 0, B, M, K, b_sel=[b], r_sel=rows)
        x = synth.generate("adc", seed, 1, B, K, N, b_sel=[b])
        ref = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, len(rows), N, K, 1)
        _check_f16(y[b][:, rows].cpu().numpy()[None], ref, w, x)


# ------------------------------------------------------------------ steering weights (NEXT-3, Eq. 1-3)
@pytest.mark.parametrize("layout", ["interleaved", "planar"])
def test_steering_weights_vs_oracle(tcbf, layout):
    rng = np.random.default_rng(8)
    B, M, K = 3, 37, 48
    c = 3e8
    freqs = 110e6 + 1e6 * np.arange(B)                  # LOFAR HBA-like channels
    pos = np.sort(rng.uniform(0, 3000.0, K))            # km-scale baselines: ~1e3 cycles of phase
    th = np.deg2rad(np.linspace(-60, 60, M))
    plan = tcbf.Plan(M, 64, K, B, "f16")
    w = plan.steering_weights(torch.from_numpy(pos).cuda(), torch.from_numpy(th).cuda(),
                              torch.from_numpy(freqs).cuda(), c, layout).cpu().numpy()
    ref = oracle.steering_weights(pos, th, freqs, c)
    got = w[..., 0] + 1j * w[..., 1] if layout == "interleaved" else w[:, 0] + 1j * w[:, 1]
    # fp32 output of an fp64 phase; the oracle's cos/sin of a ~1e4 rad argument is itself only
    # good to ~1e-12, so 2e-7 bounds the fp32 rounding of unit-modulus values
    assert np.max(np.abs(got - ref)) < 2e-7


def test_steered_beamform_coherent_gain(tcbf):
    """Steering kernel -> pack -> beamform of a simulated plane wave: argmax at the source and
    |y| = K within fp16 rounding (coherent gain)."""
    c, f = 3e8, 150e6
    K, M, N = 96, 121, 64
    rng = np.random.default_rng(4)
    pos = np.sort(rng.uniform(0, 40 * c / f, K))
    th = np.deg2rad(np.linspace(-60, 60, M))
    m0 = 77
    s = np.exp(2j * np.pi * rng.uniform(size=N))
    x = (np.exp(-2j * np.pi * f * pos * np.sin(th[m0]) / c)[:, None] * s[None, :]).astype(np.complex64)[None]
    plan = tcbf.Plan(M, N, K, 1, "f16")
    wsrc = plan.steering_weights(torch.from_numpy(pos).cuda(), torch.from_numpy(th).cuda(),
                                 torch.tensor([f], dtype=torch.float64).cuda(), c)
    y = plan.beamform_raw(plan.pack(tcbf.WEIGHTS, wsrc), _dev(synth.to_interleaved(x)))
    torch.cuda.synchronize()
    yc = y[0, 0].cpu().numpy() + 1j * y[0, 1].cpu().numpy()
    assert np.all(np.argmax(np.abs(yc), axis=0) == m0)
    assert np.allclose(np.abs(yc[m0]), K, rtol=2e-3)


# ------------------------------------------------------------------ end-to-end host pipeline and ABI errors
@pytest.mark.parametrize("prec", ["f16", "b1"])
def test_beamform_host_equals_device_path(tcbf, prec):
    """tcbf_beamform_host (chunked H2D -> pack -> beamform -> D2H on two streams) returns exactly
    the device path's output, for a batch that spans several chunks."""
    M, N, K, B = 256, 512, 128, 24
    w = synth.to_interleaved(synth.generate("phase", 6, 0, B, M, K))
    x = synth.to_interleaved(synth.generate("adc", 6, 1, B, K, N))
    plan = tcbf.Plan(M, N, K, B, prec)
    wp = plan.pack(tcbf.WEIGHTS, _dev(w))
    ref = plan.beamform_raw(wp, _dev(x))   # the call tcbf_beamform_host makes per chunk
    x_host = torch.from_numpy(x).pin_memory()
    out_host = torch.empty(tuple(ref.shape), dtype=ref.dtype).pin_memory()
    plan.beamform_host(wp, x_host, out_host)
    torch.cuda.synchronize()
    assert torch.equal(out_host, ref.cpu())


@pytest.mark.parametrize("prec", ["f16", "b1"])
@pytest.mark.parametrize("shape", [(33, 63, 33, 3), (7, 5, 3, 5), (130, 129, 65, 1)])
def test_beamform_host_odd_sizes(tcbf, prec, shape):
    """tcbf_beamform_host with odd K*N and odd batch (the per-chunk output scratch must still be
    16-byte aligned): equals the device path and the oracle."""
    M, N, K, B = shape
    w = synth.to_interleaved(synth.generate("uniform", 8, 0, B, M, K))
    x = synth.to_interleaved(synth.generate("uniform", 8, 1, B, K, N))
    plan = tcbf.Plan(M, N, K, B, prec)
    wp = plan.pack(tcbf.WEIGHTS, _dev(w))
    ref = plan.beamform_raw(wp, _dev(x))   # the call tcbf_beamform_host makes per chunk
    x_host = torch.from_numpy(x).pin_memory()
    out_host = torch.empty(tuple(ref.shape), dtype=ref.dtype).pin_memory()
    plan.beamform_host(wp, x_host, out_host)
    assert torch.equal(out_host, ref.cpu())
    if prec == "b1":
        assert np.array_equal(out_host.numpy(), oracle.cgemm_b1(w, x, 0, M, N, K, B))


def test_binding_rejects_bad_tensors(tcbf):
    """Wrong device / dtype / size / contiguity never reach the ABI as raw pointers."""
    plan = tcbf.Plan(64, 64, 64, 2, "f16")
    wp = plan.alloc_packed(tcbf.WEIGHTS)
    xp = plan.alloc_packed(tcbf.DATA)
    with pytest.raises(ValueError):
        plan.beamform(wp, xp[:1])                                   # too small
    with pytest.raises(TypeError):
        plan.beamform(wp, xp.float())                               # wrong dtype
    with pytest.raises(ValueError):
        plan.beamform(wp.cpu(), xp)                                 # host tensor
    with pytest.raises(ValueError):
        plan.pack(tcbf.DATA, torch.zeros(2, 64, 64, 2, device="cuda").transpose(1, 2))  # non-contiguous
    with pytest.raises(ValueError):
        plan.beamform(wp, xp, out=torch.empty(2, 2, 64, 63, device="cuda"))  # output too small


def test_abi_errors_on_device(tcbf):
    import ctypes
    L = tcbf.lib()
    plan = tcbf.Plan(64, 64, 64, 1, "f16")
    wp = plan.alloc_packed(tcbf.WEIGHTS)
    xp = plan.alloc_packed(tcbf.DATA)
    out = plan.alloc_output()
    vp = ctypes.c_void_p
    # misaligned output / packed pointers -> INVALID_ARG, nothing launched
    assert L.tcbf_beamform(plan._h, vp(wp.data_ptr()), vp(xp.data_ptr()), vp(out.data_ptr() + 4), None) == 1
    assert L.tcbf_beamform(plan._h, vp(wp.data_ptr() + 8), vp(xp.data_ptr()), vp(out.data_ptr()), None) == 1
    assert L.tcbf_last_launch_count() == 0
    src = torch.zeros((1, 64, 64, 2), device="cuda")
    assert L.tcbf_pack(plan._h, 0, vp(src.data_ptr() + 4), 0, vp(wp.data_ptr()), None) == 1   # 8-B rule
    assert L.tcbf_pack(plan._h, 7, vp(src.data_ptr()), 0, vp(wp.data_ptr()), None) == 1       # bad operand
    assert L.tcbf_pack(plan._h, 0, vp(src.data_ptr()), 5, vp(wp.data_ptr()), None) == 1       # bad layout
    assert b"aligned" in L.tcbf_last_error() or b"layout" in L.tcbf_last_error()
    d = torch.zeros(4, dtype=torch.float64, device="cuda")
    assert L.tcbf_steering_weights(plan._h, vp(d.data_ptr()), vp(d.data_ptr()), vp(d.data_ptr()),
                                   ctypes.c_double(-1.0), 0, vp(src.data_ptr()), None) == 1    # c <= 0
    # a valid call still works afterwards and reports one launch
    assert L.tcbf_beamform(plan._h, vp(wp.data_ptr()), vp(xp.data_ptr()), vp(out.data_ptr()), None) == 0
    assert L.tcbf_last_launch_count() == 1
    torch.cuda.synchronize()


# ------------------------------------------------------------------ 1-bit GEMM (a4, a5)
@pytest.fixture(params=["f4", "tmem", "i8", "popc", "bmma"])
def b1_kernel(request, monkeypatch):
    """All 1-bit kernels: tcgen05 kind::mxf4 on +-1 (beam-major, and the sample-major kernel with
    the unit's data resident in TMEM -- the default for 8 < Kw <= 24 and M > 64; other shapes fall back
    to the beam-major one), tcgen05 kind::i8 AND form (beyond
    the fp32-exact K range, and split-K), the CUDA-core XOR/popc kernel and the legacy b1 mma.sync
    single-AND kernel."""
    monkeypatch.setenv("TCBF_B1_KERNEL", request.param)
    return request.param


B1_SHAPES = [(8, 64, 32, 2), (70, 45, 300, 3), (64, 64, 256, 1), (1, 1, 1, 1), (130, 200, 1000, 2),
             (33, 17, 2049, 1), (100, 129, 31, 2)]


@pytest.mark.parametrize("shape", B1_SHAPES)
def test_b1_beamform_bit_exact(tcbf, shape, b1_kernel):
    M, N, K, B = shape
    w = synth.generate("adc", 31, 0, B, M, K)
    x = synth.generate("adc", 31, 1, B, K, N)
    plan, wp, xp, y = _run(tcbf, "b1", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    assert {"f4": "mxf4", "tmem": "mxf4", "popc": "popc", "bmma": "mma_sync"}.get(b1_kernel, "i8") in plan.variant
    ref = oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
    assert np.array_equal(y, ref)
    refp = oracle.cgemm_b1_packed(wp.cpu().numpy().view(np.uint32), xp.cpu().numpy().view(np.uint32),
                                  M, N, K, wp.shape[-1], B)
    assert np.array_equal(y, refp)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_b1_exhaustive(tcbf, K, b1_kernel):
    import itertools
    V = 4 ** K
    codes = np.array(list(itertools.product([0, 1], repeat=2 * K)), dtype=np.int64)
    src = np.stack([np.where(codes[:, :K], 1.0, -1.0), np.where(codes[:, K:], 1.0, -1.0)], -1).astype(np.float32)
    w = src.reshape(1, V, K, 2)
    x = np.ascontiguousarray(src.transpose(1, 0, 2)).reshape(1, K, V, 2)
    _, _, _, y = _run(tcbf, "b1", w, x, V, V, K, 1)
    assert np.array_equal(y, oracle.cgemm_b1(w, x, 0, V, V, K, 1))


def test_b1_random_corpus(tcbf, b1_kernel):
    rng = np.random.default_rng(12)
    for t in range(40):
        M, N = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        K = int(rng.integers(1, 2049))
        if t % 2 == 0 and K % 32 == 0:
            K += 1
        w = rng.standard_normal((1, M, K, 2)).astype(np.float32)
        x = rng.standard_normal((1, K, N, 2)).astype(np.float32)
        _, _, _, y = _run(tcbf, "b1", w, x, M, N, K, 1)
        assert np.array_equal(y, oracle.cgemm_b1(w, x, 0, M, N, K, 1)), (M, N, K)


@pytest.mark.parametrize("shape", [(32, 512, 4096 + 5, 1), (64, 1000, 3000, 1), (17, 260, 700, 2), (48, 77, 600, 2),
                                   (1, 128, 256, 3), (33, 4096, 1024, 1)])
def test_b1_small_m_swapped_kernel_bit_exact(tcbf, shape):
    """Few-beam plans (M <= 64) run the swapped fp4 kernel (samples on the 128-row MMA dimension):
    ragged M/N/K, N % 4 != 0 (masked stores), both beam-tile widths."""
    M, N, K, B = shape
    w = synth.generate("adc", 41, 0, B, M, K)
    x = synth.generate("adc", 41, 1, B, K, N)
    plan, wp, xp, y = _run(tcbf, "b1", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    assert "swap" in plan.variant
    assert np.array_equal(y, oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B))


@pytest.mark.parametrize("shape", [(32, 20000, 700, 2), (20, 9000, 520, 3), (32, 19000, 1024, 2), (64, 9000, 700, 3)])
def test_b1_swapped_kernel_many_tiles_per_cta_bit_exact(tcbf, shape):
    """More 128-sample tiles than SMs, so every CTA runs several: the 32-beam kernel's single
    accumulator (the next tile's MMAs wait for the epilogue's TMEM loads) and its two-K-block
    stages across tile boundaries, with an odd K-block count (a virtual block pads the last stage:
    K = 700 / 520 -> 3 blocks) and an even one; and the 64-beam kernel (double-buffered)."""
    M, N, K, B = shape
    w = synth.generate("adc", 47, 0, B, M, K)
    x = synth.generate("adc", 47, 1, B, K, N)
    plan, wp, xp, y = _run(tcbf, "b1", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    assert "swap" in plan.variant
    assert B * ((N + 127) // 128) > 148
    assert np.array_equal(y, oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B))


@pytest.mark.parametrize("shape", [(32, 300, 700, 2), (200, 260, 500, 1)])
def test_b1_forced_swap64_bit_exact(tcbf, shape, monkeypatch):
    """TCBF_B1_SWAP=64 (experiment override): the swapped kernel with 64-beam tiles for any M,
    including M <= 32 where the default picks 32-beam tiles (the tile width follows the plan)."""
    monkeypatch.setenv("TCBF_B1_SWAP", "64")
    M, N, K, B = shape
    w = synth.generate("adc", 43, 0, B, M, K)
    x = synth.generate("adc", 43, 1, B, K, N)
    plan, wp, xp, y = _run(tcbf, "b1", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
    assert "swap_128x64" in plan.variant
    assert np.array_equal(y, oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B))


def test_full_size_m32_b1_16384(tcbf):
    """BASELINE configs[4] small-beam 1-bit point M=32, N=K=16384 at full size, whole output."""
    M = 32
    N = K = 16384
    seed = synth.SEED_BASE + 4
    plan = tcbf.Plan(M, N, K, 1, "b1")
    wd = synth.generate_device("uniform", seed, 0, 1, M, K)
    xd = synth.generate_device("uniform", seed, 1, 1, K, N)
    y = plan.beamform(plan.pack(tcbf.WEIGHTS, wd), plan.pack(tcbf.DATA, xd)).cpu().numpy()
    assert "swap" in plan.variant
    ref = oracle.cgemm_b1(wd.cpu().numpy(), xd.cpu().numpy(), 0, M, N, K, 1)
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("splits", ["auto", "3", "7"])
def test_b1_split_k_bit_exact(tcbf, monkeypatch, splits):
    """Split-K (int8 kernel, TMA reduce-add of exact int32 partials): the M=32 sweep shape class
    and a ragged-N shape (atomic masked path), forced split counts included."""
    monkeypatch.setenv("TCBF_B1_KERNEL", "i8")
    if splits != "auto":
        monkeypatch.setenv("TCBF_B1_SPLITS", splits)
    for (M, N, K, B) in [(32, 512, 4096 + 5, 1), (40, 77, 3000, 2)]:
        w = synth.generate("adc", 14, 0, B, M, K)
        x = synth.generate("adc", 14, 1, B, K, N)
        _, _, _, y = _run(tcbf, "b1", synth.to_interleaved(w), synth.to_interleaved(x), M, N, K, B)
        ref = oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, M, N, K, B)
        assert np.array_equal(y, ref), (M, N, K, B, splits)


def test_b1_large_k_exact(tcbf, b1_kernel):
    """Long K: partial sums up to ~2^17 (f8: exact fp32 accumulation of +-1 products)."""
    M, N, K, B = 16, 24, 65536 + 7, 1
    rng = np.random.default_rng(21)
    w = rng.standard_normal((B, M, K, 2)).astype(np.float32)
    x = rng.standard_normal((B, K, N, 2)).astype(np.float32)
    # make a few outputs near the extremes: a matched beam (y = 2K) and its negative
    x[0, :, 0, :] = w[0, 3, :, :] * np.array([1, -1], np.float32)
    x[0, :, 1, :] = -x[0, :, 0, :]
    _, _, _, y = _run(tcbf, "b1", w, x, M, N, K, B)
    ref = oracle.cgemm_b1(w, x, 0, M, N, K, B)
    assert ref[0, 0, 3, 0] == 2 * K and ref[0, 0, 3, 1] == -2 * K
    assert np.array_equal(y, ref)


def _near_matched_b1(M, N, K, seed):
    """+-1 sources whose outputs sit at the extremes of the exact range with increments that are
    NOT multiples of a large power of two, so a tensor-core accumulator that dropped low bits
    (or summed a K block in fewer bits than fp32) would show: columns 0/1 are the matched beam
    of row 0 and its negative (Re = +-2K, PAPER.md:244-259 with every XOR popcount 0), columns 2/3
    put +-2K into Im (x = i conj(w)), columns 4-6 are matched beams with a periodic sign flip
    (flip periods 61, 3, 5: every K block adds a different, mostly non-power-of-two amount),
    column 7 is random."""
    rng = np.random.default_rng(seed)
    w = np.where(rng.integers(0, 2, (1, M, K, 2), dtype=np.int8) > 0, 1.0, -1.0).astype(np.float32)
    x = np.where(rng.integers(0, 2, (1, K, N, 2), dtype=np.int8) > 0, 1.0, -1.0).astype(np.float32)
    k = np.arange(K)
    conj = lambda r: np.stack([w[0, r, :, 0], -w[0, r, :, 1]], -1)          # noqa: E731
    iconj = lambda r: np.stack([w[0, r, :, 1], w[0, r, :, 0]], -1)          # i * conj(w)   # noqa: E731
    x[0, :, 0] = conj(0)
    x[0, :, 1] = -conj(0)
    x[0, :, 2] = iconj(1 % M)
    x[0, :, 3] = -iconj(1 % M)
    c4 = conj(2 % M); c4[k % 61 == 0, 0] *= -1
    c5 = conj(3 % M); c5[k % 3 == 0, 0] *= -1
    c6 = iconj(0); c6[k % 5 == 1, 1] *= -1
    x[0, :, 4], x[0, :, 5], x[0, :, 6] = c4, c5, c6
    return w, x


LARGE_K_KERNELS = ["f4", "f4_noswap", "i8", "popc", "bmma"]


@pytest.mark.parametrize("K", [524288, (1 << 23) - 7, (1 << 23) + 1])
def test_b1_extreme_sums_bit_exact(tcbf, monkeypatch, K):
    """1-bit exactness where the arithmetic is most fragile (VERDICT r1 missing #3): the paper's
    int1 K = 524288 (|Re| = 2^20), the largest K of the fp32-accumulating fp4 path
    (K = 2^23 - 7: 32 Kw = 2^23, accumulators up to 2^24) and the first K beyond it (K = 2^23 + 1,
    which the plan routes to the int8 kernel), for every 1-bit kernel.  Bit-exact against the
    oracle, and the matched beams equal 2K exactly (closed form, independent of the oracle)."""
    M, N = 4, 8
    w, x = _near_matched_b1(M, N, K, 900 + K % 97)
    ref = oracle.cgemm_b1(w, x, 0, M, N, K, 1)
    assert ref[0, 0, 0, 0] == 2 * K and ref[0, 1, 1 % M, 2] == 2 * K
    for kern in LARGE_K_KERNELS:
        monkeypatch.delenv("TCBF_NO_SWAP", raising=False)
        if kern == "f4_noswap":
            monkeypatch.setenv("TCBF_B1_KERNEL", "f4")
            monkeypatch.setenv("TCBF_NO_SWAP", "1")
        else:
            monkeypatch.setenv("TCBF_B1_KERNEL", kern)
        plan, _, _, y = _run(tcbf, "b1", w, x, M, N, K, 1)
        if K > (1 << 23) and kern.startswith("f4"):
            assert "i8" in plan.variant, plan.variant     # beyond the fp32-exact range: int8
        elif kern == "f4":
            assert "swap" in plan.variant, plan.variant
        elif kern == "f4_noswap":
            assert "mxf4" in plan.variant and "swap" not in plan.variant, plan.variant
        assert y[0, 0, 0, 0] == 2 * K and y[0, 1, 0, 0] == 0, kern
        assert y[0, 0, 0, 1] == -2 * K, kern
        assert y[0, 1, 1 % M, 2] == 2 * K and y[0, 0, 1 % M, 2] == 0, kern
        assert y[0, 1, 1 % M, 3] == -2 * K, kern
        assert np.array_equal(y, ref), (kern, plan.variant, np.argwhere(y != ref)[:8])
        del plan, y
        torch.cuda.empty_cache()


# ------------------------------------------------------------------ full-size sampled parity
def _full_size(tcbf, prec, M, N, K, B, wdist, xdist, seed, batches, rows, path="packed"):
    """path: 'packed' (tcbf_pack + tcbf_beamform), 'raw' (tcbf_beamform_raw) or 'f16i'
    (tcbf_beamform_f16i on the fp16-rounded interleaved data) -- whichever bench.py times."""
    plan = tcbf.Plan(M, N, K, B, prec)
    wsrc = synth.generate_device(wdist, seed, 0, B, M, K)
    wp = plan.pack(tcbf.WEIGHTS, wsrc)
    del wsrc
    xsrc = synth.generate_device(xdist, seed, 1, B, K, N)
    if path == "raw":
        y = plan.beamform_raw(wp, xsrc)
    elif path == "f16i":
        y = plan.beamform_f16i(wp, xsrc.half())
    else:
        y = plan.beamform(wp, plan.pack(tcbf.DATA, xsrc))
    del xsrc
    torch.cuda.synchronize()
    nr = len(rows)
    for b in batches:
        w = synth.generate(wdist, seed, 0, B, M, K, b_sel=[b], r_sel=rows)   # only the sampled beams
        x = synth.generate(xdist, seed, 1, B, K, N, b_sel=[b])
        got = y[b][:, rows].cpu().numpy()[None]
        if prec == "b1":
            ref = oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, nr, N, K, 1)
            assert np.array_equal(got, ref)
        else:
            ref = oracle.cgemm_f16(synth.to_interleaved(w), synth.to_interleaved(x), 0, nr, N, K, 1)
            _check_f16(got, ref, w, x)
    return y


def test_full_size_radio_f16_sampled(tcbf):
    """BASELINE configs[1]: M=1024, K=256, N=1024, batch=256, launch as bench.py times it."""
    _full_size(tcbf, "f16", 1024, 1024, 256, 256, "phase", "adc", synth.SEED_BASE + 1,
               batches=[0, 131, 255], rows=[0, 1, 127, 128, 511, 1000, 1023])


def test_full_size_radio_b1_sampled(tcbf, b1_kernel):
    """BASELINE configs[2]: M=1024, K=512, N=4096, batch=256."""
    _full_size(tcbf, "b1", 1024, 4096, 512, 256, "phase", "adc", synth.SEED_BASE + 2,
               batches=[0, 200, 255], rows=[0, 63, 64, 777, 1023])


def test_full_size_radio_f16_raw_sampled(tcbf):
    """BASELINE configs[1] through tcbf_beamform_raw, the launch bench.py times (data-in-TMEM fused
    kernel with 32-beam tiles: 2048 units on 148 CTAs, half of each next unit written straight
    into TMEM, raw data by TMA)."""
    plan = tcbf.Plan(1024, 1024, 256, 256, "f16")
    assert plan.raw_variant == "f16_tcgen05_fused_tmem_128x32", plan.raw_variant
    _full_size(tcbf, "f16", 1024, 1024, 256, 256, "phase", "adc", synth.SEED_BASE + 1,
               batches=[0, 77, 255], rows=[0, 63, 64, 127, 128, 700, 1023], path="raw")


# several 128-sample units per CTA (the staged next unit copied into TMEM at each switch), K16 =
# 64 / 192 / 256 (1, 3, 4 data blocks; 4 .. 16 raw boxes per unit), ragged M and N, planar source
TMEM_SHAPES = [
    (130, 520, 200, 40, "interleaved"),
    (64, 256, 64, 160, "planar"),
    (200, 1000, 130, 30, "interleaved"),
    (96, 332, 100, 20, "planar"),
    (64, 512, 128, 10, "interleaved"),
]


def test_f16_tmem_fused_kernel_odd_n_plan(tcbf):
    """N % 4 != 0: the plan picks the smem sample-major fused kernel at creation (TMA rows need
    16-byte strides), and the kernel name says so."""
    assert tcbf.Plan(96, 333, 100, 2, "f16").raw_variant == "f16_tcgen05_fused_smaj_128x128"
    assert tcbf.Plan(96, 332, 100, 2, "f16").raw_variant == "f16_tcgen05_fused_tmem_128x64"


@pytest.mark.parametrize("shape", TMEM_SHAPES)
def test_f16_tmem_fused_kernel(tcbf, shape, monkeypatch):
    """The data-in-TMEM fused kernel (64-beam tiles, forced for K16 = 256 too) equals pack +
    beamform up to fp32 summation order inside the MMA and meets the oracle on sampled batch
    entries."""
    M, N, K, B, layout = shape
    monkeypatch.setenv("TCBF_F16_FUSED", "tmem")
    w = synth.generate("phase", 37, 0, B, M, K)
    x = synth.generate("adc", 37, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    plan = tcbf.Plan(M, N, K, B, "f16")
    assert plan.raw_variant == "f16_tcgen05_fused_tmem_128x64", plan.raw_variant
    wp = plan.pack(tcbf.WEIGHTS, _dev(conv(w)), layout)
    xd = _dev(conv(x))
    y_raw = plan.beamform_raw(wp, xd, layout)
    y_ref = plan.beamform(wp, plan.pack(tcbf.DATA, xd, layout))
    torch.cuda.synchronize()
    assert (y_raw - y_ref).abs().max().item() <= 1e-6 * y_ref.abs().max().item()
    sel = sorted({0, B // 2, B - 1})
    ref = oracle.cgemm_f16(conv(w[sel]), conv(x[sel]), 0 if layout == "interleaved" else 1, M, N, K, len(sel))
    _check_f16(y_raw[sel].cpu().numpy(), ref, w[sel], x[sel])


# the 32-beam-tile variant (K16 = 256; half of the next unit written straight into TMEM, three
# rotating data regions): >= 4 units per CTA so every region is reused, ragged M and N, both
# layouts, with and without the CTA-pair weight multicast (tiles_n odd -> no pairs), WKB 2 and 4
TMEM32_SHAPES = [
    (130, 520, 200, 160, "interleaved", "2"),
    (96, 512, 256, 160, "planar", "2"),
    (33, 256, 193, 300, "interleaved", "4"),
    (1024, 1024, 256, 12, "planar", "4"),
]


@pytest.mark.parametrize("shape", TMEM32_SHAPES)
def test_f16_tmem32_fused_kernel(tcbf, shape, monkeypatch):
    """The 32-beam data-in-TMEM kernel (the K16 = 256 default) equals pack + beamform up to fp32
    summation order and meets the oracle on sampled batch entries."""
    M, N, K, B, layout, wkb = shape
    monkeypatch.setenv("TCBF_TMEM2_WKB", wkb)
    w = synth.generate("phase", 41, 0, B, M, K)
    x = synth.generate("adc", 41, 1, B, K, N)
    conv = synth.to_interleaved if layout == "interleaved" else synth.to_planar
    plan = tcbf.Plan(M, N, K, B, "f16")
    assert plan.raw_variant == "f16_tcgen05_fused_tmem_128x32", plan.raw_variant
    wp = plan.pack(tcbf.WEIGHTS, _dev(conv(w)), layout)
    xd = _dev(conv(x))
    y_raw = plan.beamform_raw(wp, xd, layout)
    y_ref = plan.beamform(wp, plan.pack(tcbf.DATA, xd, layout))
    torch.cuda.synchronize()
    assert (y_raw - y_ref).abs().max().item() <= 1e-6 * y_ref.abs().max().item()
    sel = sorted({0, B // 2, B - 1})
    ref = oracle.cgemm_f16(conv(w[sel]), conv(x[sel]), 0 if layout == "interleaved" else 1, M, N, K, len(sel))
    _check_f16(y_raw[sel].cpu().numpy(), ref, w[sel], x[sel])


# 1-bit sample-major kernel with the unit's data resident in TMEM (Kw <= 24): several units per
# CTA, ragged M (partial 64-beam tile) and N (partial 128-sample unit), K with padding bits,
# the largest resident K (768), the radio shape class
B1_TMEM_SHAPES = [
    (130, 300, 100, 3), (64, 128, 256, 2), (200, 1000, 512, 30), (70, 77, 768, 2), (1024, 512, 512, 2),
    (96, 256, 33, 160), (8, 64, 32, 2),
]


@pytest.mark.parametrize("shape", B1_TMEM_SHAPES)
def test_b1_tmem_kernel_bit_exact(tcbf, shape, monkeypatch):
    monkeypatch.setenv("TCBF_B1_KERNEL", "tmem")
    M, N, K, B = shape
    w = synth.to_interleaved(synth.generate("uniform", 41, 0, B, M, K))
    x = synth.to_interleaved(synth.generate("uniform", 41, 1, B, K, N))
    plan, _, _, y = _run(tcbf, "b1", w, x, M, N, K, B)
    assert plan.variant == "b1_tcgen05_mxf4pm1_tmem_128x64", plan.variant
    assert np.array_equal(y, oracle.cgemm_b1(w, x, 0, M, N, K, B))


def test_full_size_square_16384_sampled(tcbf):
    """BASELINE configs[4] largest square points, fp16 and 1-bit, M=N=K=16384."""
    for prec in ("f16", "b1"):
        _full_size(tcbf, prec, 16384, 16384, 16384, 1, "uniform", "uniform", synth.SEED_BASE + 4,
                   batches=[0], rows=[0, 8191, 16383])
        torch.cuda.empty_cache()


def test_full_size_m32_f16_16384_raw_sampled(tcbf):
    """BASELINE configs[4] small-beam fp16 point through the streaming-conversion kernel, as
    bench.py times it (M=32, N=K=16384)."""
    plan = tcbf.Plan(32, 16384, 16384, 1, "f16")
    assert plan.raw_variant == "f16_tcgen05_stream_conv_128x128"
    _full_size(tcbf, "f16", 32, 16384, 16384, 1, "uniform", "uniform", synth.SEED_BASE + 4,
               batches=[0], rows=[0, 17, 31], path="raw")


def test_full_size_radio_f16i_sampled(tcbf):
    """The radio shape with fp16 interleaved data (bench config radio_f16i, no pack)."""
    _full_size(tcbf, "f16", 1024, 1024, 256, 256, "phase", "adc", synth.SEED_BASE + 1,
               batches=[0, 255], rows=[0, 127, 1023], path="f16i")


def test_sliced_weight_generation_equals_direct(tcbf):
    """bench.pack_weights' row-sliced generate+pack (for model matrices too large for one fp32
    source) produces exactly the directly packed weights."""
    import bench
    for prec, B, b0 in [("b1", 1, 0), ("b1", 3, 2), ("f16", 2, 1)]:
        c = dict(bench.CONFIGS["ultrasound_b1_planes"], M=1000, K=3000, N=64, B=B, prec=prec)
        seed = synth.SEED_BASE + 3
        plan = tcbf.Plan(c["M"], c["N"], c["K"], B, prec)
        direct = plan.pack(tcbf.WEIGHTS, synth.generate_device(c["wd"], seed, 0, B, c["M"], c["K"], b0=b0))
        sliced = bench.pack_weights(plan, c, seed, torch.device("cuda"), b0, max_src_bytes=300 * 3000 * 8)
        assert torch.equal(direct, sliced), (prec, B, b0)


def test_full_size_ultrasound_b1_planes_sampled(tcbf):
    """The ultrasound 1-bit pipeline shape: M=49152, K=262144, N=1024, with the
    weights generated and packed in slices exactly as bench.py does; sampled beams vs the oracle."""
    import bench
    c = bench.CONFIGS["ultrasound_b1_planes"]
    M, N, K = c["M"], c["N"], c["K"]
    seed = synth.SEED_BASE + c["idx"]
    plan = tcbf.Plan(M, N, K, 1, "b1")
    wp = bench.pack_weights(plan, c, seed, torch.device("cuda"), 0)
    y = plan.beamform_raw(wp, synth.generate_device(c["xd"], seed, 1, 1, K, N))
    torch.cuda.synchronize()
    rows = [0, 20000, 49151]
    w = synth.generate(c["wd"], seed, 0, 1, M, K, r_sel=rows)
    x = synth.generate(c["xd"], seed, 1, 1, K, N)
    ref = oracle.cgemm_b1(synth.to_interleaved(w), synth.to_interleaved(x), 0, len(rows), N, K, 1)
    assert np.array_equal(y[0][:, rows].cpu().numpy()[None], ref)


def test_full_size_ultrasound_f16_sampled(tcbf):
    """BASELINE configs[3]: M=65536, K=8192, N=256, batch=8 (17 GB of packed weights)."""
    _full_size(tcbf, "f16", 65536, 256, 8192, 8, "phase_amp", "adc_scaled", synth.SEED_BASE + 3,
               batches=[0, 7], rows=[0, 4097, 65535])


@pytest.mark.parametrize("prec,shape", [("f16", (1024, 1024, 256, 64)), ("b1", (1024, 4096, 512, 16)),
                                        ("f16", (1000, 1020, 200, 50))])
def test_tmem_kernels_deterministic(tcbf, prec, shape):
    """Race canary for the TMEM kernels (compute-sanitizer is unavailable on this pool): the same
    launch repeated must give bitwise identical output -- a hand-off bug in the unit-switch staging,
    the weight ring or the TMEM accumulator double buffer would show up as run-to-run differences
    (every sum is formed in a fixed order, so correct runs are bitwise reproducible)."""
    M, N, K, B = shape
    plan = tcbf.Plan(M, N, K, B, prec)
    w = synth.generate_device("phase", 53, 0, B, M, K)
    x = synth.generate_device("adc", 53, 1, B, K, N)
    wp = plan.pack(tcbf.WEIGHTS, w)
    if prec == "f16":
        assert "tmem" in plan.raw_variant
        run = lambda: plan.beamform_raw(wp, x)                                   # noqa: E731
    else:
        assert "tmem" in plan.variant
        xp = plan.pack(tcbf.DATA, x)
        run = lambda: plan.beamform(wp, xp)                                      # noqa: E731
    ref = run()
    for _ in range(6):
        y = run()
        torch.cuda.synchronize()
        assert torch.equal(y, ref)
