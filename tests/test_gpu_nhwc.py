"""GPU parity of the channels-last options: snn_conv_fire_ex(SNN_CONV_OUT_NHWC) and
snn_pool_ex(SNN_POOL_IN_NHWC), and of v_out = NULL.

The conv's channels-last output is the planar oracle result transposed (same neurons, other layout);
the pool reading it must equal the oracle pool of the planar map.  Bit-exact (N1).
"""
import math

import numpy as np
import pytest
import torch

from test_gpu_kernels import CONV_CASES, cu, exact_weights, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1903_02440_b200 import build, snn
    build.build()
    snn.lib()
    return snn


@pytest.mark.parametrize("path", ["walk", "tct", "ref"])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fire_nhwc_vs_oracle(G, orc, case, path, monkeypatch):
    monkeypatch.setenv("SNN_CONV_PATH", path)
    B, C, H, W, pad, F, K, T, theta, p = case
    rng = np.random.default_rng((abs(hash(case)) + 7) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K))
    lat, v = G.conv_fire(cu(lat_in), cu(w), pad, T, theta, nhwc=True)
    lat_only, none_v = G.conv_fire(cu(lat_in), cu(w), pad, T, theta, nhwc=True, want_v=False)
    G.sync_status()
    assert none_v is None
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    assert np.array_equal(host(lat), ol.transpose(0, 2, 3, 1))
    assert np.array_equal(host(v), ov.transpose(0, 2, 3, 1))
    assert np.array_equal(host(lat_only), ol.transpose(0, 2, 3, 1))


@pytest.mark.parametrize("case", CONV_CASES[:6])
def test_conv_fire_planar_without_v(G, orc, case):
    B, C, H, W, pad, F, K, T, theta, p = case
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K))
    lat, v = G.conv_fire(cu(lat_in), cu(w), pad, T, theta, want_v=False)
    G.sync_status()
    assert v is None
    ol, _ = orc.conv_fire(lat_in, w, pad, T, theta)
    assert np.array_equal(host(lat), ol)


@pytest.mark.parametrize("win,stride,pad,with_v,F,flags", [
    ((2, 2), (2, 2), (0, 0), True, 256, 0), ((2, 2), (2, 2), (0, 0), False, 30, 0),
    ((3, 3), (3, 3), (0, 0), False, 250, 0), ((7, 7), (6, 6), (0, 0), False, 20, 0),
    ((7, 7), (6, 6), (0, 0), True, 33, 0), ((3, 2), (2, 1), (1, 1), True, 5, 0),
    ((2, 3), (3, 2), (1, 0), True, 70, 0), ((1, 1), (1, 1), (0, 0), True, 1, 0),
    ((3, 3), (2, 2), (1, 1), True, 40, 1), ((2, 2), (2, 2), (0, 0), True, 64, 2),
    ((3, 3), (3, 3), (0, 0), True, 31, 3)])
def test_pool_nhwc_vs_oracle(G, orc, win, stride, pad, with_v, F, flags):
    """flags: 1 = SNN_POOL_EQ3, 2 = SNN_POOL_VFINAL (combined with SNN_POOL_IN_NHWC)."""
    import synth
    rng = np.random.default_rng(F * 7 + flags)
    T = 9
    lat = synth.random_latencies(rng, (3, F, 37, 70), T, 0.5)
    v = synth.random_potentials_at_spike(rng, lat, 4)
    lat_h = np.ascontiguousarray(lat.transpose(0, 2, 3, 1))
    v_h = np.ascontiguousarray(v.transpose(0, 2, 3, 1))
    gl, gv = G.pool(cu(lat_h), cu(v_h) if with_v else None, win, stride, pad, flags=flags | G.POOL_IN_NHWC)
    gl2, gv2 = G.pool(cu(lat), cu(v) if with_v else None, win, stride, pad, flags=flags)
    ol, ov = orc.pool(lat, v if with_v else None, *win, *stride, *pad, T, eq3=bool(flags & 1), vfinal=bool(flags & 2))
    assert np.array_equal(host(gl), ol) and np.array_equal(host(gl2), ol)
    if with_v:
        assert np.array_equal(host(gv), ov) and np.array_equal(host(gv2), ov)


def test_nhwc_conv_then_pool_chain(G, orc):
    """C5-shaped chain (smaller): conv (channels-last, lat + v) -> pool 2/2 reading it == oracle."""
    import synth
    rng = np.random.default_rng(21)
    B, C, H, W, pad, F, K, T, theta = 2, 32, 24, 24, 2, 256, 5, 32, 40.0
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, 0.5)
    w = exact_weights(rng, (F, C, K, K), lo=2 ** -5)
    lat, v = G.conv_fire(cu(lat_in), cu(w), pad, T, theta, nhwc=True)
    pl, pv = G.pool(lat, v, 2, 2, 0, flags=G.POOL_IN_NHWC)
    G.sync_status()
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    opl, opv = orc.pool(ol, ov, 2, 2, 2, 2, 0, 0, T)
    assert np.array_equal(host(pl), opl) and np.array_equal(host(pv), opv)


def test_conv_fire_ex_bad_flags(G):
    lat_in = torch.zeros((1, 1, 4, 4), dtype=torch.uint8, device="cuda")
    w = torch.full((2, 1, 3, 3), 0.5, dtype=torch.float32, device="cuda")
    out = torch.empty((1, 2, 2, 2), dtype=torch.uint8, device="cuda")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    L = G.lib()
    rc = L.snn_conv_fire_ex(G._ptr(lat_in), 1, 1, 4, 4, 0, G._ptr(w), 2, 3, 3, 4, 1.0, 8, G._ptr(out), None, None,
                            G._ptr(ws), ws.numel(), G._stream(None))
    assert rc == G.SNN_EINVAL


# ----------------------------------------------------------------- channels-last inputs (encode -> conv -> pool)
@pytest.mark.parametrize("shape,T", [((1, 2, 28, 28), 15), ((7, 6, 28, 28), 15), ((3, 4, 60, 70), 30),
                                     ((2, 32, 40, 40), 32), ((2, 1, 1, 5), 10)])
def test_encode_nhwc_vs_oracle(G, orc, shape, T):
    """all three encode paths (bitonic: few small images; one-CTA select; multi-kernel radix select)."""
    rng = np.random.default_rng(sum(shape) + T)
    x = rng.random(shape).astype(np.float32)
    x[rng.random(shape) < 0.4] = 0
    x.reshape(-1)[::13] = 0.5
    got = host(G.encode(cu(x), T, nhwc=True))
    assert np.array_equal(got, orc.encode(x, T).transpose(0, 2, 3, 1))


@pytest.mark.parametrize("out_nhwc", [True, False])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fire_in_nhwc_vs_oracle(G, orc, case, out_nhwc):
    """channels-last input on the default path: fused / presorted walk (finite theta), tcgen05 (theta = inf)."""
    B, C, H, W, pad, F, K, T, theta, p = case
    rng = np.random.default_rng((abs(hash(case)) + 11) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K))
    lat, v = G.conv_fire(cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))), cu(w), pad, T, theta,
                         nhwc=out_nhwc, in_nhwc=True)
    G.sync_status()
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    if out_nhwc:
        ol, ov = ol.transpose(0, 2, 3, 1), ov.transpose(0, 2, 3, 1)
    assert np.array_equal(host(lat), ol)
    assert np.array_equal(host(v), ov)


def test_conv_in_nhwc_rejects_validation_paths(G, monkeypatch):
    lat_in = torch.zeros((1, 4, 4, 1), dtype=torch.uint8, device="cuda")
    w = torch.full((2, 1, 3, 3), 0.5, dtype=torch.float32, device="cuda")
    with pytest.raises(G.SNNError):
        G.conv_fire(lat_in, w, 0, 4, 1.0, want_pot=True, in_nhwc=True)
    monkeypatch.setenv("SNN_CONV_PATH", "ref")
    with pytest.raises(G.SNNError):
        G.conv_fire(lat_in, w, 0, 4, 1.0, in_nhwc=True)


@pytest.mark.parametrize("win,stride,pad,with_v,F,flags", [
    ((2, 2), (2, 2), (0, 0), False, 30, 0), ((3, 3), (3, 3), (0, 0), False, 250, 0),
    ((2, 2), (2, 2), (0, 0), True, 256, 0), ((2, 2), (2, 2), (0, 0), False, 64, 0),
    ((7, 7), (6, 6), (0, 0), False, 20, 0), ((3, 2), (2, 1), (1, 1), True, 5, 0),
    ((3, 3), (2, 2), (1, 1), True, 40, 1), ((2, 2), (2, 2), (0, 0), True, 64, 2),
    ((3, 3), (2, 2), (1, 1), False, 30, 1), ((3, 2), (3, 3), (1, 0), False, 7, 0), ((1, 1), (1, 1), (0, 0), False, 33, 0)])
def test_pool_nhwc_to_nhwc_vs_oracle(G, orc, win, stride, pad, with_v, F, flags):
    import synth
    rng = np.random.default_rng(F * 3 + flags + 1)
    T = 9
    lat = synth.random_latencies(rng, (3, F, 37, 70), T, 0.5)
    v = synth.random_potentials_at_spike(rng, lat, 4)
    lat_h = np.ascontiguousarray(lat.transpose(0, 2, 3, 1))
    v_h = np.ascontiguousarray(v.transpose(0, 2, 3, 1))
    gl, gv = G.pool(cu(lat_h), cu(v_h) if with_v else None, win, stride, pad,
                    flags=flags | G.POOL_IN_NHWC | G.POOL_OUT_NHWC)
    ol, ov = orc.pool(lat, v if with_v else None, *win, *stride, *pad, T, eq3=bool(flags & 1), vfinal=bool(flags & 2))
    assert np.array_equal(host(gl), ol.transpose(0, 2, 3, 1))
    if with_v:
        assert np.array_equal(host(gv), ov.transpose(0, 2, 3, 1))


@pytest.mark.parametrize("case", [CONV_CASES[i] for i in (0, 2, 4, 6, 13, 16, 17)])
def test_conv_fire_kstar_truncation(G, orc, case, monkeypatch):
    """SNN_KSTAR=1: sorted lists end at the first bucket that brings the count to K* (K2b)."""
    monkeypatch.setenv("SNN_KSTAR", "1")
    B, C, H, W, pad, F, K, T, theta, p = case
    rng = np.random.default_rng((abs(hash(case)) + 3) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K))
    w[1, 0, 0, 0] = 0.0
    lat, v = G.conv_fire(cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))), cu(w), pad, T, theta, nhwc=True,
                         in_nhwc=True)
    G.sync_status()
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    assert np.array_equal(host(lat), ol.transpose(0, 2, 3, 1))
    assert np.array_equal(host(v), ov.transpose(0, 2, 3, 1))


# ------------------------------------------------- K7 row tiles (fused small-receptive-field layers, NHWC input)
ROWS_CASES = [
    # (B, C, H, W, pad, F, K, T, theta, p_spike, w_lo)
    (8, 6, 28, 28, 2, 30, 5, 15, 15.0, 0.45, 2 ** -5),   # C2 L1 shape (one tile per output row), S28 slice
    (8, 6, 28, 28, 2, 30, 5, 15, 15.0, 0.45, 2 ** -8),   # the same with an int64 (2^-31) slice
    (3, 4, 40, 75, 0, 20, 5, 30, 15.0, 0.5, 2 ** -5),    # C4 L1-like: 3 tiles per row, ragged last tile
    (4, 3, 33, 70, 1, 17, 3, 6, -0.5, 0.5, 2 ** -8),     # theta < 0 (fires at t = 0), F % 4 != 0
    (5, 2, 30, 41, 2, 32, 5, 1, 1.0, 0.8, 2 ** -5),      # T = 1, F = 32
    (6, 5, 25, 37, 1, 25, 3, 9, 3.0, 1.0, 2 ** -8),      # every input spikes, 2 tiles per row
    (4, 4, 21, 130, 2, 9, 5, 12, 2.5, 0.3, 2 ** -5),     # 5 tiles per row, few features
    (8, 6, 26, 29, 0, 30, 5, 15, 40.0, 0.5, 2 ** -5),    # threshold never reached (whole lists walked)
]


@pytest.mark.parametrize("g", ["1", "2"])
@pytest.mark.parametrize("out_nhwc", [True, False])
@pytest.mark.parametrize("case", ROWS_CASES)
def test_conv_fire_rows_vs_oracle(G, orc, case, out_nhwc, g, capfd, monkeypatch):
    """K7: the fused walk by row tiles (each output row's input halo sorted once by (t, column)), bit-exact;
    g = buckets per threshold test (K7c: 2 = one test per bucket pair, snapshots locate the crossing)."""
    monkeypatch.setenv("SNN_DEBUG_PLAN", "1")
    monkeypatch.setenv("SNN_WALK_ROWS_G", g)
    B, C, H, W, pad, F, K, T, theta, p, lo = case
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K), lo=lo)
    lat, v = G.conv_fire(cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))), cu(w), pad, T, theta,
                         nhwc=out_nhwc, in_nhwc=True)
    G.sync_status()
    assert "walk rows:" in capfd.readouterr().err
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    if out_nhwc:
        ol, ov = ol.transpose(0, 2, 3, 1), ov.transpose(0, 2, 3, 1)
    assert np.array_equal(host(lat), ol)
    assert np.array_equal(host(v), ov)



# ------------------------------------------------------- K8 implicit im2col (theta = inf, tcgen05 GEMM)
IMPLICIT_CASES = [
    # (B, C, H, W, pad, F, K, p_spike)
    (320, 250, 4, 4, 2, 200, 5, 0.9),    # C2 L3 shape (8 images per M tile, 6 pad channels)
    (300, 32, 9, 11, 1, 40, 3, 0.5),     # tiles cross image boundaries mid-row
    (400, 16, 5, 7, 0, 24, 3, 0.7),      # 3 x 5 outputs: 9 images per tile, no padding
    (300, 64, 12, 12, 2, 70, 5, 0.3),    # 2 feature chunks, partial rows at both tile ends
]


@pytest.mark.parametrize("case", IMPLICIT_CASES)
def test_conv_inf_implicit_vs_oracle(G, orc, case, capfd, monkeypatch):
    """K8 (opt-in): the A operand built in the GEMM CTA from the staged binary S[T-1] footprint (Eq. 5),
    bit-exact."""
    monkeypatch.setenv("SNN_DEBUG_PLAN", "1")
    monkeypatch.setenv("SNN_TC_IMPLICIT", "1")
    monkeypatch.setenv("SNN_TC_FC", "0")                 # the im2col plan (K9 takes the C2 L3 shape otherwise)
    B, C, H, W, pad, F, K, p = case
    T = 15
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K))
    lat, v = G.conv_fire(cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))), cu(w), pad, T, math.inf,
                         nhwc=True, in_nhwc=True)
    G.sync_status()
    assert "implicit 1" in capfd.readouterr().err
    ol, ov = orc.conv_fire(lat_in, w, pad, T, math.inf)
    assert np.array_equal(host(lat), ol.transpose(0, 2, 3, 1))
    assert np.array_equal(host(v), ov.transpose(0, 2, 3, 1))


@pytest.mark.parametrize("case", ROWS_CASES)
def test_conv_fire_pool2_vs_oracle(G, orc, case, capfd, monkeypatch):
    """SNN_CONV_POOL2: the 2 x 2 / stride 2 latency pooling fused into the row-tile walk equals the oracle's
    pooling (A10-A12) of the oracle's conv output; odd Ho / Wo drop the last row / column."""
    monkeypatch.setenv("SNN_DEBUG_PLAN", "1")
    B, C, H, W, pad, F, K, T, theta, p, lo = case
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K), lo=lo)
    lat, v = G.conv_fire(cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))), cu(w), pad, T, theta,
                         nhwc=True, in_nhwc=True, want_v=False, pool2=True)
    G.sync_status()
    assert v is None and "pool2 1" in capfd.readouterr().err
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    pl, _ = orc.pool(ol, None, 2, 2, 2, 2, 0, 0, T)
    assert np.array_equal(host(lat), pl.transpose(0, 2, 3, 1))


def test_conv_fire_pool2_declined(G):
    """SNN_CONV_POOL2 where the row-tile walk does not apply: SNN_ESHAPE before any launch; with potentials
    or a planar output: SNN_EINVAL."""
    lat_in = torch.zeros((1, 28, 28, 2), dtype=torch.uint8, device="cuda")   # one image: latency mode
    w = torch.full((30, 2, 5, 5), 0.5, dtype=torch.float32, device="cuda")
    with pytest.raises(G.SNNError) as e:
        G.conv_fire(lat_in, w, 2, 15, 15.0, nhwc=True, in_nhwc=True, want_v=False, pool2=True)
    assert e.value.code == G.SNN_ESHAPE
    lat_in = torch.zeros((64, 28, 28, 2), dtype=torch.uint8, device="cuda")
    with pytest.raises(G.SNNError) as e:
        G.conv_fire(lat_in, w, 2, 15, 15.0, nhwc=True, in_nhwc=True, want_v=True, pool2=True)
    assert e.value.code == G.SNN_EINVAL
    with pytest.raises(G.SNNError) as e:
        G.conv_fire(lat_in, w, 2, 15, math.inf, nhwc=True, in_nhwc=True, want_v=False, pool2=True)
    assert e.value.code == G.SNN_EINVAL
