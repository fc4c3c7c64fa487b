"""GPU parity: every libsnn kernel (through the C ABI) vs the CPU oracle on seeded inputs.

Sizes span several tiles / chunks with ragged tails; edge cases: empty inputs, T = 1, T = 254,
N < T, all-equal intensities, negative/NaN intensities, pad > 0, window != stride, k > #candidates,
r = 0, F not a multiple of 32, theta = +inf, theta < 0, the dense theta = inf path.
Integer / index outputs must be bit-exact; fp32 potentials are exact too (N1), so v and
pot are compared bit-exactly as well.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NS = 255


@pytest.fixture(scope="module")
def G():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1903_02440_b200 import build, snn
    build.build()
    snn.lib()
    return snn


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def exact_weights(rng, shape, lo=2 ** -8):
    return rng.uniform(lo, 1.0, size=shape).astype(np.float32)


# ---------------------------------------------------------------------------------------- encode
@pytest.mark.parametrize("shape,T,seed", [((1, 2, 28, 28), 15, 0), ((3, 3, 50, 60), 32, 1), ((2, 1, 1, 5), 10, 2),
                                          ((4, 5, 7, 9), 1, 3), ((2, 4, 33, 65), 254, 4), ((1, 1, 64, 300), 7, 5)])
def test_encode_random(G, orc, shape, T, seed):
    rng = np.random.default_rng(seed)
    x = rng.random(shape).astype(np.float32)
    x[rng.random(shape) < 0.3] = 0
    x[rng.random(shape) < 0.05] = -1
    x.reshape(-1)[::97] = 0.5                        # ties
    if x.size > 10:
        x.reshape(-1)[3] = np.nan
    got = host(G.encode(cu(x), T))
    assert np.array_equal(got, orc.encode(x, T))


@pytest.mark.parametrize("shape,T,seed", [((2, 3, 100, 70), 254, 6), ((3, 2, 129, 64), 32, 7), ((1, 1, 1, 16385), 15, 8)])
def test_encode_large_path(G, orc, shape, T, seed):
    """C*H*W > 16384 takes the multi-kernel radix-select path."""
    rng = np.random.default_rng(seed)
    x = (rng.integers(0, 50, size=shape) / 49).astype(np.float32)      # heavy ties
    x[rng.random(shape) < 0.2] = 0
    assert np.array_equal(host(G.encode(cu(x), T)), orc.encode(x, T))


@pytest.mark.parametrize("shape,T,seed", [((2, 2, 150, 150), 32, 9), ((1, 3, 90, 91), 15, 10)])
def test_encode_large_path_continuous(G, orc, shape, T, seed):
    """Large path, distinct values (every radix level decides on value bits, few elements per cut bin)."""
    rng = np.random.default_rng(seed)
    x = rng.random(shape, dtype=np.float32)
    x[rng.random(shape) < 0.1] = 0
    assert np.array_equal(host(G.encode(cu(x), T)), orc.encode(x, T))


def test_encode_all_equal_and_zero(G, orc):
    x = np.full((2, 3, 20, 20), 0.25, np.float32)
    x[1] = 0
    for T in (1, 15, 254):
        assert np.array_equal(host(G.encode(cu(x), T)), orc.encode(x, T))


def test_encode_quantized_many_ties(G, orc):
    rng = np.random.default_rng(11)
    x = (rng.integers(0, 7, size=(5, 4, 40, 41)) / 6).astype(np.float32)
    for T in (15, 30, 32):
        assert np.array_equal(host(G.encode(cu(x), T)), orc.encode(x, T))


def test_encode_empty(G):
    x = torch.empty((0, 2, 4, 4), dtype=torch.float32, device="cuda")
    assert G.encode(x, 5).shape == (0, 2, 4, 4)


# ---------------------------------------------------------------------------------------- expand / validate
def test_expand_and_validate(G, orc):
    rng = np.random.default_rng(1)
    lat = rng.integers(0, 9, size=(3, 4, 5, 6)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.3] = NS
    assert np.array_equal(host(G.expand(cu(lat), 9)), orc.expand(lat, 9))
    assert G.validate_lat(cu(lat), 9) == 0
    assert G.validate_lat(cu(lat), 5) == int(((lat >= 5) & (lat != NS)).sum())


# ---------------------------------------------------------------------------------------- conv + fire
CONV_CASES = [
    # (B, C, H, W, pad, F, K, T, theta, p_spike)
    (2, 2, 28, 28, 2, 30, 5, 15, 15.0, 0.5),        # C1-like, F < 32
    (3, 6, 14, 13, 1, 70, 3, 15, 4.0, 0.7),         # F not a multiple of 32, ragged W
    (2, 30, 14, 14, 1, 250, 3, 15, 10.0, 0.9),      # C2 L2 shape
    (1, 4, 20, 31, 0, 20, 5, 30, 15.0, 0.5),        # C4 L1-like, T = 30
    (2, 32, 24, 24, 2, 256, 5, 32, 40.0, 0.5),      # C5-like
    (2, 3, 9, 9, 0, 33, 3, 1, 1.0, 0.8),            # T = 1
    (2, 3, 9, 9, 2, 40, 3, 6, -0.5, 0.5),           # theta < 0 (fires at t = 0)
    (2, 5, 8, 8, 1, 37, 3, 6, math.inf, 0.6),       # Eq. 5 on the shared-memory path
    (2, 250, 4, 4, 2, 200, 5, 15, math.inf, 0.9),   # Eq. 5 dense path (C2 L3 shape)
    (1, 20, 25, 40, 0, 100, 17, 30, math.inf, 0.7), # Eq. 5 dense path (C4 L2 shape)
    (1, 2, 5, 5, 0, 3, 5, 4, 0.5, 0.0),             # no input spikes at all
    (3, 7, 21, 19, 2, 130, 5, 9, 6.0, 0.7),         # 3 feature chunks, ragged M tile
    (1, 4, 20, 31, 0, 20, 5, 254, 2.0, 0.3),        # T = 254
    (2, 32, 12, 12, 2, 100, 5, 2, 40.0, 0.6),       # 2 huge buckets: crossings pend across walk blocks
    (2, 16, 10, 10, 1, 64, 3, 3, 20.0, 0.9),        # T = 3, 64 features (one FPL=2 group)
    (1, 9, 11, 7, 1, 256, 3, 5, 5.0, 0.5),          # 256 features on a small receptive field
    (3, 8, 10, 10, 1, 130, 3, 40, 30.0, 1.0),       # every input spikes, T > R/2: many odd buckets (list padding)
    (2, 8, 10, 10, 1, 30, 3, 40, 30.0, 1.0),        # the same on the fused sort+walk schedule
]


@pytest.mark.parametrize("path", ["walk", "tct", "ref"])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fire_vs_oracle(G, orc, case, path, monkeypatch):
    """walk = default SIMT delta walk for finite theta (tcgen05 GEMM for theta = inf);
    tct = tensor-core time-stepped kernel (SNN_CONV_PATH=tct); ref = validation kernel."""
    monkeypatch.setenv("SNN_CONV_PATH", path)
    B, C, H, W, pad, F, K, T, theta, p = case
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K))
    w[0, 0, 0, 0] = 0.0                                # zero weight is exact too
    lat, v = G.conv_fire(cu(lat_in), cu(w), pad, T, theta)
    G.sync_status()
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    assert np.array_equal(host(lat), ol)
    assert np.array_equal(host(v), ov)


KMIN_CASES = [
    # (B, C, H, W, pad, F, K, T, theta, p_spike, weights)   -- presorted bucket walk unless noted
    (2, 32, 24, 24, 2, 256, 5, 32, 40.0, 0.5, "c5"),     # C5-like: kmin ~ 5 buckets of ~12 entries
    (2, 32, 12, 12, 2, 100, 5, 2, 40.0, 0.6, "u"),       # 2 huge buckets: kmin inside bucket 0
    (2, 30, 14, 14, 1, 250, 3, 15, 10.0, 0.9, "c2"),     # C2 L2 shape, FPL = 4 groups
    (2, 30, 14, 14, 1, 250, 3, 15, 300.0, 0.9, "u"),     # no feature can ever fire (kmin = INT_MAX)
    (2, 32, 16, 16, 2, 70, 5, 32, 60.0, 0.1, "c5"),      # most lists shorter than kmin: silent without a walk
    (1, 32, 16, 16, 2, 64, 5, 32, 0.25, 0.5, "u"),       # kmin = 1 (the first non-empty bucket, as before)
    (2, 32, 16, 16, 2, 64, 5, 32, -1.0, 0.5, "u"),       # theta < 0: kmin = 0
    (2, 8, 10, 10, 1, 30, 3, 5, 6.0, 1.0, "u"),          # fused sort + bucket walk: the bound is not applied there
    (3, 16, 20, 20, 1, 96, 3, 12, 25.0, 0.8, "s28"),     # weights on the 2^-28 grid (S28 block sums)
]


@pytest.mark.parametrize("nhwc,kstar", [(False, "0"), (True, "0"), (True, "1"), (False, "1")])
@pytest.mark.parametrize("case", KMIN_CASES)
def test_conv_kmin_prefix_vs_oracle(G, orc, case, nhwc, kstar, monkeypatch):
    """K2e (SNN_KMIN=1 forces it on): buckets that end below kmin entries are added without a threshold
    test; together with the K* list truncation (K2b, SNN_KSTAR=1) on maps whose spike density and timing
    vary across positions.  Spike times and potentials stay those of Eq. 2 + R3 (oracle conv_fire)."""
    monkeypatch.setenv("SNN_KMIN", "1")
    monkeypatch.setenv("SNN_KSTAR", kstar)
    B, C, H, W, pad, F, K, T, theta, p, wk = case
    rng = np.random.default_rng(7000 + KMIN_CASES.index(case))
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    if kstar == "1":                                     # a sparse, late-spiking band next to the dense map
        band = lat_in[:, :, :, : W // 3]
        band[rng.random(band.shape) < 0.8] = 255
        late = lat_in[:, :, H // 2:, W // 3: 2 * W // 3]
        late[(late != 255) & (late < T // 2)] = T - 1
    if wk == "c5":
        w = np.clip(rng.normal(0.5, 0.1, size=(F, C, K, K)), 2.0 ** -8, 1.0).astype(np.float32)
    elif wk == "c2":
        w = np.clip(rng.normal(0.8, 0.05, size=(F, C, K, K)), 2.0 ** -8, 1.0).astype(np.float32)
    elif wk == "s28":
        w = (rng.integers(2 ** 23, 2 ** 28, size=(F, C, K, K)) / 2.0 ** 28).astype(np.float32)
        w = (np.round(w.astype(np.float64) * 2 ** 28) / 2 ** 28).astype(np.float32)
    else:
        w = exact_weights(rng, (F, C, K, K))
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    if nhwc:
        lin = cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1)))
        lat, v = G.conv_fire(lin, cu(w), pad, T, theta, nhwc=True, in_nhwc=True)
        lat, v = host(lat).transpose(0, 3, 1, 2), host(v).transpose(0, 3, 1, 2)
    else:
        lat, v = G.conv_fire(cu(lat_in), cu(w), pad, T, theta)
        lat, v = host(lat), host(v)
    G.sync_status()
    assert np.array_equal(lat, ol)
    assert np.array_equal(v, ov)
    monkeypatch.setenv("SNN_KMIN", "0")                  # and the same call without the bound
    lat0, v0 = G.conv_fire(cu(lat_in), cu(w), pad, T, theta)
    assert np.array_equal(host(lat0), ol) and np.array_equal(host(v0), ov)


FC_CASES = [
    # (B, C, H, W, pad, F, KH, KW, T, p_spike): theta = inf layers whose kernel is larger than the input (K9)
    (300, 32, 4, 4, 2, 40, 5, 5, 15, 0.8),      # C2 L3-like (4 x 4 map, 5 x 5 kernel), one M tile row ragged
    (300, 64, 3, 5, 2, 33, 5, 5, 7, 0.6),       # non-square map, F % 4 != 0
    (310, 64, 2, 4, 2, 20, 3, 7, 9, 0.7),       # non-square kernel: Ho x Wo = 4 x 2 from a 2 x 4 map
    (300, 250, 4, 4, 2, 200, 5, 5, 15, 0.9),    # C2 L3 shape (channels padded 250 -> 256, 3200 virtual features)
    (300, 48, 2, 2, 1, 16, 3, 3, 5, 0.5),       # 2 x 2 map, 3 x 3 kernel, pad 1
]


@pytest.mark.parametrize("layout", ["planar", "nhwc_out", "nhwc_in_out"])
@pytest.mark.parametrize("case", FC_CASES)
def test_conv_tc_fc_rewrite_vs_oracle(G, orc, case, layout, monkeypatch):
    """K9: Eq. 5 layers with H W < KH KW run as a fully connected tcgen05 GEMM (one row per image, Ho Wo F
    virtual features); bit-exact vs the oracle conv_fire, and identical to the im2col plan (SNN_TC_FC=0)."""
    monkeypatch.setenv("SNN_DEBUG_PLAN", "1")
    B, C, H, W, pad, F, KH, KW, T, p = case
    rng = np.random.default_rng(9100 + FC_CASES.index(case))
    import synth
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    lat_in[1] = 255                                      # an image with no input spike at all
    w = exact_weights(rng, (F, C, KH, KW))
    w[0, 0, 0, 0] = 0.0
    ol, ov = orc.conv_fire(lat_in, w, pad, T, math.inf)
    lin = cu(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))) if layout == "nhwc_in_out" else cu(lat_in)
    kw = dict(nhwc=layout != "planar", in_nhwc=layout == "nhwc_in_out")

    def run():
        lat, v = G.conv_fire(lin, cu(w), pad, T, math.inf, **kw)
        G.sync_status()
        lat, v = host(lat), host(v)
        return (lat.transpose(0, 3, 1, 2), v.transpose(0, 3, 1, 2)) if kw["nhwc"] else (lat, v)

    lat, v = run()
    assert np.array_equal(lat, ol)
    assert np.array_equal(v, ov)
    monkeypatch.setenv("SNN_TC_FC", "0")
    lat0, v0 = run()
    assert np.array_equal(lat0, ol) and np.array_equal(v0, ov)


@pytest.mark.parametrize("theta", [3.0, math.inf])
def test_conv_pot_out_vs_oracle_potentials(G, orc, theta):
    rng = np.random.default_rng(5)
    import synth
    B, C, H, W, pad, F, K, T = 2, 3, 10, 11, 1, 45, 3, 7
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, 0.6)
    w = exact_weights(rng, (F, C, K, K))
    lat, v, pot = G.conv_fire(cu(lat_in), cu(w), pad, T, theta, want_pot=True)
    for b in range(B):
        P = orc.potentials(lat_in[b], w, pad, T)
        assert np.array_equal(host(pot[b]), P.astype(np.float32))
        ol, ov = orc.fire(P, theta)
        assert np.array_equal(host(lat[b]), ol) and np.array_equal(host(v[b]), ov)


def test_conv_inexact_weight_flagged(G):
    lat_in = torch.zeros((1, 1, 4, 4), dtype=torch.uint8, device="cuda")
    w = torch.full((2, 1, 3, 3), 0.5, dtype=torch.float32, device="cuda")
    w[1, 0, 0, 0] = 1e-5                              # not a multiple of 2^-31
    G.conv_fire(lat_in, w, 0, 4, 1.0)
    with pytest.raises(G.SNNError) as e:
        G.sync_status()
    assert e.value.code == G.SNN_EINEXACT
    G.conv_fire(lat_in, w.clamp(min=0.5), 0, 4, 1.0)
    G.sync_status()                                   # cleared


def test_conv_errors(G):
    lat_in = torch.zeros((1, 1, 4, 4), dtype=torch.uint8, device="cuda")
    w = torch.full((2, 1, 7, 7), 0.5, dtype=torch.float32, device="cuda")
    with pytest.raises(G.SNNError):
        G.conv_fire(lat_in, w, 0, 4, 1.0)             # kernel larger than the padded input
    with pytest.raises(G.SNNError):
        G.conv_fire(lat_in, w[:, :, :3, :3].contiguous(), 0, 0, 1.0)   # T = 0


# ---------------------------------------------------------------------------------------- pool
@pytest.mark.parametrize("win,stride,pad,with_v", [((2, 2), (2, 2), (0, 0), True), ((3, 3), (3, 3), (0, 0), False),
                                                  ((7, 7), (6, 6), (0, 0), True), ((3, 2), (2, 1), (1, 1), True),
                                                  ((2, 3), (3, 2), (1, 0), True), ((1, 1), (1, 1), (0, 0), True)])
def test_pool_vs_oracle(G, orc, win, stride, pad, with_v):
    import synth
    rng = np.random.default_rng(3)
    T = 9
    lat = synth.random_latencies(rng, (3, 5, 37, 29), T, 0.5)
    v = synth.random_potentials_at_spike(rng, lat, 4)
    gl, gv = G.pool(cu(lat), cu(v) if with_v else None, win, stride, pad)
    ol, ov = orc.pool(lat, v if with_v else None, *win, *stride, *pad, T)
    assert np.array_equal(host(gl), ol)
    if with_v:
        assert np.array_equal(host(gv), ov)


# ---------------------------------------------------------------------------------------- inhibit
@pytest.mark.parametrize("F,levels,hw", [(1, 0, (13, 17)), (6, 3, (13, 17)), (30, 0, (13, 17)), (257, 2, (13, 17)),
                                         (7, 2, (131, 129)),
                                         (9, 3, (100, 100)), (1, 0, (128, 128)), (40, 2, (96, 96))])  # 4 positions/thread
def test_inhibit_vs_oracle(G, orc, F, levels, hw):
    """Small maps take the warp-per-position kernel, large ones (> 16384 positions) the thread one."""
    import synth
    rng = np.random.default_rng(F)
    lat = synth.random_latencies(rng, (2, F) + hw, 5, 0.4)
    v = synth.random_potentials_at_spike(rng, lat, levels)
    gl, gv, gw = G.inhibit(cu(lat), cu(v))
    ol, ov, ow = orc.inhibit(lat, v)
    assert np.array_equal(host(gl), ol) and np.array_equal(host(gv), ov) and np.array_equal(host(gw), ow)


# ---------------------------------------------------------------------------------------- k-WTA
@pytest.mark.parametrize("B,F,H,W,k,r,p,levels", [(4, 30, 28, 28, 5, 3, 0.3, 0), (3, 250, 14, 14, 8, 2, 0.5, 3),
                                                 (2, 7, 5, 6, 20, 0, 0.5, 2), (2, 3, 4, 4, 5, 1, 0.05, 0),
                                                 (2, 256, 64, 64, 16, 4, 0.2, 0), (3, 1, 9, 9, 3, 0, 1.0, 1),
                                                 (2, 4, 3, 3, 2, 5, 0.0, 0), (1, 9, 140, 141, 6, 3, 0.3, 2),
                                                 (2, 500, 12, 12, 16, 1, 0.7, 3),   # candidate lists, F near 512
                                                 (2, 600, 10, 10, 6, 1, 0.6, 2),    # F > 512: rescan path
                                                 (5, 200, 4, 4, 1, 0, 0.3, 3),      # k = 1: reduction path
                                                 (1, 100, 9, 24, 1, 0, 0.5, 2), (3, 40, 70, 70, 1, 2, 0.1, 1),
                                                 (2, 8, 5, 5, 1, 0, 0.0, 0),        # k = 1, nothing spikes
                                                 (4, 64, 64, 64, 8, 40, 0.3, 2),    # rescan path, window clipped
                                                 (1, 2, 128, 128, 3, 0, 0.9, 1),    # requeue overflow (smem map)
                                                 (1, 3, 150, 150, 4, 1, 0.9, 0),    # requeue overflow (global map)
                                                 (2, 20, 100, 100, 6, 2, 0.4, 1),   # 4-position best-key stage
                                                 (2, 5, 99, 101, 4, 1, 0.5, 2)])    # H*W odd: 1-position stage
def test_k_winners_vs_oracle(G, orc, B, F, H, W, k, r, p, levels):
    import synth
    rng = np.random.default_rng(B * 1000 + F)
    lat = synth.random_latencies(rng, (B, F, H, W), 6, p)
    v = synth.random_potentials_at_spike(rng, lat, levels)
    gw, gc = G.k_winners(cu(lat), cu(v), k, r)
    ow, oc = orc.k_winners(lat, v, k, r)
    assert np.array_equal(host(gc), oc)
    assert np.array_equal(host(gw), ow)


# ---------------------------------------------------------------------------------------- STDP
@pytest.mark.parametrize("reward,stab", [(1.0, 1), (-1.0, 1), (0.0, 1), (None, 0), (1.0, 0)])
def test_stdp_vs_oracle(G, orc, reward, stab):
    import synth
    rng = np.random.default_rng(7)
    F, C, K, H, W, pad, T = 12, 5, 3, 11, 9, 1, 8
    w = rng.random((F, C, K, K)).astype(np.float32)
    w[0, 0, 0, :] = [0.0, 1.0, 0.5]
    lat_in = synth.random_latencies(rng, (C, H, W), T, 0.6)
    Ho, Wo = H + 2 * pad - K + 1, W + 2 * pad - K + 1
    lat_out = synth.random_latencies(rng, (F, Ho, Wo), T, 0.7)
    v_out = synth.random_potentials_at_spike(rng, lat_out)
    win, cnt = orc.k_winners(lat_out[None], v_out[None], 4, 1)
    lb, ub = (0.0, 1.0) if stab else (0.2, 0.8)
    gw = cu(w)
    rt = None if reward is None else torch.tensor([reward], dtype=torch.float32, device="cuda")
    G.stdp_update(gw, cu(lat_in), pad, cu(lat_out), cu(win[0]), cu(cnt), 0.004, -0.003, lb, ub, stab, rt)
    ow = orc.stdp(w, lat_in, pad, lat_out, win[0], int(cnt[0]), 0.004, -0.003, lb, ub, stab,
                  1 if reward is None else int(reward))
    assert np.array_equal(host(gw), ow)


def test_decide_vs_oracle(G, orc):
    win = np.array([[[57, 1, 2]], [[3, 0, 0]], [[-1, -1, -1]]], np.int32)
    cnt = np.array([1, 1, 0], np.int32)
    lab = np.array([1, 1, 0], np.int32)
    d, rw = G.decide(cu(win), cu(cnt), 100, 2, cu(lab))
    exp = [orc.decide(win[b], cnt[b], 100, 2, int(lab[b])) for b in range(3)]
    assert host(d).tolist() == [e[0] for e in exp]
    assert host(rw).tolist() == [float(e[1]) for e in exp]


@pytest.mark.parametrize("shape", [(2, 3, 16, 24), (1, 2, 8, 4), (3, 5, 36, 40), (2, 4, 6, 12)])
@pytest.mark.parametrize("flags", [0, 2])
def test_pool_2x2_vector_path(G, orc, shape, flags):
    """2 x 2 / stride 2 pooling with potentials on W % 4 == 0 maps (the vectorised pair kernel), with
    latency ties inside windows, plain (R12) and final-potential (SNN_POOL_VFINAL) readings."""
    rng = np.random.default_rng(sum(shape) + flags)
    lat = rng.integers(0, 4, shape).astype(np.uint8)
    lat[rng.random(shape) < 0.4] = NS
    v = (rng.integers(1, 9, shape) / 8).astype(np.float32)
    gl, gv = G.pool(cu(lat), cu(v), 2, 2, 0, flags=flags)
    ol, ov = orc.pool(lat, v, 2, 2, 2, 2, 0, 0, T=4, vfinal=bool(flags & 2))
    assert np.array_equal(host(gl), ol) and np.array_equal(host(gv), ov)


@pytest.mark.parametrize("B,C,H,W,F,K,pad", [(1, 20, 25, 40, 100, 17, 0), (2, 64, 12, 12, 70, 5, 2)])
def test_conv_inf_split_k(G, orc, B, C, H, W, F, K, pad):
    """theta = inf on a grid too small to fill the GPU: the split-K GEMM (exact int64 partial sums)."""
    plan = G.conv_fire_plan(B, C, H, W, pad, F, K, K, 30, float("inf"))
    assert plan["launches"] == 4, plan  # prep B, prep A, split GEMM, finalize
    rng = np.random.default_rng(B + C)
    lat = rng.integers(0, 30, (B, C, H, W)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.5] = NS
    w = exact_weights(rng, (F, C, K, K))
    gl, gv = G.conv_fire(cu(lat), cu(w), pad, 30, float("inf"))
    ol, ov = orc.conv_fire(lat, w, pad, 30, float("inf"))
    assert np.array_equal(host(gl), ol) and np.array_equal(host(gv), ov)


@pytest.mark.parametrize("B,C,H,W,F,K,pad", [(5, 20, 25, 40, 100, 17, 0), (3, 6, 9, 11, 12, 3, 1)])
def test_conv_inf_prepared(G, orc, B, C, H, W, F, K, pad):
    """snn_conv_inf_prepare + snn_conv_fire_prepared (image by image) == the theta = inf conv per image."""
    rng = np.random.default_rng(B * 7 + C)
    lat = rng.integers(0, 30, (B, C, H, W)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.5] = NS
    w = exact_weights(rng, (F, C, K, K))
    prep = G.conv_inf_prepare(cu(lat), F, K, K, pad, 30)
    ol, ov = orc.conv_fire(lat, w, pad, 30, float("inf"))
    gw = cu(w)
    for b in range(B):
        gl, gv = G.conv_fire_prepared(prep, b, C, H, W, gw, pad, 30)
        assert np.array_equal(host(gl)[0], ol[b]) and np.array_equal(host(gv)[0], ov[b]), b


@pytest.mark.parametrize("shape", [(2, 3, 16, 24), (1, 30, 28, 28), (2, 2, 7, 8)])
def test_pool_2x2_latency_only(G, orc, shape):
    """2 x 2 / stride 2 pooling of latencies alone on W % 4 == 0 maps (the byte-SIMD word kernel)."""
    rng = np.random.default_rng(sum(shape))
    lat = rng.integers(0, 9, shape).astype(np.uint8)
    lat[rng.random(shape) < 0.5] = NS
    gl, _ = G.pool(cu(lat), None, 2)
    ol, _ = orc.pool(lat, None, 2, 2, 2, 2, 0, 0, T=9)
    assert np.array_equal(host(gl), ol)


@pytest.mark.parametrize("shape,win,stride", [((3, 7, 14, 14), 3, 3), ((2, 4, 12, 10), 2, 1), ((2, 3, 8, 8), 3, 2),
                                              ((1, 250, 14, 14), 3, 3)])
def test_pool_small_planes(G, orc, shape, win, stride):
    """Latency-only pooling of planes of <= 256 entries (one thread per plane through shared memory)."""
    rng = np.random.default_rng(sum(shape) + win)
    lat = rng.integers(0, 9, shape).astype(np.uint8)
    lat[rng.random(shape) < 0.5] = NS
    gl, _ = G.pool(cu(lat), None, win, stride)
    ol, _ = orc.pool(lat, None, win, win, stride, stride, 0, 0, T=9)
    assert np.array_equal(host(gl), ol)
