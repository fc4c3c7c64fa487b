"""Pins for oracle a4 (pooling) and a5 (pointwise inhibition).  CPU only."""
import numpy as np
import pytest
import torch

NS = 255


def _rand(seed, B=2, F=3, H=9, W=8, T=7, p=0.6, levels=0):
    import synth
    rng = np.random.default_rng(seed)
    lat = synth.random_latencies(rng, (B, F, H, W), T, p)
    v = synth.random_potentials_at_spike(rng, lat, levels)
    return lat, v


def test_shape_eq3_window_equals_stride(orc):
    # Eq. 3 holds when window = stride; e.g. 28 / 2 -> 14
    rng = np.random.default_rng(1)
    for _ in range(100):
        P = int(rng.integers(1, 5))
        H, W = [int(v) for v in rng.integers(P, 20, size=2)]
        D = int(rng.integers(0, P))
        assert orc.pool_out_hw(H, W, P, P, P, P, D, D) == ((H + 2 * D) // P, (W + 2 * D) // P)
    assert orc.pool_out_hw(28, 28, 2, 2, 2, 2) == (14, 14)
    assert orc.pool_out_hw(156, 246, 7, 7, 6, 6) == (25, 40)   # C4, reading A10


@pytest.mark.parametrize("win,stride,pad", [((2, 2), (2, 2), (0, 0)), ((3, 3), (3, 3), (0, 0)),
                                           ((7, 7), (6, 6), (0, 0)), ((3, 2), (2, 1), (1, 1)),
                                           ((2, 3), (3, 2), (1, 0))])
def test_pool_vs_torch_maxpool(orc, win, stride, pad):
    """Library cross-check (P:97 two-dimensional max-pooling): per time step, max_pool2d of the
    materialised wave S[t] (padding = no spike) gives the pooled wave; v is the max of
    thr(P)[lat_o] = v_i over the window entries that spiked at lat_o."""
    T = 7
    lat, v = _rand(hash(win + stride + pad) % 1000, T=T)
    lo, vo = orc.pool(lat, v, win[0], win[1], stride[0], stride[1], pad[0], pad[1], T)
    S = torch.from_numpy(orc.expand(lat, T)).double()                       # [B, T, F, H, W]
    B, _, F, H, W = S.shape
    pooled = torch.nn.functional.max_pool2d(S.reshape(B * T, F, H, W), win, stride, pad)
    pooled = pooled.reshape(B, T, F, *pooled.shape[-2:]).numpy()
    assert np.array_equal(orc.expand(lo, T), pooled.astype(np.float32))
    # v: per-t max-pool of thresholded potentials read at lat_o.  thr(P_i)[t] = v_i at t = lat_i;
    # for t > lat_i the paper's P_i[t] is not represented, but no window member has lat_i < lat_o.
    thr = np.where(lat == NS, 0.0, v).astype(np.float64)
    tv = torch.nn.functional.max_pool2d(
        torch.from_numpy(np.where(lat[:, None] == np.arange(T)[None, :, None, None, None], thr[:, None], 0.0))
        .reshape(B * T, F, H, W), win, stride, pad).reshape(B, T, F, *lo.shape[-2:]).numpy()
    exp_v = np.where(lo == NS, 0.0, np.take_along_axis(tv, np.minimum(lo, T - 1)[:, None].astype(np.int64), 1)[:, 0])
    assert np.array_equal(vo, exp_v.astype(np.float32))


def test_pool_window_min_bruteforce(orc):
    # S:340 / S:614: pooled latency = window-minimum latency (500 random tensors)
    rng = np.random.default_rng(5)
    for it in range(500):
        H, W = [int(x) for x in rng.integers(2, 7, size=2)]
        PH, PW = [int(x) for x in rng.integers(1, 3, size=2)]
        SH, SW = [int(x) for x in rng.integers(1, 3, size=2)]
        lat = rng.integers(0, 5, size=(1, 2, H, W)).astype(np.uint8)
        lat[rng.random(lat.shape) < 0.3] = NS
        lo, _ = orc.pool(lat, None, PH, PW, SH, SW, 0, 0, 5)
        Ho, Wo = orc.pool_out_hw(H, W, PH, PW, SH, SW)
        for f in range(2):
            for y in range(Ho):
                for x in range(Wo):
                    assert lo[0, f, y, x] == lat[0, f, y * SH:y * SH + PH, x * SW:x * SW + PW].min()


def test_inhibit_spec_examples(orc):
    # S:312 single feature -> identity
    lat = np.array([[[[3, NS]]]], np.uint8)
    v = np.array([[[[2.0, 0.0]]]], np.float32)
    lo, vo, wf = orc.inhibit(lat, v)
    assert np.array_equal(lo, lat) and np.array_equal(vo, v) and wf.tolist() == [[[0, -1]]]
    # S:313 latencies (1, 2) -> the latency-1 feature survives regardless of potentials
    lat = np.array([1, 2], np.uint8).reshape(1, 2, 1, 1)
    v = np.array([0.1, 99.0], np.float32).reshape(1, 2, 1, 1)
    lo, vo, wf = orc.inhibit(lat, v)
    assert lo.ravel().tolist() == [1, NS] and vo.ravel().tolist() == [np.float32(0.1), 0.0] and wf.ravel().tolist() == [0]
    # S:314 equal latencies, potentials (0.4, 0.9) -> second survives
    lat = np.array([3, 3], np.uint8).reshape(1, 2, 1, 1)
    v = np.array([0.4, 0.9], np.float32).reshape(1, 2, 1, 1)
    lo, vo, wf = orc.inhibit(lat, v)
    assert lo.ravel().tolist() == [NS, 3] and wf.ravel().tolist() == [1]
    # full tie -> lowest feature (R14)
    v = np.array([0.9, 0.9], np.float32).reshape(1, 2, 1, 1)
    assert orc.inhibit(lat, v)[2].ravel().tolist() == [0]


def test_inhibit_invariants(orc):
    lat, v = _rand(3, F=6, levels=3)
    lo, vo, wf = orc.inhibit(lat, v)
    assert np.all((lo != NS).sum(axis=1) <= 1)                 # <= 1 feature per position
    B, F, H, W = lat.shape
    for b in range(B):
        for y in range(H):
            for x in range(W):
                cand = [(int(lat[b, f, y, x]), -float(v[b, f, y, x]), f) for f in range(F) if lat[b, f, y, x] != NS]
                if not cand:
                    assert wf[b, y, x] == -1 and np.all(lo[b, :, y, x] == NS)
                else:
                    f = min(cand)[2]
                    assert wf[b, y, x] == f and lo[b, f, y, x] == lat[b, f, y, x] and vo[b, f, y, x] == v[b, f, y, x]
