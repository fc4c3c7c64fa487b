"""GPU parity of the f3 variants against the oracle, bit-exact:
encoding bin rules (snn_encode_ex), Eq. 3 pooling size and pooled final potentials (snn_pool_ex),
the final-potential (A13) inhibition / k-WTA flow, stabilized no-clamp STDP and the paper's
stabilizer-off [0.2, 0.8] R-STDP bounds, per call and through the persistent kernel."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import synth

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


ENC = [((3, 6, 28, 28), 15, 0.5), ((2, 32, 40, 40), 32, 0.5), ((2, 1, 5, 5), 30, 0.0), ((2, 2, 9, 9), 1, 0.2),
       ((1, 4, 80, 80), 254, 0.3), ((2, 3, 17, 19), 7, 0.97)]


@pytest.mark.parametrize("bins", [1, 2])
@pytest.mark.parametrize("case", ENC, ids=[f"{'x'.join(map(str, c[0]))}-T{c[1]}" for c in ENC])
def test_encode_bins(G, case, bins):
    shape, T, zero = case
    rng = np.random.default_rng(T + shape[1])
    x = rng.random(shape).astype(np.float32)
    x[rng.random(shape) < zero] = 0.0
    x.reshape(-1)[::7] = np.float32(0.25)  # ties
    assert np.array_equal(host(G.encode(cu(x), T, bins=bins)), oracle.encode(x, T, bins=bins))


POOL = [(2, 5, 156, 246, 7, 6, 0), (2, 8, 13, 17, 3, 2, 1), (3, 4, 24, 24, 2, 2, 0), (1, 3, 9, 11, 3, 3, 0)]


@pytest.mark.parametrize("flags", [1, 2, 3])
@pytest.mark.parametrize("case", POOL, ids=[f"{c[2]}x{c[3]}-p{c[4]}s{c[5]}d{c[6]}" for c in POOL])
def test_pool_ex(G, case, flags):
    B, F, H, W, P, S, D = case
    rng = np.random.default_rng(H + W + flags)
    lat = rng.integers(0, 12, (B, F, H, W)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.6] = NS
    v = rng.random(lat.shape).astype(np.float32)
    lo, vo = G.pool(cu(lat), cu(v), P, S, D, flags=flags)
    rl, rv = oracle.pool(lat, v, P, P, S, S, D, D, T=12, eq3=bool(flags & 1), vfinal=bool(flags & 2))
    assert np.array_equal(host(lo), rl) and np.array_equal(host(vo), rv)


@pytest.mark.parametrize("pooled", [False, True])
def test_final_potential_flow(G, pooled):
    """A13: inhibition and k-WTA ranked by the final potential P[T-1] instead of the potential at the
    spike.  GPU: P[T-1] from the Eq. 5 conv (theta = inf, tensor cores), pooled with SNN_POOL_VFINAL.
    Oracle: P[T-1] read off the per-t potentials (orc_potentials), pooled with vfinal."""
    rng = np.random.default_rng(7 + pooled)
    B, C, H, W, F, T, theta, k, r = 3, 8, 24, 24, 32, 16, 30.0, 4, 2
    x = rng.random((B, C, H, W)).astype(np.float32)
    x[rng.random(x.shape) < 0.5] = 0.0
    w = np.clip(rng.normal(0.5, 0.1, (F, C, 5, 5)), 0, 1).astype(np.float32)
    lat_in = oracle.encode(x, T)
    lat, _ = oracle.conv_fire(lat_in, w, 2, T, theta)
    vfin = np.stack([oracle.potentials(lat_in[b], w, 2, T)[T - 1] for b in range(B)]).astype(np.float32)
    if pooled:
        lat, vfin = oracle.pool(lat, vfin, 2, 2, 2, 2, T=T, vfinal=True)
    il, iv, _ = oracle.inhibit(lat, vfin)
    rwin, rcnt = oracle.k_winners(il, iv, k, r)

    gl_in = cu(lat_in)
    gl, _ = G.conv_fire(gl_in, cu(w), 2, T, theta)
    _, gvf = G.conv_fire(gl_in, cu(w), 2, T, float("inf"))
    if pooled:
        gl, gvf = G.pool(gl, gvf, 2, flags=G.POOL_VFINAL)
    gil, giv, _ = G.inhibit(gl, gvf)
    gwin, gcnt = G.k_winners(gil, giv, k, r)
    assert np.array_equal(host(gil), il) and np.array_equal(host(giv), iv)
    assert np.array_equal(host(gwin), rwin) and np.array_equal(host(gcnt), rcnt)


@pytest.mark.parametrize("stab,lb,ub,reward", [(2, 0.2, 0.8, 1), (0, 0.2, 0.8, -1), (0, 0.2, 0.8, 1), (2, 0.0, 1.0, -1)])
def test_stdp_variants(G, stab, lb, ub, reward):
    rng = np.random.default_rng(stab * 10 + reward + 5)
    C, H, W, F, KH, T = 6, 14, 14, 20, 5, 15
    w = np.clip(rng.normal(0.8, 0.05, (F, C, KH, KH)), 0, 1).astype(np.float32)
    lat_in = rng.integers(0, T, (C, H, W)).astype(np.uint8)
    lat_in[rng.random(lat_in.shape) < 0.4] = NS
    lat_out = rng.integers(0, T, (F, H, W)).astype(np.uint8)
    win = np.array([[3, 2, 7], [11, 9, 1], [0, 13, 13]], np.int32)
    ref = oracle.stdp(w, lat_in, 2, lat_out, win, 3, 0.004, -0.003, lb, ub, stabilizer=stab, reward=reward)
    gw = cu(w)
    G.stdp_update(gw, cu(lat_in), 2, cu(lat_out), cu(win), cu(np.array([3], np.int32)), 0.004, -0.003, lb, ub,
                  stabilizer=stab, reward=cu(np.array([float(reward)], np.float32)))
    assert np.array_equal(host(gw), ref)


@pytest.mark.parametrize("stab", [0, 2])
def test_persistent_sequence_variant_bounds(G, stab):
    """C3's chain with the paper's tutorial bounds [0.2, 0.8] through snn_stdp_sequence."""
    from oracle import flows
    from paper_1903_02440_b200 import pipeline
    n = 120
    wl = synth.C3(n=n)
    wl = dataclasses.replace(wl, extra=dict(wl.extra, stdp=dict(wl.extra["stdp"], lb=0.2, ub=0.8, stabilizer=stab)))
    ref = flows.c3(wl, snapshot_every=60)
    lat0 = G.encode(cu(wl.X), wl.T)
    l1 = pipeline.Layer(wl.convs[0], cu(wl.weights[0]), n, 6, 28, 28, wl.T, wl.pools[0], pool_v=False)
    l1(lat0)
    s, st = wl.convs[1], wl.extra["stdp"]
    w = cu(wl.weights[1]).clone()
    win, cnt = G.stdp_sequence(l1.plat.contiguous(), w, s.pad, wl.T, s.theta, wl.extra["k"], wl.extra["r"],
                               st["a_plus"], st["a_minus"], st["lb"], st["ub"], st["stabilizer"])
    G.sync_status()
    assert np.array_equal(host(win), ref["winners"])
    assert np.array_equal(host(w), ref["w2"])


def test_variant_argument_errors(G):
    x = cu(np.ones((1, 1, 4, 4), np.float32))
    with pytest.raises(G.SNNError):
        G.encode(x, 4, bins=3)
    lat = cu(np.zeros((1, 1, 4, 4), np.uint8))
    with pytest.raises(G.SNNError):
        G.pool(lat, None, 2, flags=4)
