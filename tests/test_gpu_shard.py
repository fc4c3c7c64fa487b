"""GPU parity of the f4 feature-sharding kernels (snn_position_keys, snn_k_winners_keys,
snn_stdp_update_shard) and of FeatureShardedSTDP with two feature shards emulated in one process
(the MIN all-reduce replaced by torch.minimum of the two ranks' keys; one GPU is all this pool has)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_dist_shard import pack_keys

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


def _maps(seed, shape, T=8, p_ns=0.6, vq=None):
    rng = np.random.default_rng(seed)
    lat = rng.integers(0, T, shape).astype(np.uint8)
    lat[rng.random(shape) < p_ns] = NS
    v = (rng.integers(1, vq + 1, shape) / vq).astype(np.float32) if vq else rng.random(shape).astype(np.float32)
    return lat, v


@pytest.mark.parametrize("shape,f0", [((2, 9, 5, 7), 0), ((3, 40, 14, 14), 125), ((1, 300, 11, 13), 7)])
def test_position_keys(G, shape, f0):
    lat, v = _maps(shape[1], shape, vq=4)
    assert np.array_equal(G.position_keys(cu(lat), cu(v), f0).cpu().numpy(), pack_keys(lat, v, f0))


@pytest.mark.parametrize("shape,k,r", [((2, 30, 14, 14), 8, 2), ((3, 64, 20, 20), 16, 1), ((1, 16, 170, 170), 12, 4),
                                       ((2, 5, 3, 3), 9, 0)])
def test_k_winners_keys(G, shape, k, r):
    lat, v = _maps(shape[2] + k, shape, vq=3)
    il, iv, _ = oracle.inhibit(lat, v)
    rw, rc = oracle.k_winners(il, iv, k, r)
    keys = cu(pack_keys(lat, v, 0))
    gw, gc = G.k_winners_keys(keys, shape[1], k, r)
    assert np.array_equal(gw.cpu().numpy(), rw) and np.array_equal(gc.cpu().numpy(), rc)


def test_feature_sharded_c3_two_virtual_ranks(G):
    from oracle import flows
    from paper_1903_02440_b200 import dist, pipeline
    n = 60
    wl = synth.C3(n=n)
    ref = flows.c3(wl, n=n)
    lat0 = G.encode(cu(wl.X), wl.T)
    l1 = pipeline.Layer(wl.convs[0], cu(wl.weights[0]), n, 6, 28, 28, wl.T, wl.pools[0], pool_v=False)
    l1(lat0)
    assert np.array_equal(l1.plat.cpu().numpy(), ref["l1_pool_lat"])
    s, st = wl.convs[1], wl.extra["stdp"]
    ranks = [dist.FeatureShardedSTDP(s, cu(wl.weights[1]), wl.T, wl.extra["k"], wl.extra["r"], st, g, 2)
             for g in range(2)]
    for b in range(n):
        x = l1.plat[b:b + 1].contiguous()
        keys = torch.minimum(ranks[0].keys(x), ranks[1].keys(x))  # the all-reduce(MIN)
        outs = [rk.apply(x, keys) for rk in ranks]
        for win, cnt in outs:
            assert np.array_equal(win[0].cpu().numpy(), ref["winners"][b]), f"image {b}"
    w = torch.cat([rk.w for rk in ranks]).cpu().numpy()
    assert np.array_equal(w, ref["w2"])
