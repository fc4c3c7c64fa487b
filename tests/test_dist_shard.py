"""f4 feature sharding: the FeatureShardedSTDP orchestration run by two gloo ranks on CPU,
with reference ops built from the oracle (conv+fire, STDP) and an independent numpy packing of the
position keys, must reproduce the unsharded oracle C3 chain image by image.  This pins the protocol --
the key format, the MIN all-reduce, k-WTA on the reduced map, STDP ownership -- independently of the GPU
kernels, which tests/test_gpu_variants.py checks against the same packing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

NS = 255


def pack_keys(lat, v, f0):
    """Independent numpy packing: (lat << 55) | (~order(v) << 23) | f, INT64_MAX where nothing spikes."""
    B, F, H, W = lat.shape
    bits = v.astype(np.float32).view(np.uint32).astype(np.uint64)
    order = np.where(bits & 0x80000000, ~bits & 0xFFFFFFFF, bits | 0x80000000)
    key = (lat.astype(np.uint64) << 55) | ((~order & 0xFFFFFFFF) << 23) | (np.arange(F, dtype=np.uint64) + f0)[None, :, None, None]
    key = np.where(lat == NS, np.uint64((1 << 63) - 1), key)
    return key.min(axis=1).astype(np.int64)


def unpack_to_map(keys, F):
    """Inhibited map [B, F, H, W] (lat, v) described by reduced keys."""
    B, H, W = keys.shape
    lat = np.full((B, F, H, W), NS, np.uint8)
    v = np.zeros((B, F, H, W), np.float32)
    k = keys.astype(np.uint64)
    live = keys != (1 << 63) - 1
    f = (k & 0x7FFFFF).astype(np.int64)
    order = ~((k >> 23) & 0xFFFFFFFF) & 0xFFFFFFFF
    vb = (order & 0x7FFFFFFF).astype(np.uint32).view(np.float32)
    b, y, x = np.nonzero(live)
    lat[b, f[b, y, x], y, x] = (k[b, y, x] >> 55).astype(np.uint8)
    v[b, f[b, y, x], y, x] = vb[b, y, x]
    return lat, v


class OracleOps:
    def __init__(self):
        import oracle
        self.o = oracle

    def conv_fire(self, lat_in, w, pad, T, theta):
        lat, v = self.o.conv_fire(lat_in.numpy(), w.numpy(), pad, T, theta)
        return torch.from_numpy(lat), torch.from_numpy(v)

    def position_keys(self, lat, v, f0):
        return torch.from_numpy(pack_keys(lat.numpy(), v.numpy(), f0))

    def k_winners_keys(self, keys, F, k, r):
        lat, v = unpack_to_map(keys.numpy(), F)
        win, cnt = self.o.k_winners(lat, v, k, r)
        return torch.from_numpy(win), torch.from_numpy(cnt)

    def stdp_update_shard(self, w, lat_in, pad, lat_out, winners, count, rates, f0):
        F = w.shape[0]
        win = winners.numpy()[: int(count[0])]
        own = win[(win[:, 0] >= f0) & (win[:, 0] < f0 + F)].copy()
        own[:, 0] -= f0
        new = self.o.stdp(w.numpy(), lat_in.numpy(), pad, lat_out.numpy(), own, len(own), rates["a_plus"],
                          rates["a_minus"], rates["lb"], rates["ub"], rates["stabilizer"], 1)
        w.copy_(torch.from_numpy(new))
        return w


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


N_IMG = 10


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), OMP_NUM_THREADS="2")
    import synth
    from oracle import flows
    from paper_1903_02440_b200 import dist
    dist.init("gloo")
    wl = synth.C3(n=N_IMG)
    ref = flows.c3(wl, n=N_IMG)
    s = wl.convs[1]
    sh = dist.FeatureShardedSTDP(s, torch.from_numpy(wl.weights[1]), wl.T, wl.extra["k"], wl.extra["r"],
                                 wl.extra["stdp"], rank, world, ops=OracleOps())
    lat_in = torch.from_numpy(ref["l1_pool_lat"])
    ok_win = True
    for b in range(N_IMG):
        win, cnt = sh.step(lat_in[b:b + 1])
        ok_win &= np.array_equal(win[0].numpy(), ref["winners"][b])
    ok_w = np.array_equal(sh.w.numpy(), ref["w2"][sh.f0:sh.f1])
    q.put((rank, sh.f0, sh.f1, bool(ok_win), bool(ok_w)))
    import torch.distributed as td
    td.destroy_process_group()


def test_pack_unpack_matches_oracle_inhibition():
    import oracle
    rng = np.random.default_rng(3)
    lat = rng.integers(0, 6, (2, 9, 5, 7)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.5] = NS
    v = (rng.integers(1, 4, lat.shape) / 4).astype(np.float32)   # ties in (lat, v): feature order decides
    il, iv, _ = oracle.inhibit(lat, v)
    keys = np.minimum(pack_keys(lat[:, :4], v[:, :4], 0), pack_keys(lat[:, 4:], v[:, 4:], 4))
    ml, mv = unpack_to_map(keys, 9)
    assert np.array_equal(ml, il)
    assert np.array_equal(np.where(ml == NS, 0, mv), np.where(il == NS, 0, iv))


def test_feature_sharded_c3_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, w0, ww0), (r1, a1, b1, w1, ww1) = res
    assert (a0, b0, a1, b1) == (0, 125, 125, 250)
    assert w0 and w1, "winners differ from the unsharded chain"
    assert ww0 and ww1, "weights differ from the unsharded chain"
