"""GPU robustness of the C ABI: device-side error reporting per stream, malformed winners in STDP,
pointer alignment of the vector pool paths, per-device caches."""
import numpy as np
import pytest
import torch

from test_gpu_kernels import cu, exact_weights, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1903_02440_b200 import build, snn
    build.build()
    snn.lib()
    return snn


def test_error_word_is_per_stream(G):
    """An inexact weight flagged by work on stream A is reported by snn_sync_status(A) only."""
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    lat_in = torch.zeros((1, 1, 4, 4), dtype=torch.uint8, device="cuda")
    w_bad = torch.full((2, 1, 3, 3), 0.5, dtype=torch.float32, device="cuda")
    w_bad[1, 0, 0, 0] = 1e-5                       # not a multiple of 2^-31
    w_ok = torch.full((2, 1, 3, 3), 0.5, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    G.conv_fire(lat_in, w_bad, 0, 4, 1.0, stream=sa)
    G.conv_fire(lat_in, w_ok, 0, 4, 1.0, stream=sb)
    G.sync_status(sb)                              # stream B saw no inexact weight
    with pytest.raises(G.SNNError) as e:
        G.sync_status(sa)
    assert e.value.code == G.SNN_EINEXACT
    G.sync_status(sa)                              # read and cleared
    torch.cuda.synchronize()


@pytest.mark.parametrize("bad", [(3, 0, 0), (-1, 0, 0), (0, 9, 0), (0, 0, -2)])
def test_stdp_rejects_winner_outside_map(G, orc, bad):
    """snn_stdp_update skips a winner outside [0, F) x [0, Ho) x [0, Wo) and reports SNN_EINVAL at
    snn_sync_status; the valid winners are still updated exactly (oracle)."""
    import synth
    rng = np.random.default_rng(7)
    F, C, H, W, K, pad, T = 3, 2, 8, 8, 3, 1, 6
    lat_in = synth.random_latencies(rng, (C, H, W), T, 0.6)
    lat_out = synth.random_latencies(rng, (F, H, W), T, 0.6)
    w = exact_weights(rng, (F, C, K, K))
    win = np.array([[1, 2, 3], list(bad)], dtype=np.int32)
    cnt = np.array([2], dtype=np.int32)
    wg = cu(w).clone()
    G.stdp_update(wg, cu(lat_in), pad, cu(lat_out), cu(win), cu(cnt), 0.004, -0.003)
    with pytest.raises(G.SNNError) as e:
        G.sync_status()
    assert e.value.code == G.SNN_EINVAL
    ref = orc.stdp(w, lat_in, pad, lat_out, win[:1], 1, 0.004, -0.003, 0.0, 1.0, 1)
    assert np.array_equal(host(wg), ref)


def test_stdp_shard_skips_other_ranks_silently(G):
    F, C, H, W, K, pad, T = 3, 2, 8, 8, 3, 1, 6
    lat_in = torch.zeros((C, H, W), dtype=torch.uint8, device="cuda")
    lat_out = torch.zeros((F, H, W), dtype=torch.uint8, device="cuda")
    w = torch.full((F, C, K, K), 0.5, dtype=torch.float32, device="cuda")
    win = torch.tensor([[7, 1, 1]], dtype=torch.int32, device="cuda")   # owned by another rank
    cnt = torch.tensor([1], dtype=torch.int32, device="cuda")
    G.stdp_update(w, lat_in, pad, lat_out, win, cnt, 0.004, -0.003, f_offset=0)
    G.sync_status()
    assert bool((w == 0.5).all())


@pytest.mark.parametrize("with_v", [True, False])
def test_pool_vector_paths_on_misaligned_views(G, orc, with_v):
    """2 x 2 / 2 pooling of tensors that start at an odd offset inside their storage: the 4-/16-byte
    vector kernels are not used (they would fault); the result is still exact."""
    import synth
    rng = np.random.default_rng(3)
    T = 9
    lat = synth.random_latencies(rng, (2, 5, 16, 24), T, 0.5)
    v = synth.random_potentials_at_spike(rng, lat, 3)
    lbuf = torch.empty(lat.size + 3, dtype=torch.uint8, device="cuda")
    vbuf = torch.empty(v.size + 3, dtype=torch.float32, device="cuda")
    lview = lbuf[1:1 + lat.size].view(lat.shape)
    vview = vbuf[1:1 + v.size].view(v.shape)
    lview.copy_(cu(lat))
    vview.copy_(cu(v))
    obuf = torch.empty(lat.size // 4 + 3, dtype=torch.uint8, device="cuda")
    ovbuf = torch.empty(lat.size // 4 + 3, dtype=torch.float32, device="cuda")
    lo = obuf[1:1 + lat.size // 4].view(2, 5, 8, 12)
    vo = ovbuf[1:1 + lat.size // 4].view(2, 5, 8, 12)
    G.pool(lview, vview if with_v else None, 2, 2, 0, lat_out=lo, v_out=vo if with_v else None)
    G.sync_status()
    ol, ov = orc.pool(lat, v if with_v else None, 2, 2, 2, 2, 0, 0, T)
    assert np.array_equal(host(lo), ol)
    if with_v:
        assert np.array_equal(host(vo), ov)
