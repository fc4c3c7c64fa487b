"""f1 for theta = +inf: snn_rstdp_inf_sequence vs the oracle chain image by image
(conv Eq. 5 -> k-WTA k = 1 -> decide -> R-STDP, Eq. 4): every winner,
decision, reward and the final weights bit-exact, with silent images, labels = NULL (no plasticity),
both clamp variants and a split-K GEMM (one-image plan); the persistent one-launch kernel and the
per-image kernels."""
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


def oracle_chain(orc, lat_in, w, pad, T, labels, n_classes, ap, am, lb, ub, stab):
    w = w.copy()
    win_all, dec_all, rw_all = [], [], []
    F = w.shape[0]
    for b in range(lat_in.shape[0]):
        lat, v = orc.conv_fire(lat_in[b:b + 1], w, pad, T, float("inf"))
        win, cnt = orc.k_winners(lat, v, 1, 0)
        lab = -1 if labels is None else int(labels[b])
        d, rw = orc.decide(win[0], cnt[0], F, n_classes, lab)
        if labels is None:
            rw = 0
        w = orc.stdp(w, lat_in[b], pad, lat[0], win[0], cnt[0], ap, am, lb, ub, stab, rw)
        win_all.append(win[0, 0]); dec_all.append(d); rw_all.append(rw)
    return w, np.array(win_all), np.array(dec_all), np.array(rw_all, dtype=np.float32)


@pytest.mark.parametrize("shape,n_cls,stab,lb,ub,use_labels", [
    ((6, 5, 9, 13, 0, 20, 5, 5, 12), 2, 1, 0.0, 1.0, True),      # (N, C, H, W, pad, F, KH, KW, T)
    ((5, 20, 25, 40, 0, 100, 17, 17, 30), 2, 1, 0.0, 1.0, True),  # C4's layer shape
    ((4, 3, 8, 8, 1, 12, 3, 3, 7), 3, 0, 0.2, 0.8, True),         # the tutorial's stabilizer-off bounds
    ((4, 3, 8, 8, 1, 12, 3, 3, 7), 4, 2, 0.0, 1.0, True),         # stabilized, no clamp (A20 variant)
    ((3, 4, 10, 10, 0, 16, 5, 5, 9), 2, 1, 0.0, 1.0, False),      # labels NULL: decisions, no plasticity
])
@pytest.mark.parametrize("path", ["persistent", "percall"])
def test_rstdp_inf_sequence_vs_oracle(G, orc, shape, n_cls, stab, lb, ub, use_labels, path, monkeypatch):
    """persistent = one cooperative kernel for the whole chain (SNN_RSTDP_PERSIST=1); percall = the default
    per-image GEMM + two tail kernels"""
    if path == "persistent":
        monkeypatch.setenv("SNN_RSTDP_PERSIST", "1")
    N, C, H, W, pad, F, KH, KW, T = shape
    rng = np.random.default_rng(sum(shape) + stab)
    import synth
    lat_in = synth.random_latencies(rng, (N, C, H, W), T, 0.5)
    lat_in[1] = 255                                     # a silent image: no spike anywhere
    w = exact_weights(rng, (F, C, KH, KW), lo=0.3)
    labels = rng.integers(0, n_cls, size=N).astype(np.int32)
    ap, am = 0.004, -0.003
    prep = G.conv_inf_prepare(cu(lat_in), F, KH, KW, pad, T)
    wg = cu(w).clone()
    win, cnt, dec, rw = G.rstdp_inf_sequence(prep, 0, cu(lat_in), wg, pad, T, cu(labels) if use_labels else None,
                                             n_cls, ap, am, lb, ub, stab)
    G.sync_status()
    ow, owin, odec, orw = oracle_chain(orc, lat_in, w, pad, T, labels if use_labels else None, n_cls, ap, am, lb, ub,
                                       stab)
    assert np.array_equal(host(win), owin)
    assert np.array_equal(host(cnt), (owin[:, 0] >= 0).astype(np.int32))
    assert np.array_equal(host(dec), odec)
    assert np.array_equal(host(rw), orw)
    assert np.array_equal(host(wg), ow)
