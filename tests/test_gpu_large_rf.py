"""GPU parity: finite-threshold conv+fire on receptive fields too large for a shared-memory weight
slice (Eq. 2 at any kernel size): the presorted walk gathering from the prepared fixed-point
slice in global memory (conv_walk.cu, GW).  Bit-exact against the oracle's conv_fire (lat and v)."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [
    # (B, C, H, W, pad, F, K, T, theta, p_spike)
    (3, 250, 4, 4, 2, 200, 5, 15, 300.0, 0.9),     # C2 layer 3 at a finite threshold (R = 6,250)
    (3, 250, 4, 4, 2, 200, 5, 15, 2900.0, 0.9),    # threshold near the full sum: many never fire
    (1, 20, 25, 40, 0, 100, 17, 30, 400.0, 0.7),   # C4 layer 2 at a finite threshold (R = 5,780)
    (2, 80, 7, 9, 1, 33, 5, 9, 150.0, 0.6),        # R = 2,000, F = 33 (FPL 1, two groups, ragged)
    (2, 120, 6, 6, 2, 64, 5, 20, -0.5, 0.5),       # theta < 0: every neuron fires at t = 0
]


@pytest.fixture(scope="module")
def G():
    from paper_1903_02440_b200 import build, snn
    build.build()
    snn.lib()
    return snn


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("layout", ["planar", "nhwc"])
def test_large_rf_walk_vs_oracle(G, orc, case, layout):
    B, C, H, W, pad, F, K, T, theta, p = case
    plan = G.conv_fire_plan(B, C, H, W, pad, F, K, K, T, theta)
    assert plan["path"] == "walk_presorted_global", plan
    import synth
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = rng.uniform(2 ** -8, 1.0, size=(F, C, K, K)).astype(np.float32)
    w[0, :3, 0, 0] = 0.0
    if layout == "nhwc":
        li = torch.from_numpy(np.ascontiguousarray(lat_in.transpose(0, 2, 3, 1))).cuda()
        lat, v = G.conv_fire(li, torch.from_numpy(w).cuda(), pad, T, theta, nhwc=True, in_nhwc=True)
        lat, v = lat.permute(0, 3, 1, 2), v.permute(0, 3, 1, 2)
    else:
        lat, v = G.conv_fire(torch.from_numpy(lat_in).cuda(), torch.from_numpy(w).cuda(), pad, T, theta)
    G.sync_status()
    ol, ov = orc.conv_fire(lat_in, w, pad, T, theta)
    assert np.array_equal(lat.cpu().numpy(), ol)
    assert np.array_equal(v.cpu().numpy(), ov)
    if theta > 0 and theta < 1000:
        assert (ol != 255).mean() > 0.2   # the case exercises firing
