"""Config-level oracle flows on small samples: north_star invariants.  CPU only."""
import itertools

import numpy as np
import pytest

import synth

NS = 255


def _winner_ok(win, cnt, r):
    ws = win[:cnt]
    assert len({int(w[0]) for w in ws}) == len(ws)
    for a, b in itertools.combinations(ws, 2):
        assert max(abs(a[1] - b[1]), abs(a[2] - b[2])) > r


def test_c1_flow(orc):
    from oracle import flows
    wl = synth.C1()
    out = flows.c1(wl)
    assert out["lat1"].shape == (1, 30, 28, 28)
    assert np.all((out["inh_lat"] != NS).sum(axis=1) <= 1)
    assert out["count"][0] == 5
    _winner_ok(out["winners"][0], out["count"][0], 3)
    w0, w1 = wl.weights[0], out["w_new"]
    assert np.all((w1 >= 0) & (w1 <= 1))
    changed = np.where(np.any(w0 != w1, axis=(1, 2, 3)))[0]
    assert set(changed.tolist()) <= set(out["winners"][0, :, 0].tolist())


def test_c2_flow_small(orc):
    from oracle import flows
    wl = synth.C2(n=4)
    out = flows.c2(wl)
    assert out["l1"]["pool_lat"].shape == (4, 30, 14, 14)
    assert out["l2"]["pool_lat"].shape == (4, 250, 4, 4)
    assert out["l3"]["lat"].shape == (4, 200, 4, 4)
    l3 = out["l3"]["lat"]
    assert np.all((l3 == 14) | (l3 == NS))                     # Eq. 5: spikes only at T-1
    for b in range(4):
        if out["count"][b]:
            f, y, x = out["winners"][b, 0]
            assert out["l3"]["v"][b, f, y, x] == out["l3"]["v"][b].max()   # argmax readout


def test_c3_flow_small(orc):
    from oracle import flows
    wl = synth.C3(n=3)
    out = flows.c3(wl, snapshot_every=1)
    assert len(out["snapshots"]) == 3
    for b in range(3):
        _winner_ok(out["winners"][b], out["count"][b], 2)
    assert np.all((out["w2"] >= 0) & (out["w2"] <= 1))


def test_c4_flow_small(orc):
    from oracle import flows
    wl = synth.C4(n=2)
    assert wl.X.shape == (2, 4, 160, 250)
    out = flows.c4(wl)
    assert out["l1_pool_lat"].shape == (2, 20, 25, 40)
    assert set(out["reward"].tolist()) <= {-1, 0, 1}
    assert np.all((out["w2"] >= 0) & (out["w2"] <= 1))
