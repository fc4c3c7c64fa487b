"""Pins for oracle a6 (k-WTA) and a7 (STDP / R-STDP).  CPU only."""
import itertools

import numpy as np
import pytest

NS = 255


def _sort_then_greedy(lat, v, k, r):
    """Independent twin: sort all candidates by (lat, -v, flat index) once,
    then accept greedily unless excluded.  Equal to the round-based definition because exclusion
    only grows."""
    F, H, W = lat.shape
    cand = sorted((int(lat[f, y, x]), -float(v[f, y, x]), (f * H + y) * W + x, f, y, x)
                  for f in range(F) for y in range(H) for x in range(W) if lat[f, y, x] != NS)
    out = []
    for _, _, _, f, y, x in cand:
        if len(out) == k:
            break
        if any(f == g or (abs(y - yy) <= r and abs(x - xx) <= r) for g, yy, xx in out):
            continue
        out.append((f, y, x))
    return out


def test_spec_examples(orc):
    # S:332 single nonzero -> that location wins
    lat = np.full((1, 2, 3, 3), NS, np.uint8)
    v = np.zeros((1, 2, 3, 3), np.float32)
    lat[0, 1, 2, 0], v[0, 1, 2, 0] = 4, 1.0
    win, cnt = orc.k_winners(lat, v, 1, 0)
    assert cnt.tolist() == [1] and win[0, 0].tolist() == [1, 2, 0]
    # S:333 latencies (0, 1), potentials (0.1, 99) -> latency-0 wins
    lat = np.full((1, 1, 1, 2), NS, np.uint8)
    lat[0, 0, 0] = [0, 1]
    v = np.array([0.1, 99.0], np.float32).reshape(1, 1, 1, 2)
    win, cnt = orc.k_winners(lat, v, 1, 0)
    assert win[0, 0].tolist() == [0, 0, 0]
    # S:334 k=2, radius 1, two adjacent top candidates in different features -> the second winner
    # comes from outside the 3x3 inhibited square
    lat = np.full((1, 2, 4, 4), NS, np.uint8)
    v = np.zeros((1, 2, 4, 4), np.float32)
    lat[0, 0, 1, 1], v[0, 0, 1, 1] = 0, 5.0
    lat[0, 1, 1, 2], v[0, 1, 1, 2] = 0, 4.0      # adjacent -> inhibited
    lat[0, 1, 3, 3], v[0, 1, 3, 3] = 2, 1.0
    win, cnt = orc.k_winners(lat, v, 2, 1)
    assert cnt.tolist() == [2] and win[0].tolist() == [[0, 1, 1], [1, 3, 3]]


def test_fewer_than_k_and_padding(orc):
    lat = np.full((1, 3, 2, 2), NS, np.uint8)
    v = np.zeros((1, 3, 2, 2), np.float32)
    lat[0, 0, 0, 0], v[0, 0, 0, 0] = 1, 2.0
    win, cnt = orc.k_winners(lat, v, 4, 0)
    assert cnt.tolist() == [1] and win[0, 1:].tolist() == [[-1, -1, -1]] * 3
    lat[:] = NS
    win, cnt = orc.k_winners(lat, v, 2, 0)
    assert cnt.tolist() == [0] and np.all(win == -1)


def test_exhaustive_small_vs_sort_greedy(orc):
    # S:341 / S:613: 1000 random tensors, T<=4, F<=4, H=W<=6, k<=3, r<=2, exact incl. order
    rng = np.random.default_rng(123)
    for it in range(1000):
        T = int(rng.integers(1, 5)); F = int(rng.integers(1, 5)); H = int(rng.integers(1, 7))
        k = int(rng.integers(1, 4)); r = int(rng.integers(0, 3))
        lat = rng.integers(0, T, size=(1, F, H, H)).astype(np.uint8)
        lat[rng.random(lat.shape) < 0.5] = NS
        v = (rng.integers(1, 4, size=lat.shape) / 3).astype(np.float32)   # frequent ties
        v[lat == NS] = 0
        win, cnt = orc.k_winners(lat, v, k, r)
        ref = _sort_then_greedy(lat[0], v[0], k, r)
        assert cnt[0] == len(ref)
        assert [tuple(w) for w in win[0, :cnt[0]]] == ref


def test_winner_invariants(orc):
    import synth
    rng = np.random.default_rng(9)
    lat = synth.random_latencies(rng, (3, 8, 12, 12), 10, 0.5)
    v = synth.random_potentials_at_spike(rng, lat)
    win, cnt = orc.k_winners(lat, v, 6, 2)
    for b in range(3):
        ws = win[b, :cnt[b]]
        assert len({int(w[0]) for w in ws}) == len(ws)                  # distinct features
        for a, c in itertools.combinations(ws, 2):
            assert max(abs(a[1] - c[1]), abs(a[2] - c[2])) > 2           # > r apart
        for w in ws:
            assert lat[b, w[0], w[1], w[2]] != NS


# ------------------------------------------------------------------------------------ STDP

def _one_synapse(w0, pre, post, a_plus=0.1, a_minus=-0.05, lb=0.0, ub=1.0, stab=1, reward=1):
    w = np.array([[[[w0]]]], np.float32)                    # [F=1, C=1, 1, 1]
    lat_in = np.array([[[pre]]], np.uint8)
    lat_out = np.array([[[post]]], np.uint8)
    win = np.array([[0, 0, 0]], np.int32)
    return float(orc_ref.stdp(w, lat_in, 0, lat_out, win, 1, a_plus, a_minus, lb, ub, stab, reward)[0, 0, 0, 0])


@pytest.fixture(autouse=True)
def _bind(orc):
    global orc_ref
    orc_ref = orc


def test_eq4_closed_form():
    # W=0.5, LB=0, UB=1, A+=0.1, pre before post -> dW = 0.1*0.5*0.5 = 0.025
    assert abs(_one_synapse(0.5, 1, 3) - 0.525) < 1e-7
    # T_j == T_i counts as causal (Eq. 4 "T_j <= T_i")
    assert abs(_one_synapse(0.5, 3, 3) - 0.525) < 1e-7
    # anti-causal and no-spike pre -> A- branch: 0.5 - 0.05*0.25
    assert abs(_one_synapse(0.5, 4, 3) - 0.4875) < 1e-7
    assert abs(_one_synapse(0.5, NS, 3) - 0.4875) < 1e-7


def test_stabilizer_vanishes_at_bounds():
    # W in {LB, UB} -> dW = 0 exactly
    assert _one_synapse(0.0, 1, 3) == 0.0
    assert _one_synapse(1.0, 1, 3) == 1.0
    assert _one_synapse(0.2, 1, 3, lb=0.2, ub=0.8) == np.float32(0.2)


def test_stabilizer_off_and_clamp():
    # stabilizer off -> dW = A exactly, clamped at UB
    assert _one_synapse(0.5, 1, 3, a_plus=0.004, stab=0) == np.float32(np.float32(0.5) + np.float32(0.004))
    assert _one_synapse(0.799, 1, 3, a_plus=0.004, lb=0.2, ub=0.8, stab=0) == np.float32(0.8)


def test_rstdp_reward_punish_silent():
    # P:161 anti-STDP = negated learning rates; reward == STDP; 0 -> no change (R25)
    r = _one_synapse(0.5, 1, 3, reward=1)
    p = _one_synapse(0.5, 1, 3, reward=-1)
    s = _one_synapse(0.5, 1, 3, reward=0)
    assert abs(r - 0.525) < 1e-7 and abs(p - 0.475) < 1e-7 and s == 0.5


def test_locality_containment_sign(orc):
    # weights stay in [0,1]; non-winner features bit-identical; causal synapses never
    # decrease and anti-causal never increase (A+ > 0, A- < 0, stabilizer on)
    rng = np.random.default_rng(0)
    w = rng.random((5, 3, 3, 3)).astype(np.float32)
    w[0, 0, 0, 0], w[1, 0, 0, 0] = 0.0, 1.0
    lat_in = rng.integers(0, 6, size=(3, 6, 6)).astype(np.uint8)
    lat_in[rng.random(lat_in.shape) < 0.3] = NS
    lat_out = rng.integers(0, 6, size=(5, 6, 6)).astype(np.uint8)
    win = np.array([[0, 2, 3], [3, 5, 0], [1, 0, 0]], np.int32)
    w2 = orc.stdp(w, lat_in, 1, lat_out, win, 3, 0.004, -0.003)
    assert np.all((w2 >= 0) & (w2 <= 1))
    assert np.array_equal(w2[[2, 4]], w[[2, 4]])
    for f, y, x in win:
        post = lat_out[f, y, x]
        for c in range(3):
            for ky in range(3):
                for kx in range(3):
                    yy, xx = y + ky - 1, x + kx - 1
                    pre = lat_in[c, yy, xx] if 0 <= yy < 6 and 0 <= xx < 6 else NS
                    if pre != NS and pre <= post:
                        assert w2[f, c, ky, kx] >= w[f, c, ky, kx]
                    else:
                        assert w2[f, c, ky, kx] <= w[f, c, ky, kx]


def test_soft_bound_containment_random():
    # 10,000 random updates with |A| <= 1/(UB-LB) keep W in [LB, UB]
    rng = np.random.default_rng(1)
    for _ in range(10000 // 100):
        w0s = rng.random(100).astype(np.float32)
        for w0 in w0s[:100]:
            a = float(rng.uniform(-1, 1))
            out = _one_synapse(float(w0), 1, 3, a_plus=a, a_minus=a)
            assert 0.0 <= out <= 1.0


def test_decide(orc):
    win = np.array([[57, 1, 2]], np.int32)
    assert orc.decide(win, 1, 100, 2, 1) == (1, 1)       # 57 // 50 = 1 == label -> reward
    assert orc.decide(win, 1, 100, 2, 0) == (1, -1)      # mismatch -> punish
    assert orc.decide(win, 0, 100, 2, 0) == (-1, 0)      # silent
    assert orc.decide(np.array([[39, 0, 0]], np.int32), 1, 200, 10, 1) == (1, 1)   # C2: 39 // 20
