"""Pins for oracle a2 (potentials) and a3 (fire).  CPU only."""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

from conftest import read_golden

NS = 255


def _rand_case(seed, C=3, H=7, W=6, F=4, K=3, T=6, p=0.6):
    rng = np.random.default_rng(seed)
    lat = rng.integers(0, T, size=(C, H, W)).astype(np.uint8)
    lat[rng.random(lat.shape) >= p] = NS
    w = rng.random((F, C, K, K)).astype(np.float32)
    return lat, w


def test_fig2_worked_example(orc):
    lat_in, P_exp, theta, lat_exp, v_exp = read_golden("fig2_conv_fire.txt")
    w = np.ones((1, 1, 3, 3), np.float32)
    P = orc.potentials(lat_in.astype(np.uint8), w, 0, 3)
    assert P.shape == (3, 1, 3, 3)                          # Eq. 2: 5 - 3 + 1 = 3
    assert np.array_equal(P, P_exp)
    lat, v = orc.fire(P, theta)
    assert np.array_equal(lat, lat_exp.astype(np.uint8))
    assert np.array_equal(v, v_exp.astype(np.float32))


@pytest.mark.parametrize("seed,pad", [(0, 0), (1, 1), (2, 2), (3, 0)])
def test_potentials_vs_torch_conv2d(orc, seed, pad):
    """Library cross-check (PyTorch conv2d with time as the batch dim) in float64 on the
    materialised wave S[t] (Eq. 1) with zero padding (R6)."""
    lat, w = _rand_case(seed)
    T = 6
    P = orc.potentials(lat, w, pad, T)
    S = torch.from_numpy(orc.expand(lat[None], T)[0]).double()          # [T, C, H, W]
    ref = torch.nn.functional.conv2d(S, torch.from_numpy(w).double(), padding=pad).numpy()
    assert P.shape == ref.shape
    np.testing.assert_allclose(P, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_potentials_vs_bruteforce(orc, seed):
    lat, w = _rand_case(seed, C=2, H=6, W=5, F=3, K=3, T=5)
    for pad in (0, 1, 2):
        a = orc.potentials(lat, w, pad, 5)
        b = orc.potentials(lat, w, pad, 5, brute=True)
        assert np.array_equal(a, b)


def test_potentials_exact_rational(orc):
    """fp64 accumulation is exact for fp32 weights >= 2^-17 (N1): compare with Fractions."""
    lat, w = _rand_case(11, C=2, H=4, W=4, F=2, K=3, T=4)
    w = np.maximum(w, np.float32(2 ** -8))
    P = orc.potentials(lat, w, 1, 4)
    for t in range(4):
        for f in range(2):
            for y in range(4):
                for x in range(4):
                    s = Fraction(0)
                    for c in range(2):
                        for ky in range(3):
                            for kx in range(3):
                                yy, xx = y + ky - 1, x + kx - 1
                                if 0 <= yy < 4 and 0 <= xx < 4 and lat[c, yy, xx] != NS and lat[c, yy, xx] <= t:
                                    s += Fraction(float(w[f, c, ky, kx]))
                    assert Fraction(P[t, f, y, x]) == s


def test_shape_eq2(orc):
    rng = np.random.default_rng(5)
    for _ in range(50):
        H, W = rng.integers(3, 12, size=2)
        KH, KW = rng.integers(1, 4, size=2)
        pad = int(rng.integers(0, 3))
        lat = np.full((1, H, W), NS, np.uint8)
        w = np.ones((1, 1, KH, KW), np.float32)
        P = orc.potentials(lat, w, pad, 2)
        assert P.shape == (2, 1, H + 2 * pad - KH + 1, W + 2 * pad - KW + 1)


def test_potentials_monotone_nonneg_weights(orc):
    lat, w = _rand_case(9)
    P = orc.potentials(lat, w, 1, 6)
    assert np.all(np.diff(P, axis=0) >= 0)


def test_fire_strict_threshold_and_first_spike(orc):
    P = np.array([[0.0], [1.0], [2.0], [2.0], [5.0]])     # [T=5, n=1]
    lat, v = orc.fire(P, 2.0)                              # P = 2 is not > 2 (R3)
    assert lat.tolist() == [4] and v.tolist() == [5.0]
    lat, v = orc.fire(P, 1.5)
    assert lat.tolist() == [2] and v.tolist() == [2.0]
    lat, v = orc.fire(P, 7.0)
    assert lat.tolist() == [NS] and v.tolist() == [0.0]


def test_fire_infinite_threshold_eq5(orc):
    # Eq. 5: only the last step survives; spike at T-1 iff P[T-1] > 0
    P = np.array([[0.0, 1.0, 0.0], [0.0, 2.0, 0.0], [3.5, 2.0, 0.0]])
    lat, v = orc.fire(P, math.inf)
    assert lat.tolist() == [2, 2, NS]
    assert v.tolist() == [3.5, 2.0, 0.0]


def test_fire_wave_invariants(orc):
    # <= 1 spike per neuron and the output wave is monotone in t (Eq. 1)
    lat_in, w = _rand_case(21, F=5)
    P = orc.potentials(lat_in, w, 1, 6)
    lat, v = orc.fire(P, 2.0)
    S = orc.expand(lat[None], 6)[0]
    assert np.all(np.diff(S, axis=0) >= 0)
    thr = np.where(P > 2.0, P, 0.0)                        # sf.threshold
    first = np.argmax(thr > 0, axis=0)
    spk = (thr > 0).any(axis=0)
    assert np.array_equal(np.where(spk, first, NS), lat)
    assert np.array_equal(v, np.where(spk, np.take_along_axis(P, first[None], 0)[0], 0).astype(np.float32))


@pytest.mark.parametrize("theta", [2.5, math.inf])
def test_conv_fire_batch_and_sample_agree(orc, theta):
    rng = np.random.default_rng(4)
    lat = rng.integers(0, 6, size=(3, 3, 7, 6)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.4] = NS
    w = rng.random((4, 3, 3, 3)).astype(np.float32)
    L, V = orc.conv_fire(lat, w, 1, 6, theta)
    for b in range(3):
        P = orc.potentials(lat[b], w, 1, 6)
        l2, v2 = orc.fire(P, theta)
        assert np.array_equal(L[b], l2) and np.array_equal(V[b], v2)
    idx = rng.choice(L.size, 40, replace=False)
    ls, vs = orc.conv_fire_sample(lat, w, 1, 6, theta, idx)
    assert np.array_equal(ls, L.ravel()[idx]) and np.array_equal(vs, V.ravel()[idx])


def test_events_count(orc):
    lat, w = _rand_case(2)
    n = orc.events(lat[None], F=4, KH=3, KW=3, pad=1)
    S = torch.from_numpy((lat != NS).astype(np.float64))[None]
    ones = torch.ones(1, 3, 3, 3, dtype=torch.float64)
    assert n == 4 * int(torch.nn.functional.conv2d(S, ones, padding=1).sum())
