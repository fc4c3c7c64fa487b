"""Pins of the f2 front-end oracle (R33-R35): filter banks,
local normalization and intensity lateral inhibition.  The paper gives intent only; SPEC.md's
examples and independent implementations (numpy, pure-Python sweeps) pin the readings."""
import math

import numpy as np
import pytest

import oracle
import synth


def test_filter_bank_matches_independent_numpy():
    """R33 vs the workload generator's vectorised numpy cross-correlation (an independent code path)."""
    imgs = synth.stroke_images(77, 6)
    dog = oracle.filter_bank(imgs, synth.dog_bank(), 3, mode=1)
    assert np.array_equal(dog, synth._dog_input(77, 6))
    sh = synth.shape_images(78, 2, 40, 50)
    r = synth.filter_bank(sh, synth.gabor_bank(), 2)
    assert np.array_equal(oracle.filter_bank(sh, synth.gabor_bank(), 2, mode=2), np.maximum(r, 0).astype(np.float32))


def test_filter_bank_impulse_zero_threshold_shape():
    ker = np.arange(25, dtype=np.float64).reshape(1, 5, 5) / 7.0 - 1.0
    img = np.zeros((1, 9, 9))
    img[0, 4, 4] = 1.0
    out = oracle.filter_bank(img, ker, 2, mode=0)
    # cross-correlation (no flip, SPEC): output at (4 - dy + 2, 4 - dx + 2) = ker[dy, dx]
    assert np.allclose(out[0, 0, 2:7, 2:7], ker[0, ::-1, ::-1].astype(np.float32))
    assert not oracle.filter_bank(np.zeros((2, 9, 9)), ker, 2).any()
    rng = np.random.default_rng(0)
    t = oracle.filter_bank(rng.random((2, 12, 12)), ker, 2, mode=0, threshold=0.5)
    assert not ((t > 0) & (t < 0.5)).any()
    assert oracle.filter_bank(rng.random((3, 28, 28)), synth.dog_bank(), 3, mode=1).shape == (3, 6, 28, 28)


def _local_norm_brute(x, radius, eps):
    B, C, H, W = x.shape
    out = np.zeros_like(x)
    for b in range(B):
        for c in range(C):
            for y in range(H):
                for xx in range(W):
                    win = x[b, c, max(0, y - radius):y + radius + 1, max(0, xx - radius):xx + radius + 1]
                    m = max(float(np.sum(win.astype(np.float64))) / win.size, eps)
                    out[b, c, y, xx] = np.float32(float(x[b, c, y, xx]) / m)
    return out


def test_local_norm_pins():
    const = np.full((1, 2, 7, 6), 0.7, np.float32)
    assert np.array_equal(oracle.local_norm(const, 2), np.ones_like(const))      # value / own mean
    assert not oracle.local_norm(np.zeros((1, 1, 5, 5), np.float32), 1).any()      # eps guard, 0 / eps
    rng = np.random.default_rng(1)
    x = rng.random((2, 2, 9, 9)).astype(np.float32)
    assert np.allclose(oracle.local_norm(x, 2), _local_norm_brute(x, 2, 1e-12), rtol=1e-6, atol=0)


def _lateral_brute(x, factors):
    """SPEC's sweep, written independently: process in descending original intensity (ties row-major)."""
    B, C, H, W = x.shape
    n = len(factors)
    out = x.copy()
    for b in range(B):
        for c in range(C):
            xc = x[b, c]
            order = sorted(range(H * W), key=lambda i: (-float(xc.flat[i]), i))
            for p in order:
                py, px = divmod(p, W)
                for yy in range(max(0, py - n), min(H, py + n + 1)):
                    for x2 in range(max(0, px - n), min(W, px + n + 1)):
                        if (yy, x2) != (py, px) and xc[yy, x2] < xc[py, px]:
                            d = max(abs(yy - py), abs(x2 - px))
                            out[b, c, yy, x2] = np.float32(out[b, c, yy, x2] * np.float32(factors[d - 1]))
    return out


def test_lateral_inhibition_pins():
    eq = np.full((1, 1, 5, 5), 0.4, np.float32)
    assert np.array_equal(oracle.lateral_inhibition(eq, [0.5, 0.2]), eq)          # nobody strictly stronger
    single = np.zeros((1, 1, 5, 5), np.float32)
    single[0, 0, 2, 2] = 0.9
    assert np.array_equal(oracle.lateral_inhibition(single, [0.5]), single)        # zeros stay zero
    two = np.zeros((1, 1, 1, 2), np.float32)
    two[0, 0, 0, 0], two[0, 0, 0, 1] = 1.0, 0.5
    out = oracle.lateral_inhibition(two, [0.6])
    assert out[0, 0, 0, 0] == np.float32(1.0) and out[0, 0, 0, 1] == np.float32(np.float32(0.5) * np.float32(0.6))
    rng = np.random.default_rng(2)
    x = (rng.integers(0, 6, (2, 2, 7, 8)) / 5.0).astype(np.float32)             # many ties
    assert np.array_equal(oracle.lateral_inhibition(x, [0.5, 0.8]), _lateral_brute(x, [0.5, 0.8]))
