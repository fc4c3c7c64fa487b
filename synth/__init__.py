"""Seeded synthetic workloads for the five BASELINE.json configs (C1..C5).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic (no encoding, convolution, firing,
pooling, inhibition, k-WTA or STDP).  It only draws the inputs the method
consumes:

* fp32 intensity maps X[B, C, H, W] (the input of step a1, "encode");
* fp32 synaptic weights W[F, C, KH, KW] ~ N(mu, sigma) clamped to [0, 1]
  ("randomly initialized using a normal distribution");
* seeded labels for the R-STDP config (C4).

The image-like configs are stand-ins for the paper's MNIST / Caltech inputs
(PAPER.md:148, :278): same shapes and value ranges, generated from seeded
strokes (C2/C3) and shapes (C4).  Their pre-processing (DoG / Gabor filter
banks) lives here because it is part of the workload
generator, not the hot path.  The filter
formulas are the standard definitions, chosen by this repo
(DESIGN.md "Input recipe").

Seeds: data seed 1000+i and weight seed 2000+i for config Ci.
Per-image streams come from ``SeedSequence(seed).spawn(B)``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

__all__ = [
    "ConvSpec", "PoolSpec", "Workload", "make", "CONFIG_NAMES",
    "init_weights", "stroke_images", "shape_images", "dog_bank", "gabor_bank",
    "filter_bank", "C1", "C2", "C3", "C4", "C5",
]

CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")


@dataclasses.dataclass(frozen=True)
class ConvSpec:
    F: int
    C: int
    KH: int
    KW: int
    pad: int
    theta: float          # math.inf => Eq. 5 infinite threshold


@dataclasses.dataclass(frozen=True)
class PoolSpec:
    PH: int
    PW: int
    SH: int
    SW: int
    DH: int = 0
    DW: int = 0


@dataclasses.dataclass
class Workload:
    name: str
    T: int
    X: np.ndarray                         # fp32 [B, C, H, W] intensities
    convs: List[ConvSpec]
    weights: List[np.ndarray]             # fp32 [F, C, KH, KW] per conv layer
    pools: List[Optional[PoolSpec]]       # pool after each conv (None = none)
    extra: Dict[str, object]              # k, r, learning rates, labels, ...


# ---------------------------------------------------------------------------
# weights
# ---------------------------------------------------------------------------

def init_weights(rng: np.random.Generator, shape, mu: float, sigma: float) -> np.ndarray:
    """N(mu, sigma) drawn in fp64, cast to fp32, clamped to [0, 1] (A31)."""
    w = rng.normal(mu, sigma, size=shape).astype(np.float32)
    return np.clip(w, np.float32(0.0), np.float32(1.0)).astype(np.float32)


# ---------------------------------------------------------------------------
# filter banks (workload pre-processing; standard definitions)
# ---------------------------------------------------------------------------

def _normalize_kernel(k: np.ndarray) -> np.ndarray:
    k = k - k.mean()
    m = np.abs(k).max()
    return k / m if m > 0 else k


def dog_bank(size: int = 7, pairs=((0.5, 1.0), (1.0, 2.0), (1.5, 3.0))) -> np.ndarray:
    r = size // 2
    yy, xx = np.mgrid[-r:r + 1, -r:r + 1].astype(np.float64)
    d2 = xx * xx + yy * yy
    ks = []
    for s1, s2 in pairs:
        k = (1.0 / (2 * math.pi)) * (np.exp(-d2 / (2 * s1 * s1)) / (s1 * s1)
                                      - np.exp(-d2 / (2 * s2 * s2)) / (s2 * s2))
        ks.append(_normalize_kernel(k))
    return np.stack(ks)


def gabor_bank(size: int = 5, lam: float = 5.0, sigma: float = 2.0, gamma: float = 0.5,
               thetas_deg=(0.0, 45.0, 90.0, 135.0)) -> np.ndarray:
    r = size // 2
    yy, xx = np.mgrid[-r:r + 1, -r:r + 1].astype(np.float64)
    ks = []
    for th in thetas_deg:
        t = math.radians(th)
        xp = xx * math.cos(t) + yy * math.sin(t)
        yp = -xx * math.sin(t) + yy * math.cos(t)
        k = np.exp(-(xp * xp + gamma * gamma * yp * yp) / (2 * sigma * sigma)) * np.cos(2 * math.pi * xp / lam)
        ks.append(_normalize_kernel(k))
    return np.stack(ks)


def filter_bank(img: np.ndarray, bank: np.ndarray, pad: int) -> np.ndarray:
    """Same-size zero-padded cross-correlation of [N,H,W] images with [K,s,s] kernels -> [N,K,H,W] fp64."""
    n, h, w = img.shape
    k, s, _ = bank.shape
    p = np.pad(img, ((0, 0), (pad, pad), (pad, pad)))
    out = np.zeros((n, k, h + 2 * pad - s + 1, w + 2 * pad - s + 1))
    for dy in range(s):
        for dx in range(s):
            win = p[:, dy:dy + out.shape[2], dx:dx + out.shape[3]]
            out += win[:, None] * bank[None, :, dy, dx, None, None]
    return out


def _gauss_blur(img: np.ndarray, sigma: float = 1.0, radius: int = 3) -> np.ndarray:
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-x * x / (2 * sigma * sigma))
    g /= g.sum()
    k = np.outer(g, g)[None]
    return filter_bank(img, k, radius)[:, 0]


# ---------------------------------------------------------------------------
# images
# ---------------------------------------------------------------------------

def stroke_images(seed: int, n: int, size: int = 28) -> np.ndarray:
    """3-6 line segments of width 2, intensity 1, Gaussian blur sigma 1 (BASELINE.json configs[1])."""
    children = np.random.SeedSequence(seed).spawn(n)
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    imgs = np.zeros((n, size, size))
    for i, ss in enumerate(children):
        rng = np.random.default_rng(ss)
        nseg = int(rng.integers(3, 7))
        im = np.zeros((size, size))
        for _ in range(nseg):
            (y0, x0), (y1, x1) = rng.uniform(3, 25, size=(2, 2))
            dy, dx = y1 - y0, x1 - x0
            L2 = dy * dy + dx * dx
            tt = np.clip(((yy - y0) * dy + (xx - x0) * dx) / L2, 0, 1) if L2 > 0 else np.zeros_like(yy)
            d = np.hypot(yy - (y0 + tt * dy), xx - (x0 + tt * dx))
            im[d <= 1.0] = 1.0
        imgs[i] = im
    return _gauss_blur(imgs)


def shape_images(seed: int, n: int, h: int = 160, w: int = 250) -> np.ndarray:
    """2-8 ellipses / rectangles, intensity U(0.3,1), + N(0,0.05) noise, clipped (configs[3])."""
    children = np.random.SeedSequence(seed).spawn(n)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    imgs = np.zeros((n, h, w))
    for i, ss in enumerate(children):
        rng = np.random.default_rng(ss)
        im = np.zeros((h, w))
        for _ in range(int(rng.integers(2, 9))):
            ell = rng.random() < 0.5
            cy, cx = rng.uniform(0, h), rng.uniform(0, w)
            ay, ax = rng.uniform(5, 40, size=2)
            inten = rng.uniform(0.3, 1.0)
            if ell:
                m = ((yy - cy) / ay) ** 2 + ((xx - cx) / ax) ** 2 <= 1.0
            else:
                m = (np.abs(yy - cy) <= ay) & (np.abs(xx - cx) <= ax)
            im[m] = inten
        im += rng.normal(0.0, 0.05, size=(h, w))
        imgs[i] = np.clip(im, 0.0, 1.0)
    return imgs


def _dog_input(seed: int, n: int) -> np.ndarray:
    imgs = stroke_images(seed, n)
    r = filter_bank(imgs, dog_bank(), 3)                    # [n, 3, 28, 28]
    on, off = np.maximum(r, 0), np.maximum(-r, 0)
    X = np.stack([on, off], axis=2).reshape(n, 6, 28, 28)   # [on1, off1, on2, off2, on3, off3]
    return X.astype(np.float32)


# ---------------------------------------------------------------------------
# the five configs (BASELINE.json "configs")
# ---------------------------------------------------------------------------

STDP_RATES = dict(a_plus=0.004, a_minus=-0.003, lb=0.0, ub=1.0, stabilizer=1)


def C1() -> Workload:
    rng = np.random.default_rng(1001)
    x = rng.random((28, 28), dtype=np.float32)
    x[rng.random((28, 28)) < 0.7] = 0.0
    half = np.float32(0.5)
    on = np.maximum(x - half, np.float32(0))
    off = np.maximum(half - x, np.float32(0))
    X = np.stack([on, off])[None].astype(np.float32)        # [1, 2, 28, 28]
    W = init_weights(np.random.default_rng(2001), (30, 2, 5, 5), 0.8, 0.05)
    return Workload("c1", 15, X, [ConvSpec(30, 2, 5, 5, 2, 15.0)], [W], [None],
                    dict(k=5, r=3, inhibit=True, stdp=dict(STDP_RATES)))


def _c2_weights():
    rng = np.random.default_rng(2002)
    return [init_weights(rng, (30, 6, 5, 5), 0.8, 0.05),
            init_weights(rng, (250, 30, 3, 3), 0.8, 0.05),
            init_weights(rng, (200, 250, 5, 5), 0.8, 0.05)]


def C2(n: int = 1000) -> Workload:
    X = _dog_input(1002, n)
    raw = stroke_images(1002, n)                            # the images X was filtered from (f2 front end)
    return Workload("c2", 15, X,
                    [ConvSpec(30, 6, 5, 5, 2, 15.0), ConvSpec(250, 30, 3, 3, 1, 10.0),
                     ConvSpec(200, 250, 5, 5, 2, math.inf)],
                    _c2_weights(),
                    [PoolSpec(2, 2, 2, 2), PoolSpec(3, 3, 3, 3), None],
                    dict(k=1, r=0, n_classes=10, raw=raw, bank=dog_bank(), front=dict(pad=3, mode=1)))


def C3(n: int = 2000) -> Workload:
    X = _dog_input(1003, n)
    w = _c2_weights()
    return Workload("c3", 15, X,
                    [ConvSpec(30, 6, 5, 5, 2, 15.0), ConvSpec(250, 30, 3, 3, 1, 10.0)],
                    w[:2], [PoolSpec(2, 2, 2, 2), None],
                    dict(k=8, r=2, inhibit=True, stdp=dict(STDP_RATES), snapshot_every=500))


def C4(n: int = 1000) -> Workload:
    imgs = shape_images(1004, n)
    r = filter_bank(imgs, gabor_bank(), 2)
    X = np.maximum(r, 0).astype(np.float32)                  # [n, 4, 160, 250]
    rng = np.random.default_rng(2004)
    W1 = init_weights(rng, (20, 4, 5, 5), 0.8, 0.05)
    W2 = init_weights(rng, (100, 20, 17, 17), 0.8, 0.05)
    labels = np.random.default_rng(np.random.SeedSequence(1004).spawn(n + 1)[n]).integers(0, 2, size=n).astype(np.int32)
    return Workload("c4", 30, X,
                    [ConvSpec(20, 4, 5, 5, 0, 15.0), ConvSpec(100, 20, 17, 17, 0, math.inf)],
                    [W1, W2], [PoolSpec(7, 7, 6, 6), None],
                    dict(k=1, r=0, n_classes=2, labels=labels, stdp=dict(STDP_RATES)))


def C5(n: int = 64) -> Workload:
    X = np.empty((n, 32, 256, 256), dtype=np.float32)
    for i, ss in enumerate(np.random.SeedSequence(1005).spawn(n)):
        rng = np.random.default_rng(ss)
        x = rng.random((32, 256, 256), dtype=np.float32)
        x[rng.random((32, 256, 256)) < 0.5] = 0.0
        X[i] = x
    W = init_weights(np.random.default_rng(2005), (256, 32, 5, 5), 0.5, 0.1)
    return Workload("c5", 32, X, [ConvSpec(256, 32, 5, 5, 2, 40.0)], [W], [PoolSpec(2, 2, 2, 2)],
                    dict(k=16, r=4, inhibit=True))


def make(name: str, **kw) -> Workload:
    return {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c5": C5}[name.lower()](**kw)


# ---------------------------------------------------------------------------
# generic seeded random inputs for fuzz / parity tests
# ---------------------------------------------------------------------------

def random_latencies(rng: np.random.Generator, shape, T: int, p_spike: float = 0.6) -> np.ndarray:
    """uint8 latency grid: each neuron spikes with prob p_spike at U{0..T-1}, else 255 (NO_SPIKE)."""
    lat = rng.integers(0, T, size=shape).astype(np.uint8)
    lat[rng.random(shape) >= p_spike] = 255
    return lat


def random_potentials_at_spike(rng: np.random.Generator, lat: np.ndarray, n_levels: int = 0) -> np.ndarray:
    """fp32 'v' values for a latency grid (0 where NO_SPIKE).  n_levels>0 draws from a few levels to force ties."""
    if n_levels > 0:
        v = (rng.integers(1, n_levels + 1, size=lat.shape) / n_levels).astype(np.float32)
    else:
        v = rng.uniform(0.01, 50.0, size=lat.shape).astype(np.float32)
    v[lat == 255] = 0.0
    return v
