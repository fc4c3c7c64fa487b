"""Pins for oracle a1 (intensity -> latency) and Eq. 1 (expand).  CPU only."""
import numpy as np
import pytest

from conftest import read_golden

NS = 255


def _check_rank_bins(x_img, lat_img, T):
    """Invariants that together fix the encoding (reading R1): positives spike, non-positives do
    not; bin t holds q+1 (t < m) or q entries; values never increase across bins; equal values in
    different bins are ordered by flat index."""
    x = x_img.ravel().astype(np.float64)
    lat = lat_img.ravel()
    pos = x > 0
    assert np.all(lat[~pos] == NS)
    assert np.all(lat[pos] < T)
    N = int(pos.sum())
    q, m = divmod(N, T)
    counts = np.bincount(lat[pos], minlength=T)
    assert counts.tolist() == [q + 1 if t < m else q for t in range(T)]
    # ordering: for every pair of bins t < u, min value of t >= max value of u, and ties by index
    for t in range(T - 1):
        a, b = np.where(lat == t)[0], np.where(lat == t + 1)[0]
        if a.size == 0 or b.size == 0:
            continue
        assert x[a].min() >= x[b].max()
        if x[a].min() == x[b].max():
            v = x[a].min()
            assert a[x[a] == v].max() < b[x[b] == v].min()


def test_spec_worked_example(orc):
    # intensities (9, 7, 5, 1), t_max = 4 -> latencies (0, 1, 2, 3)
    lat = orc.encode(np.array([[9, 7, 5, 1]], np.float32), 4)
    assert lat.tolist() == [[0, 1, 2, 3]]


def test_all_zero_never_spikes(orc):
    # SPEC.md:192, reading R2 (x <= 0 never spikes); also negative and NaN
    x = np.zeros((2, 3, 4, 4), np.float32)
    x[1, 0, 0, 0] = -1.0
    x[1, 0, 0, 1] = np.nan
    assert np.all(orc.encode(x, 7) == NS)


def test_fewer_spikes_than_bins(orc):
    # N < T: the first N bins hold one spike each (R1)
    x = np.array([[0.1, 0.0, 0.7, 0.3]], np.float32)
    assert orc.encode(x, 10).tolist() == [[2, NS, 0, 1]]


def test_permutation_equivariance(orc):
    # permuting the layout permutes latencies identically (distinct values)
    rng = np.random.default_rng(0)
    x = rng.permutation(np.arange(1, 201, dtype=np.float32))[None]
    perm = rng.permutation(200)
    a = orc.encode(x, 9)[0]
    b = orc.encode(x[:, perm], 9)[0]
    assert np.array_equal(a[perm], b)


def test_ties_by_flat_index(orc):
    x = np.full((1, 12), 0.5, np.float32)
    lat = orc.encode(x, 4)[0]
    assert lat.tolist() == [0, 0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3]


@pytest.mark.parametrize("seed,T", [(1, 15), (2, 32), (3, 1), (4, 254), (5, 7)])
def test_invariants_random(orc, seed, T):
    rng = np.random.default_rng(seed)
    x = rng.random((3, 4, 9, 7)).astype(np.float32)
    x[rng.random(x.shape) < 0.4] = 0
    x[0, 0, :3] = 0.25       # tie groups
    lat = orc.encode(x, T)
    for b in range(3):
        _check_rank_bins(x[b], lat[b], T)


def test_monotone_against_library_sort(orc):
    """Rank order agrees with numpy's stable lexsort (library routine): the element of rank r
    lies in the bin that contains r."""
    rng = np.random.default_rng(7)
    x = (rng.integers(0, 20, size=(1, 500)) / 19).astype(np.float32)   # many ties
    T = 13
    lat = orc.encode(x, T)[0]
    order = np.lexsort((np.arange(500), -x[0].astype(np.float64)))
    order = order[x[0][order] > 0]
    N = order.size
    q, m = divmod(N, T)
    bins = np.concatenate([np.full(q + (t < m), t) for t in range(T)])
    assert np.array_equal(lat[order], bins)


def test_c1_closed_form(orc):
    """C1 (configs[0]): every pixel gives exactly one positive channel, so N = 784 and the bins
    are 4 x 53 + 11 x 52; the zeroed pixels all have off = 0.5, the unique maximum, so they fill
    ranks 0..n_tie-1 in pixel row-major order (reading A27)."""
    import synth
    wl = synth.C1()
    X = wl.X
    lat = orc.encode(X, 15)[0]
    assert int((X > 0).sum()) == 784
    counts = np.bincount(lat[lat != NS], minlength=15)
    assert counts.tolist() == [53] * 4 + [52] * 11
    off = X[0, 1].ravel()
    tied = np.where(off == np.float32(0.5))[0]
    assert X.max() == np.float32(0.5) and tied.size > 400
    sizes = [53] * 4 + [52] * 11
    start = np.cumsum([0] + sizes)
    expect = np.searchsorted(start, np.arange(tied.size), side="right") - 1
    assert np.array_equal(lat[1].ravel()[tied], expect)


def test_fig1_expand(orc):
    lat, wave = read_golden("fig1_expand.txt")
    got = orc.expand(lat.astype(np.uint8)[None], 4)[0]
    assert got.shape == (4, 3, 2, 2)
    assert np.array_equal(got, wave)


def test_expand_invariants(orc):
    # S:85 sum over t of S = T - lat for spiking neurons, 0 otherwise; monotone in t
    rng = np.random.default_rng(3)
    lat = rng.integers(0, 9, size=(2, 5, 6, 6)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.3] = NS
    w = orc.expand(lat, 9)
    s = w.sum(axis=1)
    assert np.array_equal(s, np.where(lat == NS, 0, 9 - lat.astype(int)))
    assert np.all(np.diff(w, axis=1) >= 0)
