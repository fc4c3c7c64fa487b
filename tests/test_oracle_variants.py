"""Pins of the f3 variant paths of the oracle (R36-R39): the encoding
bin-size alternatives (A4), Eq. 3's literal pooling size (A10), pooled final potentials (A13) and the
stabilized no-clamp STDP (A20).  Each is checked against an independent brute-force definition."""
import numpy as np
import pytest

import oracle

NS = 255


def _ranks(x):
    """Rank of every positive entry by (value desc, flat index asc), via numpy lexsort (library)."""
    flat = x.reshape(-1)
    pos = np.flatnonzero(flat > 0)
    order = pos[np.lexsort((pos, -flat[pos].astype(np.float64)))]
    r = np.full(flat.shape, -1, np.int64)
    r[order] = np.arange(order.size)
    return r, order.size


@pytest.mark.parametrize("n,T,zero", [(100, 15, 0.3), (7, 15, 0.0), (784, 30, 0.5), (45, 9, 0.9)])
def test_encode_bins_variants(n, T, zero):
    rng = np.random.default_rng(n + T)
    x = rng.random((3, n)).astype(np.float32)
    x[rng.random((3, n)) < zero] = 0.0
    x[:, ::5] = np.float32(0.5)            # ties broken by index
    for b in range(3):
        r, N = _ranks(x[b])
        prop = np.where(r >= 0, (r * T) // max(N, 1), NS)
        q = N // T
        flo = np.where((r >= 0) & (r < T * q), r // max(q, 1), NS)
        assert np.array_equal(oracle.encode(x[b:b + 1], T, bins=1)[0], prop.astype(np.uint8))
        assert np.array_equal(oracle.encode(x[b:b + 1], T, bins=2)[0], flo.astype(np.uint8))
    # N < T: proportional spreads the N entries over distinct bins; floor spikes nothing
    few = np.zeros((1, 50), np.float32)
    few[0, [3, 9, 20]] = [0.2, 0.9, 0.5]
    assert list(oracle.encode(few, 10, bins=1)[0, [9, 20, 3]]) == [0, 3, 6]
    assert (oracle.encode(few, 10, bins=2) == NS).all()


def _pool_brute(lat, v, P, S, D, eq3, vfinal):
    B, F, H, W = lat.shape
    Ho, Wo = ((H + 2 * D) // S, (W + 2 * D) // S) if eq3 else ((H + 2 * D - P) // S + 1, (W + 2 * D - P) // S + 1)
    lo = np.full((B, F, Ho, Wo), NS, np.uint8)
    vo = np.zeros((B, F, Ho, Wo), np.float32)
    for b in range(B):
        for f in range(F):
            for oy in range(Ho):
                for ox in range(Wo):
                    ys = slice(max(oy * S - D, 0), max(min(oy * S - D + P, H), 0))
                    xs = slice(max(ox * S - D, 0), max(min(ox * S - D + P, W), 0))
                    wl, wv = lat[b, f, ys, xs].reshape(-1), v[b, f, ys, xs].reshape(-1)
                    sp = wl != NS
                    if not sp.any():
                        continue
                    lo[b, f, oy, ox] = wl[sp].min()
                    sel = sp if vfinal else (wl == wl[sp].min())
                    vo[b, f, oy, ox] = wv[sel].max()
    return lo, vo


@pytest.mark.parametrize("H,W,P,S,D", [(156, 246, 7, 6, 0), (13, 17, 3, 2, 1), (12, 12, 2, 2, 0), (9, 11, 3, 3, 0)])
def test_pool_eq3_and_vfinal(H, W, P, S, D):
    rng = np.random.default_rng(H * W)
    lat = rng.integers(0, 12, (1, 2, H, W)).astype(np.uint8)
    lat[rng.random(lat.shape) < 0.6] = NS
    v = rng.random(lat.shape).astype(np.float32)
    for eq3 in (False, True):
        for vfinal in (False, True):
            lo, vo = oracle.pool(lat, v, P, P, S, S, D, D, T=12, eq3=eq3, vfinal=vfinal)
            blo, bvo = _pool_brute(lat, v, P, S, D, eq3, vfinal)
            assert np.array_equal(lo, blo) and np.array_equal(vo, bvo), (eq3, vfinal)
    if (H, W, P, S) == (156, 246, 7, 6):   # C4's pool: Eq. 3 gives 26 x 41, R10 gives 25 x 40
        assert oracle.pool(lat, v, 7, 7, 6, 6, T=12, eq3=True)[0].shape[2:] == (26, 41)
        assert oracle.pool(lat, v, 7, 7, 6, 6, T=12)[0].shape[2:] == (25, 40)


def test_stdp_stabilized_no_clamp():
    """A20 variant: with the stabilizer on and no clamp, a weight above UB moves by the (negative)
    stabilized step instead of being clamped to UB; inside the bounds it equals the clamped rule."""
    w = np.array([0.9, 0.5, 0.1, 0.79], np.float32).reshape(1, 1, 2, 2)
    lat_in = np.zeros((1, 2, 2), np.uint8)
    lat_out = np.zeros((1, 1, 1), np.uint8)
    win = np.array([[0, 0, 0]], np.int32)
    a = np.float32(0.004)
    nc = oracle.stdp(w, lat_in, 0, lat_out, win, 1, 0.004, -0.003, 0.2, 0.8, stabilizer=2)
    cl = oracle.stdp(w, lat_in, 0, lat_out, win, 1, 0.004, -0.003, 0.2, 0.8, stabilizer=1)
    exp = [np.float32(wi + np.float32(np.float32(a * np.float32(wi - np.float32(0.2))) * np.float32(np.float32(0.8) - wi)))
           for wi in w.reshape(-1)]
    assert np.array_equal(nc.reshape(-1), np.array(exp, np.float32))
    assert nc.reshape(-1)[0] < np.float32(0.9) and nc.reshape(-1)[0] > np.float32(0.8)
    assert cl.reshape(-1)[0] == np.float32(0.8) and cl.reshape(-1)[2] == np.float32(0.2)
    assert nc.reshape(-1)[1] == cl.reshape(-1)[1] and nc.reshape(-1)[3] == cl.reshape(-1)[3]
