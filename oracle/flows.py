"""Per-config compositions of the oracle steps -- TEST INFRASTRUCTURE ONLY.

Each flow strings the oracle's step functions together in the order the config
(BASELINE.json "configs") and the paper's tutorial forward pass
 prescribe.  No arithmetic of its own beyond
calling ``oracle`` functions.
"""
from __future__ import annotations

import math
from typing import Dict, List

import numpy as np

from . import conv_fire, decide, encode, filter_bank, inhibit, k_winners, pool, stdp


def layer(lat_in, w, spec, T, pool_spec=None):
    lat, v = conv_fire(lat_in, w, spec.pad, T, spec.theta)
    out = {"lat": lat, "v": v}
    if pool_spec is not None:
        pl, pv = pool(lat, v, pool_spec.PH, pool_spec.PW, pool_spec.SH, pool_spec.SW,
                      pool_spec.DH, pool_spec.DW, T)
        out["pool_lat"], out["pool_v"] = pl, pv
    return out


def c1(wl) -> Dict[str, np.ndarray]:
    """encode -> conv+fire -> pointwise inhibition -> kWTA(k5, r3) -> one STDP step."""
    T = wl.T
    lat0 = encode(wl.X, T)
    spec = wl.convs[0]
    l1 = layer(lat0, wl.weights[0], spec, T)
    il, iv, wf = inhibit(l1["lat"], l1["v"])
    win, cnt = k_winners(il, iv, wl.extra["k"], wl.extra["r"])
    s = wl.extra["stdp"]
    w_new = stdp(wl.weights[0], lat0[0], spec.pad, l1["lat"][0], win[0], cnt[0],
                 s["a_plus"], s["a_minus"], s["lb"], s["ub"], s["stabilizer"], 1)
    return dict(lat0=lat0, lat1=l1["lat"], v1=l1["v"], inh_lat=il, inh_v=iv, winner_f=wf,
                winners=win, count=cnt, w_new=w_new)


def c2(wl, n: int = None, front: bool = False) -> Dict[str, np.ndarray]:
    """3-layer inference: encode -> [conv+fire -> pool] x2 -> conv (theta=inf) -> 1 winner -> class.
    front=True starts from the raw images (extra["raw"]) through the f2 filter bank (R33) instead of X."""
    X = wl.X if n is None else wl.X[:n]
    if front:
        fr = wl.extra["front"]
        raw = wl.extra["raw"] if n is None else wl.extra["raw"][:n]
        X = filter_bank(raw, wl.extra["bank"], fr["pad"], mode=fr["mode"])
    T = wl.T
    lat0 = encode(X, T)
    l1 = layer(lat0, wl.weights[0], wl.convs[0], T, wl.pools[0])
    l2 = layer(l1["pool_lat"], wl.weights[1], wl.convs[1], T, wl.pools[1])
    l3 = layer(l2["pool_lat"], wl.weights[2], wl.convs[2], T)
    win, cnt = k_winners(l3["lat"], l3["v"], 1, 0)
    F3 = wl.convs[2].F
    ncls = wl.extra["n_classes"]
    cls = np.where(cnt > 0, win[:, 0, 0] // (F3 // ncls), -1).astype(np.int32)
    return dict(lat0=lat0, l1=l1, l2=l2, l3=l3, winners=win, count=cnt, decision=cls)


def c3(wl, n: int = None, snapshot_every: int = None) -> Dict[str, object]:
    """Sequential L2 STDP: per image conv+fire -> inhibit -> kWTA(k8, r2) -> STDP on W2."""
    X = wl.X if n is None else wl.X[:n]
    T = wl.T
    lat0 = encode(X, T)
    l1 = layer(lat0, wl.weights[0], wl.convs[0], T, wl.pools[0])
    lat_in = l1["pool_lat"]
    spec = wl.convs[1]
    w2 = wl.weights[1].copy()
    s = wl.extra["stdp"]
    every = snapshot_every or wl.extra.get("snapshot_every", 500)
    snaps: List[np.ndarray] = []
    winners, counts = [], []
    for b in range(X.shape[0]):
        lat, v = conv_fire(lat_in[b:b + 1], w2, spec.pad, T, spec.theta)
        il, iv, _ = inhibit(lat, v)
        win, cnt = k_winners(il, iv, wl.extra["k"], wl.extra["r"])
        w2 = stdp(w2, lat_in[b], spec.pad, lat[0], win[0], cnt[0], s["a_plus"], s["a_minus"],
                  s["lb"], s["ub"], s["stabilizer"], 1)
        winners.append(win[0]); counts.append(cnt[0])
        if (b + 1) % every == 0:
            snaps.append(w2.copy())
    return dict(w2=w2, snapshots=snaps, winners=np.array(winners), count=np.array(counts),
                l1_pool_lat=lat_in)


def c4(wl, n: int = None) -> Dict[str, object]:
    """R-STDP: L1 conv+fire -> pool 7/6 (batched); per image L2 conv (theta=inf) -> 1 winner
    -> decision vs seeded label -> reward (+1) / punish (-1) / silent (0) on W2."""
    X = wl.X if n is None else wl.X[:n]
    T = wl.T
    labels = wl.extra["labels"]
    lat0 = encode(X, T)
    l1 = layer(lat0, wl.weights[0], wl.convs[0], T, wl.pools[0])
    lat_in = l1["pool_lat"]
    spec = wl.convs[1]
    w2 = wl.weights[1].copy()
    s = wl.extra["stdp"]
    F2 = spec.F
    decisions, rewards, winners = [], [], []
    for b in range(X.shape[0]):
        lat, v = conv_fire(lat_in[b:b + 1], w2, spec.pad, T, spec.theta)
        win, cnt = k_winners(lat, v, 1, 0)
        d, rw = decide(win[0], cnt[0], F2, wl.extra["n_classes"], int(labels[b]))
        w2 = stdp(w2, lat_in[b], spec.pad, lat[0], win[0], cnt[0], s["a_plus"], s["a_minus"],
                  s["lb"], s["ub"], s["stabilizer"], rw)
        decisions.append(d); rewards.append(rw); winners.append(win[0])
    return dict(w2=w2, decision=np.array(decisions), reward=np.array(rewards),
                winners=np.array(winners), l1_pool_lat=lat_in)


def c5(wl, n: int = None) -> Dict[str, np.ndarray]:
    """encode -> conv+fire -> pool 2/2 -> pointwise inhibition -> kWTA(k16, r4) (reading A16)."""
    X = wl.X if n is None else wl.X[:n]
    T = wl.T
    lat0 = encode(X, T)
    l1 = layer(lat0, wl.weights[0], wl.convs[0], T, wl.pools[0])
    il, iv, wf = inhibit(l1["pool_lat"], l1["pool_v"])
    win, cnt = k_winners(il, iv, wl.extra["k"], wl.extra["r"])
    return dict(lat0=lat0, l1=l1, inh_lat=il, inh_v=iv, winner_f=wf, winners=win, count=cnt)
