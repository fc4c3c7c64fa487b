"""Walk statistics of one conv layer (numpy model of conv_walk's schedule, for design only).
For every position and feature group: list length, entries walked until all features fired, and
how many 8-entry blocks the FAST test would push into SLOW mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

def stats(lat_in, w, pad, T, theta, FGS, npos_max=20000, seed=0, blk=8):
    B, C, H, W = lat_in.shape
    F, _, K, _ = w.shape
    Ho, Wo = H + 2 * pad - K + 1, W + 2 * pad - K + 1
    lp = np.full((B, C, H + 2 * pad, W + 2 * pad), 255, np.uint8)
    lp[:, :, pad:pad + H, pad:pad + W] = lat_in
    wq = (w.reshape(F, -1).astype(np.float64) * 2.0 ** 31).astype(np.int64)
    thr = int(np.floor(theta * 2.0 ** 31))
    rng = np.random.default_rng(seed)
    allpos = [(b, y, x) for b in range(B) for y in range(Ho) for x in range(Wo)]
    sel = rng.choice(len(allpos), size=min(npos_max, len(allpos)), replace=False)
    tot_list = walked = necessary = fast_blocks = slow_blocks = 0
    ngroups = (F + FGS - 1) // FGS
    for si in sel:
        b, y, x = allpos[si]
        rf = lp[b, :, y:y + K, x:x + K].reshape(-1)
        idx = np.nonzero(rf < T)[0]
        order = idx[np.argsort(rf[idx], kind="stable")]
        lats = rf[order]
        n = len(order)
        tot_list += n
        if n == 0:
            continue
        ends = np.nonzero(np.r_[lats[1:] != lats[:-1], True])[0] + 1   # bucket end (exclusive index)
        P = np.cumsum(wq[:, order], axis=1)                              # [F, n]
        for g in range(ngroups):
            Pg = P[g * FGS:(g + 1) * FGS]
            # x_f: first entry where prefix > thr; e_f: the bucket end at or after x_f
            over = Pg > thr
            fires = over.any(axis=1)
            x = np.where(fires, over.argmax(axis=1) + 1, n + 1)
            e = ends[np.minimum(np.searchsorted(ends, x), len(ends) - 1)]
            e = np.where(fires, e, n)
            necessary += int(e.sum())
            wend = n if not fires.all() else int(e.max())
            nb = (wend + blk - 1) // blk
            walked += nb * blk
            slow = np.zeros(nb, bool)
            for xf, ef in zip(x[fires], e[fires]):
                slow[(xf - 1) // blk:min(nb, (ef - 1) // blk + 1)] = True
            slow_blocks += int(slow.sum()); fast_blocks += int((~slow).sum())
    npos = len(sel)
    print(f"positions {npos}  groups {ngroups}  mean list {tot_list/npos:.1f}  walked/group {walked/npos/ngroups:.1f} "
          f" necessary/feature {necessary/npos/F:.1f}  blocks/group {(fast_blocks+slow_blocks)/npos/ngroups:.2f} "
          f"slow frac {slow_blocks/max(1,fast_blocks+slow_blocks):.2f}")

if __name__ == "__main__":
    import synth, oracle
    from oracle import flows
    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if which == "c2":
        wl = synth.C2(n=40)
        r = flows.c2(wl)
        print("C2 conv1:"); stats(r["lat0"], wl.weights[0], 2, 15, 15.0, 32, 4000)
        print("C2 conv2:"); stats(r["l1"]["pool_lat"], wl.weights[1], 1, 15, 10.0, 128, 3000)
    else:
        wl = synth.C5(n=1)
        lat0 = oracle.encode(wl.X[:1], 32)
        print("C5 conv1:"); stats(lat0, wl.weights[0], 2, 32, 40.0, 64, 300)
