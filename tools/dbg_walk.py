"""Debug helper: run every tests/test_gpu_kernels.py CONV_CASES case through the default conv path
and compare with the oracle, printing per case (flushes, so a hang shows where)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
from paper_1903_02440_b200 import snn as G
from test_gpu_kernels import CONV_CASES, exact_weights
sel = [eval(x) if x.startswith('(') else int(x) for x in sys.argv[1:]] or range(len(CONV_CASES))
for ci in sel:
    case = ci if isinstance(ci, tuple) else CONV_CASES[ci]
    B, C, H, W, pad, F, K, T, theta, p = case
    rng = np.random.default_rng(abs(hash(case)) % 2 ** 31)
    lat_in = synth.random_latencies(rng, (B, C, H, W), T, p)
    w = exact_weights(rng, (F, C, K, K)); w[0, 0, 0, 0] = 0.0
    t0 = time.time()
    print("case", ci, case, flush=True)
    lat, v = G.conv_fire(torch.from_numpy(lat_in).cuda(), torch.from_numpy(w).cuda(), pad, T, theta)
    try:
        G.sync_status()
    except Exception as e:
        print("  ERR", e, flush=True)
    ol, ov = oracle.conv_fire(lat_in, w, pad, T, theta)
    l, vv = lat.cpu().numpy(), v.cpu().numpy()
    if (l != ol).any():
        d = np.argwhere(l != ol)
        print("  first diffs (b,f,y,x) gpu/oracle:", [(tuple(x), int(l[tuple(x)]), int(ol[tuple(x)])) for x in d[:8]], flush=True)
        print("  diff count per feature:", np.bincount(d[:, 1], minlength=F).tolist(), flush=True)
    print(f"  lat eq {np.array_equal(l, ol)} ({(l != ol).sum()} diff)  v eq {np.array_equal(vv, ov)} ({(vv != ov).sum()} diff)  {time.time()-t0:.2f}s", flush=True)
