"""Per-image phase timings of snn_rstdp_inf_sequence on C4 (globaltimer stamps, SNN_RSTDP_DBG=8; tools only)."""
import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["SNN_RSTDP_DBG"] = "8"
import bench
step = bench.C4Step(torch, torch.device("cuda", 0))
for _ in range(2): step.run()
torch.cuda.synchronize()
from paper_1903_02440_b200 import snn
L = snn.lib()
buf = (ctypes.c_ulonglong * (4 * 1000))()
L.snn_debug_rstdp_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.snn_debug_rstdp_stamps(ctypes.cast(buf, ctypes.c_void_p), 1000)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1000, 4).astype(np.int64)
st, am, en = a[:, 0], a[:, 1], a[:, 2]
print("tail 1 (winner, decision) us: median %.2f" % (np.median(am - st) / 1e3))
ok = en > 0
print("tail 2 (R-STDP, limbs) us: median %.2f (n=%d)" % (np.median((en - am)[ok]) / 1e3, ok.sum()))
gap = st[1:] - np.where(ok[:-1], en[:-1], am[:-1])
print("tail 2 end -> next tail 1 start (GEMM + launches) us: median %.2f p90 %.2f" % (np.median(gap) / 1e3, np.percentile(gap, 90) / 1e3))
print("per image us: %.2f" % ((st[-1] - st[0]) / 999 / 1e3))
