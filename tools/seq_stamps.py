"""Phase timing of snn_stdp_sequence on C3 (CTA-0 globaltimer stamps in the workspace): A conv,
barrier 1, B inhibit/kWTA, barrier 2, C STDP.  Run on the GPU box."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1903_02440_b200 import pipeline, snn
wl = synth.C3(n=2000)
dev = torch.device("cuda")
lat0 = snn.encode(torch.from_numpy(wl.X).to(dev), wl.T)
l1 = pipeline.Layer(wl.convs[0], torch.from_numpy(wl.weights[0]).to(dev), 2000, 6, 28, 28, wl.T, wl.pools[0], pool_v=False)
l1(lat0)
seq = pipeline.SeqPersistent(wl.convs[1], wl.weights[1], l1.plat, wl.T, wl.extra["k"], wl.extra["r"], wl.extra["stdp"])
for _ in range(3):
    seq.replay()
torch.cuda.synchronize()
F, HoWo, N, k = 250, 196, 2000, wl.extra["k"]
r256 = lambda x: (x + 255) // 256 * 256
G = int(os.environ.get("SEQ_GROUPS", "8"))  # feature groups of the plan (ceil(F / (32 * FPL))); C3 default FPL 1
off = 256 + r256(F * HoWo) + r256(F * HoWo * 4) + r256(N * k * 4) + r256(G * HoWo * 8)
st = seq.ws[off:off + N * 48].view(torch.int64).cpu().numpy().reshape(N, 6).astype(np.float64)
d = np.diff(st, axis=1)[100:]
ca = seq.ws[off + N * 48: off + N * 48 + 148 * 16].view(torch.int64).cpu().numpy().reshape(148, 2).astype(np.float64)
t0 = ca[:, 0].min()
dur = (ca[:, 1] - ca[:, 0]) / 1e3
print("image 100 phase A per CTA: start skew max %.2f us, duration min %.2f median %.2f max %.2f us, slowest CTAs %s" % (
    (ca[:, 0].max() - t0) / 1e3, dur.min(), np.median(dur), dur.max(), np.argsort(-dur)[:6].tolist()))
sub = seq.ws[off + N * 48 + 400 * 8: off + N * 48 + 402 * 8].view(torch.int64).cpu().numpy().astype(np.float64)
print("image 100 B: keys %.2f us, rounds %.2f us, tail %.2f us" % ((sub[0] - st[100, 2]) / 1e3, (sub[1] - sub[0]) / 1e3,
                                                                 (st[100, 3] - sub[1]) / 1e3))
print("per image us: A %.2f  bar1 %.2f  B %.2f  bar2 %.2f  C %.2f  | next-image gap %.2f" % tuple(
    list(d.mean(0) / 1e3) + [np.mean(st[101:, 0] - st[100:-1, 5]) / 1e3]))
