"""Full-size parity in the bench's own launch configuration (bench.py's step objects, the timed code
path): C4's whole 1000-image R-STDP chain and every one of C5's 64 images downstream of the conv.

C4: the final W2 after 1000 sequential R-STDP images depends on every image's winner, decision and
update (Eq. 4), so bit-equality with the oracle chain (oracle.flows.c4) checks all of
them; the layer-1 pooled maps are compared too.  C5: the conv output of all 64 images is checked on
sampled neurons in test_gpu_configs (the oracle computes neurons one by one); here the GPU's own
conv output of all 64 images goes through the ORACLE pool / inhibition / k-WTA and every pooled map,
inhibition map and winner list must equal the GPU's (Eq. 3)."""
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def B():
    assert torch.cuda.is_available()
    sys.path.insert(0, ROOT)
    from paper_1903_02440_b200 import build
    build.build()
    import bench
    return bench


def test_c4_full_chain_bench_config(B, orc):
    from oracle import flows
    dev = torch.device("cuda", 0)
    step = B.C4Step(torch, dev)
    step.run()
    torch.cuda.synchronize()
    step.snn.sync_status()
    ref = flows.c4(step.wl)
    assert np.array_equal(step.l1.plat.cpu().numpy(), ref["l1_pool_lat"])
    assert np.array_equal(step.seq.decision.cpu().numpy(), ref["decision"])      # every image's decision
    assert np.array_equal(step.seq.winners.cpu().numpy(), np.asarray(ref["winners"]).reshape(-1, 3))
    assert np.array_equal(step.seq.w.cpu().numpy(), ref["w2"])


def test_c5_all_images_downstream_bench_config(B, orc):
    dev = torch.device("cuda", 0)
    step = B.C5Step(torch, dev)
    step.run()
    torch.cuda.synchronize()
    step.snn.sync_status()
    n, wl = step.net, step.wl
    lat = n.l1.lat.contiguous().cpu().numpy()       # planar view of the channels-last conv output
    v = n.l1.v.contiguous().cpu().numpy()
    p = wl.pools[0]
    pl, pv = orc.pool(lat, v, p.PH, p.PW, p.SH, p.SW, p.DH, p.DW, wl.T)
    assert np.array_equal(n.l1.plat.cpu().numpy(), pl)
    assert np.array_equal(n.l1.pv.cpu().numpy(), pv)
    il, iv, wf = orc.inhibit(pl, pv)
    assert np.array_equal(n.ilat.cpu().numpy(), il)
    assert np.array_equal(n.iv.cpu().numpy(), iv)
    win, cnt = orc.k_winners(il, iv, wl.extra["k"], wl.extra["r"])
    assert np.array_equal(n.count.cpu().numpy(), cnt)
    assert np.array_equal(n.winners.cpu().numpy(), win)
