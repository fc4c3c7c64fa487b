"""GPU parity of bench.py's own timed steps (the launch configuration the bench measures), at the
BASELINE.json sizes: C2 (1000 raw images, front end included), C3 (all 2000 sequential STDP images in
the persistent kernel, snapshots every 500), C4 (the per-image CUDA-graph R-STDP chain; a 250-image
prefix of the 1000-image config: the chain is sequential, so a prefix is the config's own start)."""
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


@pytest.fixture(scope="module")
def bench():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1903_02440_b200 import build
    build.build()
    import bench as b
    return b


def test_c2_bench_step(bench):
    from oracle import flows
    step = bench.C2Step(torch, torch.device("cuda", 0))
    step.run()
    torch.cuda.synchronize()
    ref = flows.c2(step.wl, front=True)
    assert np.array_equal(step.x.cpu().numpy(), step.wl.X)
    assert np.array_equal(step.net.l3.lat.cpu().numpy(), ref["l3"]["lat"])
    assert np.array_equal(step.net.l3.v.cpu().numpy(), ref["l3"]["v"])
    assert np.array_equal(step.net.decision.cpu().numpy(), ref["decision"])


def test_c3_bench_step_full(bench):
    from oracle import flows
    step = bench.C3Step(torch, torch.device("cuda", 0))
    step.run()
    torch.cuda.synchronize()
    ref = flows.c3(step.wl)
    seq = step.seq
    assert np.array_equal(seq.winners.cpu().numpy(), ref["winners"])
    for a, r in zip(seq.snaps.cpu().numpy(), ref["snapshots"]):
        assert np.array_equal(a, r)
    assert np.array_equal(seq.w.cpu().numpy(), ref["w2"])


def test_c4_bench_step_prefix(bench):
    from oracle import flows
    step = bench.C4Step(torch, torch.device("cuda", 0), batch=250)
    step.run()
    torch.cuda.synchronize()
    ref = flows.c4(step.wl)
    assert np.array_equal(step.seq.w.cpu().numpy(), ref["w2"])
