"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 bookkeeping:
image sharding is a disjoint cover, job throughput = sum of units / max of times, barrier works."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_1903_02440_b200 import dist
    dist.init("gloo")
    r, w, lr = dist.env()
    start, stop = dist.shard(1000, r, w)
    units = stop - start
    t = 0.5 + r            # rank 1 is the slowest
    dist.barrier()
    thr = dist.job_throughput(units, t)
    q.put((r, start, stop, thr, dist.max_over_ranks(t), dist.sum_over_ranks(units)))
    import torch.distributed as td
    td.destroy_process_group()


def test_shard_cover_single_process():
    from paper_1903_02440_b200 import dist
    for total in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b = dist.shard(total, r, world)
                seen.extend(range(a, b))
            assert seen == list(range(total))


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, thr0, mx0, su0), (r1, a1, b1, thr1, mx1, su1) = res
    assert (a0, b0, a1, b1) == (0, 500, 500, 1000)
    assert mx0 == mx1 == 1.5 and su0 == su1 == 1000
    assert thr0 == thr1 == pytest.approx(1000 / 1.5)


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch
    from paper_1903_02440_b200 import dist
    dist.init("gloo")
    # each rank's per-image decisions of its own equal-size batch; the gather returns all ranks', rank order
    dec = torch.arange(5, dtype=torch.int32) + 100 * rank
    dec[rank] = -1                                    # a silent image
    out = dist.gather_decisions(dec)
    q.put((rank, out.tolist()))
    import torch.distributed as td
    td.destroy_process_group()


def test_gather_decisions_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [-1, 1, 2, 3, 4, 100, -1, 102, 103, 104]
    assert res == [(0, want), (1, want)]


def test_gather_decisions_single_process_is_identity():
    import torch
    from paper_1903_02440_b200 import dist
    d = torch.tensor([3, -1, 7], dtype=torch.int32)
    assert dist.gather_decisions(d) is d


def test_bench_spawns_ranks_for_gpus(monkeypatch):
    """bench.py --gpus N without a torchrun environment re-launches itself under torchrun with N ranks
    (one process per GPU) and the same arguments; with WORLD_SIZE set it refuses a mismatch."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    cmd = bench.spawn_cmd(["--gpus", "4", "--steps", "3"], 4, 29501)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29501" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert "WORLD_SIZE=2" in str(e.value)
