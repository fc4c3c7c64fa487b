#!/usr/bin/env python
"""bench.py -- throughput of the B200 spike-wave step (SpykeTorch, arxiv 1903.02440).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

Default workload = BASELINE.json configs[1] (C2): 3-layer DCSNN inference, T = 15, on a batch of
1000 seeded synthetic 28x28 stroke images (DoG on/off, 6 channels).  One step = one pass of the hot
path over the batch: encode -> conv+fire -> pool -> conv+fire -> pool -> conv (theta = inf) ->
1-winner readout -> class.  Inputs are resident in HBM when the timed region starts; L2 is flushed
(256 MiB write) between timed steps, outside the step's event pair.

Multi-GPU (torchrun, one process per GPU, NCCL): every rank processes its own batch of the same size
(weak scaling, images are independent -- no data-path collective); time = max over
ranks of the summed step times; value = images of all ranks / that time.

``--impl reference`` times the CPU oracle (oracle/, plain C, fp64) as it stands on the host cores,
on a bounded sample of the same workload per step (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images/sec & synaptic events/sec (3-layer DCSNN, T=15); % roofline"
SMEM_BYTES_PER_CLK_SM = 128          # shared-memory crossbar (B300_MICROARCH.md "LDS/STS")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no flush/clocks/baselines")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sus=d.get("bf16_tflops_sustained", 1400.0), sm_max=d.get("sm_max_mhz", 1965.0),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_max=1965.0, src="fallback")


# --------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------------------- workloads
def _pipelined(step, dev_in, x_host, out_host, result, steps):
    """e2e with copy/compute overlap: step k's inputs are copied (pinned H2D, second stream) into one of
    two device buffers while step k-1 computes; each step still copies its own inputs and reads back its
    result (D2H on the compute stream)."""
    torch = step.torch
    if not hasattr(step, "_pipe"):
        step._pipe = ([dev_in, torch.empty_like(dev_in)], torch.cuda.Stream(),
                      [torch.cuda.Event() for _ in range(2)], [torch.cuda.Event() for _ in range(2)])
    bufs, cs, ready, done = step._pipe
    main = torch.cuda.current_stream()
    cs.wait_stream(main)
    for k in range(steps):
        b = k % 2
        with torch.cuda.stream(cs):
            if k >= 2:
                cs.wait_event(done[b])  # step k-2 has finished reading this buffer
            bufs[b].copy_(x_host, non_blocking=True)
            ready[b].record(cs)
        main.wait_event(ready[b])
        step.run(src=bufs[b])
        done[b].record(main)
        out_host.copy_(result(), non_blocking=True)
    main.wait_stream(cs)


class C2Step:
    """configs[1]: 3-layer inference over a resident batch."""
    name = "c2"

    def __init__(self, torch, dev, batch=1000):
        import synth
        from paper_1903_02440_b200 import pipeline, snn
        self.torch, self.snn = torch, snn
        self.wl = synth.C2(n=batch)
        self.B = batch
        self.net = pipeline.C2Net(self.wl, batch, device=dev)
        self.x = torch.from_numpy(self.wl.X).to(dev)
        # f2 front end: the step starts from the raw fp64 images and filters them on the GPU (R33)
        self.raw = torch.from_numpy(self.wl.extra["raw"]).to(dev)
        self.bank = torch.from_numpy(self.wl.extra["bank"]).to(dev)
        self.stages = ["dog", "encode", "conv1", "pool1", "conv2", "pool2", "conv3", "kwta", "decide"]

    def run(self, ev=None, src=None):
        n, snn, T = self.net, self.snn, self.wl.T
        s1, s2, s3 = self.wl.convs
        fr = self.wl.extra["front"]

        def mark(i):
            if ev is not None:
                ev[i].record()
        mark(0)
        snn.filter_bank(self.raw if src is None else src, self.bank, fr["pad"], mode=fr["mode"], out=self.x); mark(1)
        n.encode(self.x); mark(2)         # channels-last maps from here to layer 3's input
        if n.l1.fuse_pool:                # conv1 + its 2 x 2 pooling in one launch (K7, SNN_CONV_POOL2)
            n.l1.conv_pool(n.lat0_buf); mark(3); mark(4)
        else:
            n.l1.conv(n.lat0_buf); mark(3)    # no potentials: pool1 needs none
            n.l1.pool(); mark(4)
        n.l2.conv(n.l1.out_lat); mark(5)
        n.l2.pool(); mark(6)
        n.l3.conv(n.l2.out_lat); mark(7)
        snn.k_winners(n.l3.lat, n.l3.v, 1, 0, winners=n.winners, count=n.count, ws=n.ws_kw); mark(8)
        snn.decide(n.winners, n.count, s3.F, self.wl.extra["n_classes"], None, decision=n.decision,
                   reward=n.reward); mark(9)

    def e2e(self, x_host, out_host):
        """Public-API path with host buffers: H2D of the raw images, the step, D2H of the decisions."""
        self.raw.copy_(x_host, non_blocking=True)
        self.run()
        out_host.copy_(self.net.decision, non_blocking=True)

    def e2e_pipelined(self, x_host, out_host, steps):
        """The same per-step work with the next step's H2D copy on a second stream, overlapping the
        current step's kernels (two device input buffers, events order the reuse)."""
        return _pipelined(self, self.raw, x_host, out_host, lambda: self.net.decision, steps)

    def host_io(self):
        xh = self.torch.from_numpy(self.wl.extra["raw"]).pin_memory()
        oh = self.torch.empty((self.B,), dtype=self.torch.int32).pin_memory()
        return xh, oh

    def events(self):
        """(paper events per batch, necessary events per conv layer) -- off the clock."""
        n, snn, T = self.net, self.snn, self.wl.T
        self.run()
        n.l1.conv(n.lat0_buf)             # the unpooled conv1 map (the fused step writes only its pooling)
        out = {}
        for name, lat_in, spec, lo in (("conv1", n.lat0, self.wl.convs[0], n.l1.lat),
                                       ("conv2", n.l1.plat, self.wl.convs[1], n.l2.lat),
                                       ("conv3", n.l2.plat, self.wl.convs[2], n.l3.lat)):
            out[name] = snn.count_events(lat_in.contiguous(), spec.F, spec.KH, spec.KW, spec.pad, T, lo.contiguous())
            out["_shape_" + name] = (int(lat_in.shape[1]), int(lo.shape[0] * lo.shape[2] * lo.shape[3]))
        return out

    def config(self):
        return {"workload": "c2: BASELINE.json configs[1], 3-layer DCSNN inference, T=15",
                "global_batch": self.B, "images": "raw 28x28 fp64 strokes (synthetic) -> GPU DoG bank on/off (6 ch)",
                "layers": "F30 5x5 p2 th15 -> pool2/2 -> F250 3x3 p1 th10 -> pool3/3 -> F200 5x5 p2 th=inf -> 1 winner",
                "l2": "flushed between timed steps (256 MiB write, outside the step events)"}

    def units(self):
        return self.B

    def oracle_step(self, n):
        from oracle import flows
        import synth
        wl = self.wl if n == self.B else synth.Workload("c2", self.wl.T, self.wl.X[:n], self.wl.convs,
                                                         self.wl.weights, self.wl.pools,
                                                         dict(self.wl.extra, raw=self.wl.extra["raw"][:n]))
        flows.c2(wl, front=True)


class C5Step(C2Step):
    name = "c5"

    def __init__(self, torch, dev, batch=64):
        import synth
        from paper_1903_02440_b200 import pipeline, snn
        self.torch, self.snn = torch, snn
        self.wl = synth.C5(n=batch)
        self.B = batch
        self.net = pipeline.C5Net(self.wl, batch, device=dev)
        self.x = torch.from_numpy(self.wl.X).to(dev)
        self.stages = ["encode", "conv1", "pool1", "inhibit", "kwta"]

    def run(self, ev=None, src=None):
        n, snn, T = self.net, self.snn, self.wl.T
        s = self.wl.convs[0]

        def mark(i):
            if ev is not None:
                ev[i].record()
        mark(0)
        n.encode(self.x if src is None else src); mark(1)
        n.l1.conv(n.lat0_buf); mark(2)    # channels-last in and out (lat, v): coalesced walk loads and stores
        n.l1.pool(); mark(3)
        snn.inhibit(n.l1.plat, n.l1.pv, lat_out=n.ilat, v_out=n.iv, winner_f=n.wf); mark(4)
        snn.k_winners(n.ilat, n.iv, self.wl.extra["k"], self.wl.extra["r"], winners=n.winners, count=n.count,
                      ws=n.ws_kw); mark(5)

    def e2e(self, x_host, out_host):
        self.x.copy_(x_host, non_blocking=True)
        self.run()
        out_host.copy_(self.net.winners, non_blocking=True)

    def e2e_pipelined(self, x_host, out_host, steps):
        return _pipelined(self, self.x, x_host, out_host, lambda: self.net.winners, steps)

    def host_io(self):
        xh = self.torch.from_numpy(self.wl.X).pin_memory()
        oh = self.torch.empty(tuple(self.net.winners.shape), dtype=self.torch.int32).pin_memory()
        return xh, oh

    def events(self):
        n, snn, T = self.net, self.snn, self.wl.T
        self.run()
        s = self.wl.convs[0]
        return {"conv1": snn.count_events(n.lat0.contiguous(), s.F, s.KH, s.KW, s.pad, T, n.l1.lat.contiguous())}

    def config(self):
        return {"workload": "c5: BASELINE.json configs[4], throughput stress, T=32", "global_batch": self.B,
                "layers": "F256 5x5 p2 th40 (32 ch 256x256) -> pool2/2 -> inhibit -> kWTA k16 r4",
                "l2": "inputs (537 MB) larger than L2; also flushed between steps"}

    def oracle_step(self, n):
        from oracle import flows
        import synth
        flows.c5(synth.Workload("c5", self.wl.T, self.wl.X[:n], self.wl.convs, self.wl.weights, self.wl.pools,
                                self.wl.extra))


class SeqBase(C2Step):
    """Sequential plasticity configs: a batched fixed-weight prefix, then a CUDA graph of per-image
    plasticity steps (conv+fire -> [inhibit] -> kWTA -> [decide] -> STDP), no host sync per image."""
    def _prefix(self, src=None, mark=lambda i: None):
        snn, T = self.snn, self.wl.T
        snn.encode(self.x if src is None else src, T, out=self.lat0, ws=self.ws_enc, nhwc=self.l1 is not None)
        mark(1)
        if self.l1 is not None:  # layer 1 reads and writes channels-last maps, its pool writes planar ones
            self.l1.conv(self.lat0); mark(2)
            self.l1.pool(); mark(3)
        if getattr(self, "prep", None) is not None:  # C4: the theta = +inf layer's A operands, all images
            s2 = self.wl.convs[1]
            snn.conv_inf_prepare(self.l1.plat, s2.F, s2.KH, s2.KW, s2.pad, T, out=self.prep)
        mark(4)

    def run(self, ev=None, src=None):
        def mark(i):
            if ev is not None:
                ev[i].record()
        mark(0)
        self._prefix(src, mark)
        self.graph.replay(); mark(5)

    def e2e(self, x_host, out_host):
        self.x.copy_(x_host, non_blocking=True)
        self.run()
        out_host.copy_(self.seq.w, non_blocking=True)

    def e2e_pipelined(self, x_host, out_host, steps):
        """Each step's images copied on a second stream while the previous step trains (2 buffers)."""
        return _pipelined(self, self.x, x_host, out_host, lambda: self.seq.w, steps)

    def host_io(self):
        xh = self.torch.from_numpy(self.wl.X).pin_memory()
        oh = self.torch.empty(tuple(self.seq.w.shape), dtype=self.torch.float32).pin_memory()
        return xh, oh

    def events(self):
        self.run()
        s = self.wl.convs[-1]
        lat_in = self.l1.plat if self.l1 is not None else self.lat0
        out = {"seq": self.snn.count_events(lat_in, s.F, s.KH, s.KW, s.pad, self.wl.T, None)}
        if self.l1 is not None:  # layer 1 (batched, fixed weights): paper and necessary events
            s1 = self.wl.convs[0]
            lat0 = self.lat0.permute(0, 3, 1, 2).contiguous()
            out["conv1"] = self.snn.count_events(lat0, s1.F, s1.KH, s1.KW, s1.pad, self.wl.T, self.l1.lat.contiguous())
        return out


class C3Step(SeqBase):
    name = "c3"

    def __init__(self, torch, dev, batch=2000):
        import synth
        from paper_1903_02440_b200 import pipeline, snn
        self.torch, self.snn = torch, snn
        self.wl = wl = synth.C3(n=batch)
        self.B = batch
        self.x = torch.from_numpy(wl.X).to(dev)
        _, C, H, W = wl.X.shape
        self.ws_enc = torch.empty(snn.encode_workspace(batch, C, H, W, wl.T), dtype=torch.uint8, device=dev)
        self.lat0 = torch.empty((batch, H, W, C), dtype=torch.uint8, device=dev)   # channels-last
        self.l1 = pipeline.Layer(wl.convs[0], torch.from_numpy(wl.weights[0]).to(dev), batch, C, H, W, wl.T,
                                 wl.pools[0], pool_v=False, device=dev, nhwc=True, want_v=False, in_nhwc=True)
        self._prefix()
        s2 = wl.convs[1]
        if pipeline.SeqPersistent.supported(s2, tuple(self.l1.plat.shape), wl.weights[1].shape, wl.T, wl.extra["k"]):
            # all 2000 plasticity steps in one persistent kernel (snn_stdp_sequence)
            self.seq = self.graph = pipeline.SeqPersistent(s2, wl.weights[1], self.l1.plat, wl.T, wl.extra["k"],
                                                           wl.extra["r"], wl.extra["stdp"],
                                                           snapshot_every=wl.extra["snapshot_every"], device=dev)
            self.mode = "one persistent kernel (snn_stdp_sequence)"
        else:
            self.seq = pipeline.SeqSTDP(s2, wl.weights[1], wl.convs[0].F, self.l1.PHo, self.l1.PWo, wl.T,
                                        wl.extra["k"], wl.extra["r"], True, wl.extra["stdp"], device=dev)
            self.graph = pipeline.SeqGraph(self.seq, self.l1.plat, batch, snapshot_every=wl.extra["snapshot_every"])
            self.mode = "per-image CUDA graph, no host sync"
        self.stages = ["encode", "conv1", "pool1", "prep", "seq_stdp"]

    def config(self):
        return {"workload": "c3: BASELINE.json configs[2], sequential STDP on layer 2, 2000 images",
                "global_batch": self.B, "layers": "C2 L1 (fixed) -> pool -> L2 F250 3x3 th10 -> inhibit -> kWTA k8 r2 -> STDP",
                "plasticity": self.mode, "l2": "flushed between timed steps"}

    def oracle_step(self, n):
        from oracle import flows
        import synth
        flows.c3(synth.Workload("c3", self.wl.T, self.wl.X[:n], self.wl.convs, self.wl.weights, self.wl.pools,
                                self.wl.extra), snapshot_every=10 ** 9)


class C4Step(SeqBase):
    name = "c4"

    def __init__(self, torch, dev, batch=1000):
        import synth
        from paper_1903_02440_b200 import pipeline, snn
        self.torch, self.snn = torch, snn
        self.wl = wl = synth.C4(n=batch)
        self.B = batch
        self.x = torch.from_numpy(wl.X).to(dev)
        _, C, H, W = wl.X.shape
        self.ws_enc = torch.empty(snn.encode_workspace(batch, C, H, W, wl.T), dtype=torch.uint8, device=dev)
        self.lat0 = torch.empty((batch, H, W, C), dtype=torch.uint8, device=dev)   # channels-last
        self.l1 = pipeline.Layer(wl.convs[0], torch.from_numpy(wl.weights[0]).to(dev), batch, C, H, W, wl.T,
                                 wl.pools[0], pool_v=False, device=dev, nhwc=True, want_v=False, in_nhwc=True)
        self.labels = torch.from_numpy(wl.extra["labels"].astype(np.int32)).to(dev)
        s2 = wl.convs[1]
        _, C2, H2, W2 = self.l1.plat.shape
        # theta = +inf layer: its A operands (weight-independent) for all images, built in the prefix
        self.prep = torch.empty(max(snn.lib().snn_conv_inf_prepare_bytes(batch, C2, H2, W2, s2.pad, s2.F, s2.KH, s2.KW), 1),
                                dtype=torch.uint8, device=dev)
        self._prefix()
        # f1: every image's chain (GEMM + tail CTA) from snn_rstdp_inf_sequence, captured as one CUDA graph
        self.seq = pipeline.SeqInfRSTDP(s2, wl.weights[1], self.l1.plat, self.prep, self.labels, wl.T,
                                        wl.extra["n_classes"], wl.extra["stdp"], device=dev)
        self.graph = pipeline.StepGraph(self.seq.replay)
        self.stages = ["encode", "conv1", "pool1", "prep", "seq_rstdp"]

    def config(self):
        return {"workload": "c4: BASELINE.json configs[3], Caltech-shaped R-STDP, 1000 sequential images, T=30",
                "global_batch": self.B,
                "layers": "F20 5x5 th15 (4x160x250) -> pool7/6 -> F100 17x17 th=inf (tcgen05) -> 1 winner -> decide -> R-STDP",
                "plasticity": "snn_rstdp_inf_sequence (per image: tcgen05 GEMM + one tail CTA for winner, decision, "
                              "R-STDP and the winner's limbs), one CUDA graph, no host sync",
                "l2": "flushed between timed steps"}

    def oracle_step(self, n):
        from oracle import flows
        import synth
        ex = dict(self.wl.extra)
        flows.c4(synth.Workload("c4", self.wl.T, self.wl.X[:n], self.wl.convs, self.wl.weights, self.wl.pools, ex))


class C1Step(SeqBase):
    name = "c1"

    def __init__(self, torch, dev, batch=1):
        import synth
        from paper_1903_02440_b200 import pipeline, snn
        self.torch, self.snn = torch, snn
        self.wl = wl = synth.C1()
        self.B = 1
        self.x = torch.from_numpy(wl.X).to(dev)
        self.ws_enc = torch.empty(snn.encode_workspace(1, 2, 28, 28, wl.T), dtype=torch.uint8, device=dev)
        self.lat0 = torch.empty(wl.X.shape, dtype=torch.uint8, device=dev)
        self.l1 = None
        s1 = wl.convs[0]
        # one image: the per-call kernels in one CUDA graph beat the persistent kernel's fixed cost
        # (list presort + cooperative launch + grid barriers); SNN_C1_PERSISTENT=1 selects it anyway
        if os.environ.get("SNN_C1_PERSISTENT") == "1" and pipeline.SeqPersistent.supported(
                s1, tuple(self.lat0.shape), wl.weights[0].shape, wl.T, wl.extra["k"]):
            # encode + the plasticity step (one persistent kernel, N = 1), captured as one CUDA graph
            self.seq = pipeline.SeqPersistent(s1, wl.weights[0], self.lat0, wl.T, wl.extra["k"], wl.extra["r"],
                                              wl.extra["stdp"], device=dev)

            def body():
                self._prefix()
                self.seq.replay()
            self.mode = "encode + snn_stdp_sequence as one CUDA graph"
        else:
            self.seq = pipeline.SeqSTDP(s1, wl.weights[0], 2, 28, 28, wl.T, wl.extra["k"], wl.extra["r"], True,
                                        wl.extra["stdp"], device=dev)
            w0 = self.seq.w.clone()

            def body():
                self.seq.w.copy_(w0)
                self._prefix()
                self.seq.step(self.lat0)
            self.mode = "whole step as one CUDA graph"
        self.graph = pipeline.StepGraph(body)
        self.stages = ["step"]

    def run(self, ev=None, src=None):
        if ev is not None:
            ev[0].record()
        if src is not None and src.data_ptr() != self.x.data_ptr():
            self.x.copy_(src)  # the captured graph reads self.x (a 6 KB device copy)
        self.graph.replay()
        if ev is not None:
            ev[1].record()

    def config(self):
        return {"workload": "c1: BASELINE.json configs[0], single layer, batch 1: encode -> conv+fire -> inhibit -> kWTA k5 r3 -> STDP",
                "global_batch": 1, "plasticity": self.mode, "l2": "flushed between timed steps"}

    def oracle_step(self, n):
        from oracle import flows
        flows.c1(self.wl)


WORKLOADS = {"c1": C1Step, "c2": C2Step, "c3": C3Step, "c4": C4Step, "c5": C5Step}


# --------------------------------------------------------------------------------------- roofline
def _traffic(wl_name, stage):
    """DRAM bytes per step of the stage from the committed ncu capture (profiles/*_traffic.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return None, None
    d = json.load(open(files[-1]))
    v = d.get(f"{wl_name}:{stage}")
    return (int(v) if v is not None else None), os.path.relpath(files[-1], ROOT)


def roofline(stage, t_ms, ev, wl, clocks, pk, wl_name="c2"):
    """Roofline of the dominant stage from its algorithmic work per step."""
    f_mhz = (clocks or {}).get("sm_mhz") or pk["sm_max"]
    t = t_ms * 1e-3
    if stage.startswith("conv"):
        paper, need = ev[stage]
        idx = int(stage[-1]) - 1
        spec = wl.convs[idx]
        traffic, tsrc = _traffic(wl_name, stage)
        if math.isinf(spec.theta):
            # Eq. 5: one dense contraction of S[T-1] on the int8 tensor pipe, 4 exact u8 limbs per weight:
            # 2 ops x 4 limbs x positions x F x R (algorithmic, unpadded); peak = measured bf16 x 2 (int8 rate)
            C_in, M = ev["_shape_" + stage]  # input channels, output positions per step
            R = C_in * spec.KH * spec.KW
            ops = 2.0 * 4 * M * spec.F * R
            peak = pk["bf16"] * 2e12
            return {"bound": "tensor", "achieved": round(ops / t / 1e12, 1), "peak": round(peak / 1e12, 1),
                    "unit": "TFLOP/s", "frac": round(ops / t / peak, 4), "traffic": traffic, "traffic_src": tsrc,
                    "kernel": stage, "work": f"{ops:.3e} int8 ops (4 limbs x 2 x {M} positions x {spec.F} x {R})",
                    "peak_src": f"measured bf16 {pk['bf16']} TFLOP/s x 2 (int8:bf16 nominal ratio)"}
        peak = SMEM_BYTES_PER_CLK_SM * 148 * f_mhz * 1e6
        ach = need * 4 / t
        return {"bound": "smem", "achieved": round(ach / 1e9, 1), "peak": round(peak / 1e9, 1), "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "traffic_src": tsrc, "kernel": stage,
                "work": f"{need} necessary events x 4 B weight gather (of {paper} paper-definition events)",
                "peak_src": f"128 B/clk/SM x 148 SMs x {f_mhz:.0f} MHz (measured SM clock)"}
    if stage.startswith("seq") or stage == "step":
        return {"bound": "latency", "achieved": round(t_ms * 1e3 / max(1, wl.X.shape[0]), 3), "peak": None,
                "unit": "us/image", "frac": None, "traffic": None, "kernel": stage,
                "work": "sequential per-image plasticity chain (each image's weights feed the next, P:95)"}
    return None


# --------------------------------------------------------------------------------------- arms
def run_reference(args, rank):
    if rank != 0:
        return
    import synth  # noqa: F401
    import torch
    step = WORKLOADS[args.workload].__new__(WORKLOADS[args.workload])
    step.wl = {"c1": synth.C1, "c2": lambda: synth.C2(n=1000), "c3": lambda: synth.C3(n=200),
               "c4": lambda: synth.C4(n=20), "c5": lambda: synth.C5(n=2)}[args.workload]()
    step.B = step.wl.X.shape[0]
    sample = {"c1": 1, "c2": 100, "c3": 20, "c4": 5, "c5": 1}[args.workload]
    for _ in range(args.warmup):
        step.oracle_step(sample)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step.oracle_step(sample)
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    val = sample * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "images/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "sample_images_per_step": sample},
            "cpu_baseline": {"value": round(val, 3), "unit": "images/s", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} images of the {args.workload} batch per step"},
            "e2e": {"value": round(val, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_1903_02440_b200 import snn
    snn.lib()
    step = WORKLOADS[args.workload](torch, dev)
    torch.cuda.synchronize()

    from paper_1903_02440_b200 import dist as sdist
    barrier = sdist.barrier

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if not args.profile else None
    nst = len(step.stages)
    for _ in range(args.warmup):
        step.run()
    snn.sync_status()
    # ---------------- timed region ----------------
    sampler = ClockSampler(local) if (rank == 0 and not args.no_clocks and not args.profile) else None
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst + 1)] for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    launches0 = snn.launch_count()
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
        step.run(ev[k])
    launches = snn.launch_count() - launches0
    if getattr(step, "graph", None) is not None:      # kernels replayed from a captured CUDA graph
        launches += args.steps * step.graph.launches
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    snn.sync_status()
    step_ms = [ev[k][0].elapsed_time(ev[k][nst]) for k in range(args.steps)]
    stage_ms = [statistics.mean(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(args.steps)) for i in range(nst)]
    total_ms = sdist.max_over_ranks(sum(step_ms), dev)   # the job's time = the slowest rank
    units = step.B * args.steps * world
    value = units / (total_ms * 1e-3)
    # ---------------- off-clock: events, e2e, cpu baseline ----------------
    ev_counts = step.events()
    paper_events = sum(v[0] for k, v in ev_counts.items() if not k.startswith("_"))
    e2e = None
    if not args.no_e2e and not args.profile:
        xh, oh = step.host_io()
        pipe = getattr(step, "e2e_pipelined", None)
        for _ in range(2):
            step.e2e(xh, oh)
        if pipe:
            pipe(xh, oh, 2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record()
        if pipe:
            pipe(xh, oh, args.steps)
        else:
            for _ in range(args.steps):
                step.e2e(xh, oh)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = sdist.max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": round(step.B * args.steps * world / (e2e_ms * 1e-3), 3), "unit": "images/s",
               "h2d_bytes_per_step": int(xh.numel() * xh.element_size()),
               "d2h_bytes_per_step": int(oh.numel() * oh.element_size()),
               "copy_overlap": ("step k+1's H2D on a second stream overlaps step k's kernels (2 device buffers)"
                                if pipe else None)}
    if rank != 0:
        return
    pk = peaks()
    dom = max(range(nst), key=lambda i: stage_ms[i])
    roof = roofline(step.stages[dom], stage_ms[dom], ev_counts, step.wl, clocks, pk, step.name)
    stage_roofs = {}
    for i, st in enumerate(step.stages):  # every conv stage, for context (the dominant one is "roofline")
        if st.startswith("conv") and st in ev_counts:
            r_ = roofline(st, stage_ms[i], ev_counts, step.wl, clocks, pk, step.name)
            stage_roofs[st] = {k: r_[k] for k in ("bound", "achieved", "unit", "frac", "traffic")}
    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        n = {"c1": 1, "c2": 1000, "c3": 200, "c4": 30, "c5": 1}[step.name]
        t0 = time.perf_counter()
        step.oracle_step(n)
        dt = time.perf_counter() - t0
        cpu = {"value": round(n / dt, 3), "unit": "images/s",
               "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())), "kind": "oracle",
               "sample": f"{n} images of the {step.name} batch, one pass (OpenMP over images)"}
    line = {"metric": METRIC, "value": round(value, 3), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": step.config(),
            "events_per_sec": round(paper_events * args.steps * world / (total_ms * 1e-3), 1),
            "events_per_step": paper_events,
            "stages_ms": {s: round(m, 4) for s, m in zip(step.stages, stage_ms)},
            "roofline": roof, "stage_rooflines": stage_roofs, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": int(launches),
            "peaks": {"src": pk["src"], "hbm_gbs": pk["hbm"], "bf16_tflops": pk["bf16"]}}
    print(json.dumps(line), flush=True)


def spawn_cmd(argv, gpus: int, port: int):
    """The torchrun command that runs this bench with one process per GPU (used when ``--gpus N`` > 1 is
    given without a torchrun environment)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without torchrun: start the N ranks ourselves (one process per GPU), same arguments
        if args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
        sys.exit(subprocess.call(spawn_cmd(sys.argv[1:], args.gpus, _free_port())))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        from paper_1903_02440_b200 import dist as sdist
        torch.cuda.set_device(local)
        sdist.init("nccl", torch.device("cuda", local))
    try:
        run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
