"""Config-level compositions of the libsnn calls (the paper's forward / training passes).

Each runner owns its device buffers (allocated once with torch), then issues the C-ABI calls of one
step asynchronously on the current stream.  No arithmetic happens here; every step is a libsnn
kernel.  Sequential plasticity (C1/C3/C4) keeps each image's update on the device: the R-STDP reward
is decided by ``snn_decide`` on the GPU, so no host round trip is needed per image.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np
import torch

from . import snn


def _dev(a, device, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a)).to(device)
    return t if dtype is None else t.to(dtype)


class Layer:
    """conv+fire (+ optional pool) with preallocated outputs.

    Layouts: nhwc -- the conv writes channels-last [B, Ho, Wo, F] (snn_conv_fire_ex
    SNN_CONV_OUT_NHWC: a walk warp's features of one position are contiguous, so its stores coalesce)
    and the pool reads that layout (SNN_POOL_IN_NHWC); in_nhwc -- the layer's input is channels-last
    [B, H, W, C] (SNN_CONV_IN_NHWC: a receptive field is KH x KW runs of C contiguous bytes);
    pool_out_nhwc -- the pooled output is channels-last too (the next layer's in_nhwc input).
    want_v False: the conv's potentials are not written (latency-only pooling needs none).
    ``lat``, ``v``, ``plat``, ``pv`` are always planar [B, F, H, W] views; ``*_buf`` the buffers."""

    def __init__(self, spec, w: torch.Tensor, B: int, C: int, H: int, W: int, T: int, pool_spec=None,
                 pool_v: bool = True, device="cuda", nhwc: bool = False, want_v: bool = True,
                 in_nhwc: bool = False, pool_out_nhwc: bool = False, fuse_pool: bool = False):
        self.spec, self.w, self.T = spec, w, T
        self.B, self.C, self.H, self.W = B, C, H, W
        self.Ho, self.Wo = snn.conv_out_hw(H, W, spec.KH, spec.KW, spec.pad)
        F = spec.F
        if pool_spec is not None and pool_v and not want_v:
            raise ValueError("pooled potentials need the conv's potentials (want_v)")
        if pool_out_nhwc and not nhwc:
            raise ValueError("a channels-last pooled output needs a channels-last conv output")
        self.nhwc, self.in_nhwc, self.pool_out_nhwc = nhwc, in_nhwc, pool_out_nhwc
        shape = (B, self.Ho, self.Wo, F) if nhwc else (B, F, self.Ho, self.Wo)
        self.lat_buf = torch.empty(shape, dtype=torch.uint8, device=device)
        self.v_buf = torch.empty(shape, dtype=torch.float32, device=device) if want_v else None
        self.ws = torch.empty(snn.conv_fire_workspace(B, C, H, W, spec.pad, F, spec.KH, spec.KW, T, spec.theta),
                              dtype=torch.uint8, device=device)
        self.pool_spec = pool_spec
        if pool_spec is not None:
            self.PHo, self.PWo = snn.pool_out_hw(self.Ho, self.Wo, pool_spec.PH, pool_spec.PW, pool_spec.SH,
                                                 pool_spec.SW, pool_spec.DH, pool_spec.DW)
            pshape = (B, self.PHo, self.PWo, F) if pool_out_nhwc else (B, F, self.PHo, self.PWo)
            self.plat_buf = torch.empty(pshape, dtype=torch.uint8, device=device)
            self.pv_buf = torch.empty(pshape, dtype=torch.float32, device=device) if pool_v else None
        # fuse_pool: 2 x 2 / stride 2 latency-only pooling inside the conv (SNN_CONV_POOL2, K7 row tiles);
        # the unpooled map (lat) is then not written.  The library declines (SNN_ESHAPE, before any launch)
        # where the row-tile walk does not apply; the layer then runs conv + pool from then on.
        self.fuse_pool = bool(fuse_pool and pool_spec is not None and not pool_v and not want_v and nhwc and in_nhwc
                              and pool_out_nhwc and math.isfinite(spec.theta) and
                              (pool_spec.PH, pool_spec.PW, pool_spec.SH, pool_spec.SW, pool_spec.DH, pool_spec.DW)
                              == (2, 2, 2, 2, 0, 0))

    @staticmethod
    def _planar(t, nhwc):
        if t is None:
            return None
        return t.permute(0, 3, 1, 2) if nhwc else t

    @property
    def lat(self):
        return self._planar(self.lat_buf, self.nhwc)

    @property
    def v(self):
        return self._planar(self.v_buf, self.nhwc)

    @property
    def plat(self):
        return self._planar(self.plat_buf, self.pool_out_nhwc)

    @property
    def pv(self):
        return self._planar(self.pv_buf, self.pool_out_nhwc)

    @property
    def out_lat(self):
        """What the next layer reads (its in_nhwc = this layer's pool_out_nhwc when pooled)."""
        if self.pool_spec is not None:
            return self.plat_buf
        return self.lat_buf

    @property
    def out_v(self):
        return self.pv_buf if self.pool_spec is not None else self.v_buf

    def conv(self, lat_in: torch.Tensor, w: Optional[torch.Tensor] = None):
        s = self.spec
        snn.conv_fire(lat_in, self.w if w is None else w, s.pad, self.T, s.theta, lat_out=self.lat_buf,
                      v_out=self.v_buf, ws=self.ws, nhwc=self.nhwc, want_v=self.v_buf is not None,
                      in_nhwc=self.in_nhwc)

    def pool(self):
        p = self.pool_spec
        flags = (snn.POOL_IN_NHWC if self.nhwc else 0) | (snn.POOL_OUT_NHWC if self.pool_out_nhwc else 0)
        snn.pool(self.lat_buf, self.v_buf if self.pv_buf is not None else None, (p.PH, p.PW), (p.SH, p.SW),
                 (p.DH, p.DW), lat_out=self.plat_buf, v_out=self.pv_buf, flags=flags)

    def conv_pool(self, lat_in: torch.Tensor, w: Optional[torch.Tensor] = None):
        """conv + pool: fused into one launch when fuse_pool holds (plat only), else the two calls."""
        if self.fuse_pool:
            s = self.spec
            try:
                snn.conv_fire(lat_in, self.w if w is None else w, s.pad, self.T, s.theta, lat_out=self.plat_buf,
                              ws=self.ws, nhwc=True, want_v=False, in_nhwc=True, pool2=True)
                return
            except snn.SNNError as e:
                if e.code != snn.SNN_ESHAPE:
                    raise
                self.fuse_pool = False
        self.conv(lat_in, w)
        self.pool()

    def __call__(self, lat_in: torch.Tensor, w: Optional[torch.Tensor] = None):
        if self.pool_spec is not None:
            self.conv_pool(lat_in, w)
        else:
            self.conv(lat_in, w)
        return self.out_lat


class C2Net:
    """3-layer DCSNN inference (configs[1]): encode -> [conv+fire -> pool] x 2 -> conv (theta = inf)
    -> 1 winner (global max potential) -> class = f // (F / 10).

    nhwc (the bench configuration): every map between the encoder and layer 3 is channels-last
    (encode -> conv1 -> pool1 -> conv2 -> pool2 -> conv3's input); conv_v False: layers 1 and 2 write
    no potentials (their latency-only pools need none).  Layer 3's output stays planar."""

    def __init__(self, wl, B: int, device="cuda", nhwc: bool = True, conv_v: bool = False, fuse_pool: bool = True):
        self.wl, self.B, self.T = wl, B, wl.T
        _, C, H, W = wl.X.shape
        self.nhwc = nhwc
        self.ws_enc = torch.empty(snn.encode_workspace(B, C, H, W, wl.T), dtype=torch.uint8, device=device)
        self.lat0_buf = torch.empty((B, H, W, C) if nhwc else (B, C, H, W), dtype=torch.uint8, device=device)
        self.w = [_dev(w, device) for w in wl.weights]
        s1, s2, s3 = wl.convs
        self.l1 = Layer(s1, self.w[0], B, C, H, W, wl.T, wl.pools[0], pool_v=False, device=device, nhwc=nhwc,
                        want_v=conv_v, in_nhwc=nhwc, pool_out_nhwc=nhwc, fuse_pool=fuse_pool)
        self.l2 = Layer(s2, self.w[1], B, s1.F, self.l1.PHo, self.l1.PWo, wl.T, wl.pools[1], pool_v=False,
                        device=device, nhwc=nhwc, want_v=conv_v, in_nhwc=nhwc, pool_out_nhwc=nhwc)
        self.l3 = Layer(s3, self.w[2], B, s2.F, self.l2.PHo, self.l2.PWo, wl.T, None, device=device, in_nhwc=nhwc)
        self.winners = torch.empty((B, 1, 3), dtype=torch.int32, device=device)
        self.count = torch.empty((B,), dtype=torch.int32, device=device)
        n = int(snn.lib().snn_k_winners_workspace(B, s3.F, self.l3.Ho, self.l3.Wo))
        self.ws_kw = torch.empty(n, dtype=torch.uint8, device=device)
        self.decision = torch.empty((B,), dtype=torch.int32, device=device)
        self.reward = torch.empty((B,), dtype=torch.float32, device=device)

    @property
    def lat0(self):
        return self.lat0_buf.permute(0, 3, 1, 2) if self.nhwc else self.lat0_buf

    def encode(self, x: torch.Tensor):
        snn.encode(x, self.T, out=self.lat0_buf, ws=self.ws_enc, nhwc=self.nhwc)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        self.encode(x)
        a = self.l1(self.lat0_buf)
        a = self.l2(a)
        self.l3(a)
        snn.k_winners(self.l3.lat, self.l3.v, 1, 0, winners=self.winners, count=self.count, ws=self.ws_kw)
        snn.decide(self.winners, self.count, self.wl.convs[2].F, self.wl.extra["n_classes"], None,
                   decision=self.decision, reward=self.reward)
        return self.decision


class C5Net:
    """Throughput stress (configs[4]): encode -> conv+fire -> pool 2/2 -> inhibit -> kWTA(k16, r4).
    nhwc: encode and conv write channels-last maps (the conv reads that layout); the pool reads the
    channels-last conv output and writes the planar map inhibition and k-WTA read."""

    def __init__(self, wl, B: int, device="cuda", nhwc: bool = True):
        self.wl, self.B, self.T = wl, B, wl.T
        _, C, H, W = wl.X.shape
        self.nhwc = nhwc
        self.ws_enc = torch.empty(snn.encode_workspace(B, C, H, W, wl.T), dtype=torch.uint8, device=device)
        self.lat0_buf = torch.empty((B, H, W, C) if nhwc else (B, C, H, W), dtype=torch.uint8, device=device)
        self.w = _dev(wl.weights[0], device)
        self.l1 = Layer(wl.convs[0], self.w, B, C, H, W, wl.T, wl.pools[0], pool_v=True, device=device, nhwc=nhwc,
                        in_nhwc=nhwc)
        F, Hp, Wp = wl.convs[0].F, self.l1.PHo, self.l1.PWo
        self.ilat = torch.empty((B, F, Hp, Wp), dtype=torch.uint8, device=device)
        self.iv = torch.empty((B, F, Hp, Wp), dtype=torch.float32, device=device)
        self.wf = torch.empty((B, Hp, Wp), dtype=torch.int16, device=device)
        k = wl.extra["k"]
        self.winners = torch.empty((B, k, 3), dtype=torch.int32, device=device)
        self.count = torch.empty((B,), dtype=torch.int32, device=device)
        self.ws_kw = torch.empty(int(snn.lib().snn_k_winners_workspace(B, F, Hp, Wp)), dtype=torch.uint8,
                                 device=device)

    @property
    def lat0(self):
        return self.lat0_buf.permute(0, 3, 1, 2) if self.nhwc else self.lat0_buf

    def encode(self, x: torch.Tensor):
        snn.encode(x, self.T, out=self.lat0_buf, ws=self.ws_enc, nhwc=self.nhwc)

    def forward(self, x: torch.Tensor):
        self.encode(x)
        self.l1(self.lat0_buf)
        snn.inhibit(self.l1.plat, self.l1.pv, lat_out=self.ilat, v_out=self.iv, winner_f=self.wf)
        snn.k_winners(self.ilat, self.iv, self.wl.extra["k"], self.wl.extra["r"], winners=self.winners,
                      count=self.count, ws=self.ws_kw)
        return self.winners, self.count


class SeqSTDP:
    """Sequential per-image plasticity on one conv layer (C1, C3: STDP; C4: R-STDP).

    ``lat_in`` [N, C, H, W] is the layer's (already computed, fixed-weight) input for every image.
    Per image: conv+fire -> [inhibit] -> kWTA -> [decide] -> STDP, all on the device.
    """

    def __init__(self, spec, w0: np.ndarray, C: int, H: int, W: int, T: int, k: int, r: int, inhibit: bool,
                 rates: Dict, n_classes: int = 0, device="cuda"):
        self.spec, self.T, self.k, self.r, self.inhibit_on = spec, T, k, r, inhibit
        self.rates, self.n_classes = rates, n_classes
        self.w = _dev(w0, device).clone()
        self.layer = Layer(spec, self.w, 1, C, H, W, T, None, device=device)
        F, Ho, Wo = spec.F, self.layer.Ho, self.layer.Wo
        self.ilat = torch.empty((1, F, Ho, Wo), dtype=torch.uint8, device=device)
        self.iv = torch.empty((1, F, Ho, Wo), dtype=torch.float32, device=device)
        self.wf = torch.empty((1, Ho, Wo), dtype=torch.int16, device=device)
        self.winners = torch.empty((1, k, 3), dtype=torch.int32, device=device)
        self.count = torch.empty((1,), dtype=torch.int32, device=device)
        self.ws_kw = torch.empty(int(snn.lib().snn_k_winners_workspace(1, F, Ho, Wo)), dtype=torch.uint8,
                                 device=device)
        self.decision = torch.empty((1,), dtype=torch.int32, device=device)
        self.reward = torch.ones((1,), dtype=torch.float32, device=device)

    def step(self, lat_in_img: torch.Tensor, label: Optional[torch.Tensor] = None, prep=None, b: int = 0):
        """lat_in_img [1, C, H, W]; label int32 [1] device tensor (R-STDP) or None (plain STDP).
        prep: for a theta = +inf layer, the batch's A operands (snn_conv_inf_prepare), image index b."""
        if prep is not None:
            L = self.layer
            snn.conv_fire_prepared(prep, b, L.C, L.H, L.W, self.w, self.spec.pad, self.T, lat_out=L.lat, v_out=L.v,
                                   ws=L.ws)
        else:
            self.layer(lat_in_img, self.w)
        lat, v = self.layer.lat, self.layer.v
        if self.inhibit_on:
            snn.inhibit(lat, v, lat_out=self.ilat, v_out=self.iv, winner_f=self.wf)
            lat_k, v_k = self.ilat, self.iv
        else:
            lat_k, v_k = lat, v
        snn.k_winners(lat_k, v_k, self.k, self.r, winners=self.winners, count=self.count, ws=self.ws_kw)
        reward = None
        if label is not None:
            snn.decide(self.winners, self.count, self.spec.F, self.n_classes, label, decision=self.decision,
                       reward=self.reward)
            reward = self.reward
        R = self.rates
        snn.stdp_update(self.w, lat_in_img[0], self.spec.pad, lat[0], self.winners[0], self.count, R["a_plus"],
                        R["a_minus"], R["lb"], R["ub"], R["stabilizer"], reward)


class SeqGraph:
    """A CUDA graph of n sequential plasticity steps: one kernel chain per image, replayed without any
    host synchronisation (the paper's residual per-image CPU-GPU interaction, removed).

    ``replay()`` restores the initial weights first, so every replay is one training pass over the
    same n images.  ``snapshot_every`` adds device copies of the weights after every that many images.
    """

    def __init__(self, seq: "SeqSTDP", lat_in_all: torch.Tensor, n: int, labels: Optional[torch.Tensor] = None,
                 snapshot_every: int = 0, prep: Optional[torch.Tensor] = None):
        """prep: A operands of lat_in_all for a theta = +inf layer (snn_conv_inf_prepare), refreshed by the
        caller before each replay whenever lat_in_all changes."""
        self.seq, self.lat, self.n, self.labels, self.prep = seq, lat_in_all, n, labels, prep
        self.w0 = seq.w.clone()
        self.snaps = [torch.empty_like(seq.w) for _ in range(n // snapshot_every)] if snapshot_every else []
        self.every = snapshot_every
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):          # warm-up outside capture (lazy attribute setup)
            self._body(1)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.seq.w.copy_(self.w0)
        self.graph = torch.cuda.CUDAGraph()
        c0 = snn.launch_count()
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            self.seq.w.copy_(self.w0)
            self._body(n)
        self.launches = snn.launch_count() - c0  # libsnn kernel nodes per replay

    def _body(self, n: int):
        si = 0
        for b in range(n):
            lab = None if self.labels is None else self.labels[b:b + 1]
            self.seq.step(self.lat[b:b + 1], lab, prep=self.prep, b=b)
            if self.every and (b + 1) % self.every == 0 and si < len(self.snaps):
                self.snaps[si].copy_(self.seq.w)
                si += 1

    def replay(self):
        self.graph.replay()


class SeqPersistent:
    """All n sequential plasticity steps of one conv layer (conv+fire -> inhibit -> k-WTA -> STDP) in
    one persistent kernel (snn_stdp_sequence).  ``replay()`` restores the initial
    weights first, so every replay is one training pass over the same n images (like SeqGraph)."""

    def __init__(self, spec, w0, lat_in_all: torch.Tensor, T: int, k: int, r: int, rates: Dict,
                 snapshot_every: int = 0, device="cuda"):
        self.spec, self.T, self.k, self.r, self.rates = spec, T, k, r, rates
        self.w = _dev(w0, device).clone()
        self.w0 = self.w.clone()
        self.lat = lat_in_all.contiguous()
        n = self.lat.shape[0]
        self.every = snapshot_every
        self.snaps = (torch.empty((n // snapshot_every,) + tuple(self.w.shape), dtype=torch.float32, device=device)
                      if snapshot_every else None)
        self.winners = torch.empty((n, k, 3), dtype=torch.int32, device=device)
        self.count = torch.empty((n,), dtype=torch.int32, device=device)
        N, C, H, W = self.lat.shape
        F, _, KH, KW = self.w.shape
        nb = int(snn.lib().snn_stdp_sequence_workspace(N, C, H, W, spec.pad, F, KH, KW, T, k))
        self.ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=device)
        self.launches = 0  # replay() launches through libsnn (counted by snn_launch_count itself)

    @staticmethod
    def supported(spec, lat_shape, w_shape, T: int, k: int) -> bool:
        N, C, H, W = lat_shape
        F, _, KH, KW = w_shape
        return not math.isinf(spec.theta) and \
            int(snn.lib().snn_stdp_sequence_workspace(N, C, H, W, spec.pad, F, KH, KW, T, k)) > 0

    def run(self):
        R = self.rates
        snn.stdp_sequence(self.lat, self.w, self.spec.pad, self.T, self.spec.theta, self.k, self.r, R["a_plus"],
                          R["a_minus"], R["lb"], R["ub"], R["stabilizer"], winners=self.winners, count=self.count,
                          snapshots=self.snaps, snap_every=self.every, ws=self.ws)

    def replay(self):
        self.w.copy_(self.w0)
        self.run()


class SeqInfRSTDP:
    """f1 for a theta = +inf plastic layer (C4's R-STDP layer): all n images' chains -- conv (Eq. 5,
    tcgen05) -> 1 winner -> decision -> R-STDP -- through snn_rstdp_inf_sequence, two kernels per image
    (GEMM, tail CTA) and no host synchronisation.  ``replay()`` restores the initial weights first."""

    def __init__(self, spec, w0, lat_in_all: torch.Tensor, prep: torch.Tensor, labels: torch.Tensor, T: int,
                 n_classes: int, rates: Dict, device="cuda"):
        self.spec, self.T, self.n_classes, self.rates = spec, T, n_classes, rates
        self.w = _dev(w0, device).clone()
        self.w0 = self.w.clone()
        self.lat, self.prep, self.labels = lat_in_all, prep, labels
        n, C, H, W = lat_in_all.shape
        F, _, KH, KW = self.w.shape
        self.winners = torch.empty((n, 3), dtype=torch.int32, device=device)
        self.count = torch.empty((n,), dtype=torch.int32, device=device)
        self.decision = torch.empty((n,), dtype=torch.int32, device=device)
        self.reward = torch.empty((n,), dtype=torch.float32, device=device)
        nb = int(snn.lib().snn_rstdp_inf_workspace(C, H, W, spec.pad, F, KH, KW))
        self.ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=device)

    def run(self):
        R = self.rates
        snn.rstdp_inf_sequence(self.prep, 0, self.lat, self.w, self.spec.pad, self.T, self.labels, self.n_classes,
                               R["a_plus"], R["a_minus"], R["lb"], R["ub"], R["stabilizer"], winners=self.winners,
                               count=self.count, decision=self.decision, reward=self.reward, ws=self.ws)

    def replay(self):
        self.w.copy_(self.w0)
        self.run()


class StepGraph:
    """CUDA graph of one fixed sequence of libsnn calls (``fn``) on preallocated buffers."""

    def __init__(self, fn):
        self.fn = fn
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        c0 = snn.launch_count()
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            fn()
        self.launches = snn.launch_count() - c0  # libsnn kernel nodes per replay

    def replay(self):
        self.graph.replay()
