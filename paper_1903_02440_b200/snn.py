"""Thin Python binding of libsnn (include/snn.h): ctypes marshalling of torch CUDA tensors only.

Every step of the spike-wave path runs in the library's sm_100a kernels; this module only checks
dtypes/devices/contiguity, allocates outputs and workspaces with torch (PyTorch is the device-memory
and stream plumbing), passes raw pointers, and raises ``SNNError`` on a non-zero return code.  There
is no CPU fallback: a missing library or a missing GPU raises.

Names follow the C ABI (``snn_<name>`` -> ``<name>``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from typing import Optional, Tuple

import torch

NO_SPIKE = 255
_LIB_PATH = os.environ.get("SNN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsnn.so")  # SNN_LIB: A/B experiments with another build
_lib = None
_lock = threading.Lock()

SNN_OK, SNN_EINVAL, SNN_ESHAPE, SNN_ECUDA, SNN_EINEXACT, SNN_EWORKSPACE = 0, -1, -2, -3, -4, -5


class SNNError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libsnn error {code}: {msg}")
        self.code = code


def lib() -> C.CDLL:
    """Load libsnn.so (raises if it has not been built: run __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise RuntimeError(f"{_LIB_PATH} missing: build it with `python -m paper_1903_02440_b200.build`")
            L = C.CDLL(_LIB_PATH)
            p, i32, f32, sz = C.c_void_p, C.c_int, C.c_float, C.c_size_t
            sigs = {
                "snn_version": (i32, []),
                "snn_last_error": (C.c_char_p, []),
                "snn_sync_status": (i32, [p]),
                "snn_encode_workspace": (sz, [i32, i32, i32, i32, i32]),
                "snn_encode": (i32, [p, i32, i32, i32, i32, i32, p, p, sz, p]),
                "snn_expand": (i32, [p, i32, i32, i32, p, p]),
                "snn_validate_lat": (i32, [p, sz, i32, p, p]),
                "snn_conv_fire_workspace": (sz, [i32] * 9 + [f32]),
                "snn_conv_fire": (i32, [p, i32, i32, i32, i32, i32, p, i32, i32, i32, i32, f32, p, p, p, p, sz, p]),
                "snn_rstdp_inf_workspace": (sz, [i32] * 7),
                "snn_rstdp_inf_sequence": (i32, [p, i32, i32, i32, i32, i32, i32, p, p, i32, i32, i32, i32, p, i32,
                                                 f32, f32, f32, f32, i32, p, p, p, p, p, sz, p]),
                "snn_conv_fire_ex": (i32, [p, i32, i32, i32, i32, i32, p, i32, i32, i32, i32, f32, i32, p, p, p, p, sz,
                                           p]),
                "snn_pool": (i32, [p, p, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, p, p, p]),
                "snn_pool_ex": (i32, [p, p] + [i32] * 11 + [p, p, p]),
                "snn_encode_ex": (i32, [p, i32, i32, i32, i32, i32, i32, p, p, sz, p]),
                "snn_conv_inf_prepare_bytes": (sz, [i32] * 8),
                "snn_conv_inf_prepare": (i32, [p] + [i32] * 9 + [p, sz, p]),
                "snn_conv_fire_prepared": (i32, [p, i32, i32, i32, i32, i32, p, i32, i32, i32, i32, p, p, p, sz, p]),
                "snn_position_keys": (i32, [p, p, i32, i32, i32, i32, i32, p, p]),
                "snn_k_winners_keys_workspace": (sz, [i32, i32, i32]),
                "snn_k_winners_keys": (i32, [p, i32, i32, i32, i32, i32, i32, p, p, p, sz, p]),
                "snn_stdp_update_shard": (i32, [p, i32, i32, i32, i32, i32, p, i32, i32, i32, p, i32, i32, p, p, i32,
                                                f32, f32, f32, f32, i32, p, p]),
                "snn_inhibit": (i32, [p, p, i32, i32, i32, i32, p, p, p, p]),
                "snn_k_winners_workspace": (sz, [i32, i32, i32, i32]),
                "snn_k_winners": (i32, [p, p, i32, i32, i32, i32, i32, i32, p, p, p, sz, p]),
                "snn_stdp_update": (i32, [p, i32, i32, i32, i32, p, i32, i32, i32, p, i32, i32, p, p, i32,
                                          f32, f32, f32, f32, i32, p, p]),
                "snn_decide": (i32, [p, p, i32, i32, i32, i32, p, p, p, p]),
                "snn_count_events": (i32, [p, i32, i32, i32, i32, i32, i32, i32, i32, i32, p, p, p]),
                "snn_launch_count": (C.c_ulonglong, []),
                "snn_filter_bank": (i32, [p, i32, i32, i32, p, i32, i32, i32, C.c_double, i32, p, p]),
                "snn_local_norm": (i32, [p, i32, i32, i32, i32, i32, C.c_double, p, p]),
                "snn_lateral_inhibition": (i32, [p, i32, i32, i32, i32, p, i32, p, p]),
                "snn_conv_fire_plan": (i32, [i32] * 9 + [f32, p, p, p]),
                "snn_stdp_sequence_workspace": (sz, [i32] * 10),
                "snn_stdp_sequence": (i32, [p, i32, i32, i32, i32, i32, p, i32, i32, i32, i32, f32, i32, i32,
                                            f32, f32, f32, f32, i32, p, p, p, i32, p, sz, p]),
            }
            for name, (res, args) in sigs.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def exported_symbols():
    return ["snn_version", "snn_last_error", "snn_sync_status", "snn_encode_workspace", "snn_encode",
            "snn_expand", "snn_validate_lat", "snn_conv_fire_workspace", "snn_conv_fire", "snn_pool",
            "snn_inhibit", "snn_k_winners_workspace", "snn_k_winners", "snn_stdp_update", "snn_decide",
            "snn_count_events", "snn_launch_count", "snn_conv_fire_plan", "snn_stdp_sequence_workspace",
            "snn_stdp_sequence", "snn_filter_bank", "snn_local_norm", "snn_lateral_inhibition",
            "snn_encode_ex", "snn_pool_ex", "snn_position_keys", "snn_k_winners_keys_workspace",
            "snn_k_winners_keys", "snn_stdp_update_shard", "snn_conv_inf_prepare_bytes", "snn_conv_inf_prepare",
            "snn_conv_fire_prepared", "snn_conv_fire_ex", "snn_rstdp_inf_workspace", "snn_rstdp_inf_sequence"]


def _check(rc: int):
    if rc != SNN_OK:
        raise SNNError(rc, lib().snn_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _req(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


class _Workspace:
    """Grow-only device scratch buffers, one per (device, tag, stream): calls on different streams never
    share scratch.  A buffer replaced by a larger one is released to torch's caching allocator; when it
    was used on a side stream, record_stream keeps it from being reused before that stream's work ends."""

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int, device, tag: str = "", stream=None) -> torch.Tensor:
        s = stream if stream is not None else torch.cuda.current_stream(device)
        key = (str(device), tag, s.cuda_stream)
        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            if stream is not None:
                b.record_stream(stream)
            self._bufs[key] = b
        return b


_ws = _Workspace()


# ------------------------------------------------------------------------------------------ a1
def encode_workspace(B, C_, H, W, T) -> int:
    return int(lib().snn_encode_workspace(B, C_, H, W, T))


ENCODE_OUT_NHWC = 0x100  # or'ed into snn_encode_ex's bins


def encode(x: torch.Tensor, T: int, out: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
           stream=None, bins: int = 0, nhwc: bool = False) -> torch.Tensor:
    """x float32 [B, C, H, W] -> lat uint8 [B, C, H, W] (snn_encode; bins != 0: snn_encode_ex variant);
    nhwc: lat channels-last [B, H, W, C] (SNN_ENCODE_OUT_NHWC)."""
    _req(x, torch.float32, "x")
    B, C_, H, W = x.shape
    shape = (B, H, W, C_) if nhwc else tuple(x.shape)
    lat = out if out is not None else torch.empty(shape, dtype=torch.uint8, device=x.device)
    _req(lat, torch.uint8, "lat")
    n = encode_workspace(B, C_, H, W, T)
    buf = ws if ws is not None else _ws.get(n, x.device, "encode", stream)
    if nhwc:
        bins |= ENCODE_OUT_NHWC
    if bins:
        _check(lib().snn_encode_ex(_ptr(x), B, C_, H, W, T, bins, _ptr(lat), _ptr(buf), buf.numel(),
                                   _stream(stream)))
    else:
        _check(lib().snn_encode(_ptr(x), B, C_, H, W, T, _ptr(lat), _ptr(buf), buf.numel(), _stream(stream)))
    return lat


def filter_bank(img: torch.Tensor, kernels: torch.Tensor, pad: int, mode: int = 0, threshold: float = float("-inf"),
                out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """img float64 [B, H, W], kernels float64 [K, S, S] -> float32 [B, Kout, Ho, Wo] (snn_filter_bank, R33)."""
    _req(img, torch.float64, "img")
    _req(kernels, torch.float64, "kernels")
    B, H, W = img.shape
    K, S, S2 = kernels.shape
    if S != S2:
        raise ValueError("kernels must be square")
    Ho, Wo = H + 2 * pad - S + 1, W + 2 * pad - S + 1
    shape = (B, 2 * K if mode == 1 else K, max(Ho, 0), max(Wo, 0))  # the C call rejects a bad shape
    o = out if out is not None else torch.empty(shape, dtype=torch.float32, device=img.device)
    _req(o, torch.float32, "out")
    _check(lib().snn_filter_bank(_ptr(img), B, H, W, _ptr(kernels), K, S, pad, float(threshold), mode, _ptr(o),
                                 _stream(stream)))
    return o


def local_norm(x: torch.Tensor, radius: int, eps: float = 1e-12, out: Optional[torch.Tensor] = None,
               stream=None) -> torch.Tensor:
    """x float32 [B, C, H, W] -> x / max(regional mean, eps) (snn_local_norm, R34)."""
    _req(x, torch.float32, "x")
    o = out if out is not None else torch.empty_like(x)
    _req(o, torch.float32, "out")
    _check(lib().snn_local_norm(_ptr(x), *x.shape, radius, float(eps), _ptr(o), _stream(stream)))
    return o


def lateral_inhibition(x: torch.Tensor, factors: torch.Tensor, out: Optional[torch.Tensor] = None,
                       stream=None) -> torch.Tensor:
    """x float32 [B, C, H, W], factors float32 [n] (device) -> inhibited intensities (snn_lateral_inhibition, R35)."""
    _req(x, torch.float32, "x")
    _req(factors, torch.float32, "factors")
    o = out if out is not None else torch.empty_like(x)
    _req(o, torch.float32, "out")
    _check(lib().snn_lateral_inhibition(_ptr(x), *x.shape, _ptr(factors), factors.numel(), _ptr(o), _stream(stream)))
    return o


def expand(lat: torch.Tensor, T: int, stream=None) -> torch.Tensor:
    """lat uint8 [B, ...] -> wave float32 [B, T, ...] (Eq. 1)."""
    _req(lat, torch.uint8, "lat")
    B = lat.shape[0]
    n = lat[0].numel() if B else 0
    wave = torch.empty((B, T) + tuple(lat.shape[1:]), dtype=torch.float32, device=lat.device)
    _check(lib().snn_expand(_ptr(lat), B, n, T, _ptr(wave), _stream(stream)))
    return wave


def validate_lat(lat: torch.Tensor, T: int, stream=None) -> int:
    _req(lat, torch.uint8, "lat")
    nb = torch.zeros(1, dtype=torch.int32, device=lat.device)
    _check(lib().snn_validate_lat(_ptr(lat), lat.numel(), T, _ptr(nb), _stream(stream)))
    return int(nb.item())


# ------------------------------------------------------------------------------------------ a2/a3
def conv_out_hw(H, W, KH, KW, pad):
    return H + 2 * pad - KH + 1, W + 2 * pad - KW + 1


def conv_fire_workspace(B, C_, H, W, pad, F, KH, KW, T, theta) -> int:
    return int(lib().snn_conv_fire_workspace(B, C_, H, W, pad, F, KH, KW, T, float(theta)))


CONV_OUT_NHWC, CONV_IN_NHWC, CONV_POOL2 = 1, 2, 4  # snn_conv_fire_ex flags


def conv_fire(lat_in: torch.Tensor, w: torch.Tensor, pad: int, T: int, theta: float, want_pot: bool = False,
              lat_out=None, v_out=None, ws=None, stream=None, nhwc: bool = False, want_v: bool = True,
              in_nhwc: bool = False, pool2: bool = False):
    """lat_in uint8 [B, C, H, W], w float32 [F, C, KH, KW] -> (lat uint8, v float32) [B, F, Ho, Wo]
    (+ pot float32 [B, T, F, Ho, Wo] when want_pot).  nhwc: outputs channels-last [B, Ho, Wo, F]
    (snn_conv_fire_ex SNN_CONV_OUT_NHWC); in_nhwc: lat_in is [B, H, W, C] (SNN_CONV_IN_NHWC);
    want_v False: v is not written (None returned).  pool2 (SNN_CONV_POOL2, with nhwc, in_nhwc and
    want_v False): lat is the 2 x 2 / stride 2 latency pooling [B, Ho // 2, Wo // 2, F] of the spike times."""
    _req(lat_in, torch.uint8, "lat_in")
    _req(w, torch.float32, "w")
    if in_nhwc:
        B, H, W, C_ = lat_in.shape
    else:
        B, C_, H, W = lat_in.shape
    F, Cw, KH, KW = w.shape
    if Cw != C_:
        raise ValueError("channel mismatch between lat_in and w")
    Ho, Wo = conv_out_hw(H, W, KH, KW, pad)
    Ho, Wo = max(Ho, 0), max(Wo, 0)          # invalid shapes are rejected by the library (SNN_ESHAPE)
    dev = lat_in.device
    shape = (B, Ho, Wo, F) if nhwc else (B, F, Ho, Wo)
    if pool2:
        shape = (B, Ho // 2, Wo // 2, F)
    lat = lat_out if lat_out is not None else torch.empty(shape, dtype=torch.uint8, device=dev)
    v = None
    if want_v:
        v = v_out if v_out is not None else torch.empty(shape, dtype=torch.float32, device=dev)
    pot = torch.empty((B, T, F, Ho, Wo), dtype=torch.float32, device=dev) if want_pot else None
    n = conv_fire_workspace(B, C_, H, W, pad, F, KH, KW, T, theta)
    buf = ws if ws is not None else _ws.get(n, dev, "conv", stream)
    _check(lib().snn_conv_fire_ex(_ptr(lat_in), B, C_, H, W, pad, _ptr(w), F, KH, KW, T, float(theta),
                                  (CONV_OUT_NHWC if nhwc else 0) | (CONV_IN_NHWC if in_nhwc else 0) |
                                  (CONV_POOL2 if pool2 else 0), _ptr(lat),
                                  _ptr(v), _ptr(pot), _ptr(buf), buf.numel(),
                                  _stream(stream)))
    return (lat, v, pot) if want_pot else (lat, v)


def conv_inf_prepare(lat_in: torch.Tensor, F: int, KH: int, KW: int, pad: int, T: int, out=None, stream=None):
    """A operands of every image of lat_in [B, C, H, W] for theta = +inf (snn_conv_inf_prepare)."""
    _req(lat_in, torch.uint8, "lat_in")
    B, C_, H, W = lat_in.shape
    n = int(lib().snn_conv_inf_prepare_bytes(B, C_, H, W, pad, F, KH, KW))
    buf = out if out is not None else torch.empty(max(n, 1), dtype=torch.uint8, device=lat_in.device)
    _check(lib().snn_conv_inf_prepare(_ptr(lat_in), B, C_, H, W, pad, F, KH, KW, T, _ptr(buf), buf.numel(),
                                      _stream(stream)))
    return buf


def conv_fire_prepared(prep: torch.Tensor, b: int, C_: int, H: int, W: int, w: torch.Tensor, pad: int, T: int,
                       lat_out=None, v_out=None, ws=None, stream=None):
    """theta = +inf conv of image b of a snn_conv_inf_prepare batch with weights w (snn_conv_fire_prepared)."""
    _req(w, torch.float32, "w")
    F, _, KH, KW = w.shape
    Ho, Wo = conv_out_hw(H, W, KH, KW, pad)
    dev = w.device
    lat = lat_out if lat_out is not None else torch.empty((1, F, Ho, Wo), dtype=torch.uint8, device=dev)
    v = v_out if v_out is not None else torch.empty((1, F, Ho, Wo), dtype=torch.float32, device=dev)
    n = conv_fire_workspace(1, C_, H, W, pad, F, KH, KW, T, float("inf"))
    buf = ws if ws is not None else _ws.get(n, dev, "conv", stream)
    _check(lib().snn_conv_fire_prepared(_ptr(prep), int(b), C_, H, W, pad, _ptr(w), F, KH, KW, T, _ptr(lat), _ptr(v),
                                        _ptr(buf), buf.numel(), _stream(stream)))
    return lat, v


def rstdp_inf_sequence(prep: torch.Tensor, b0: int, lat_in: torch.Tensor, w: torch.Tensor, pad: int, T: int,
                       labels: Optional[torch.Tensor], n_classes: int, a_plus: float, a_minus: float, lb: float = 0.0,
                       ub: float = 1.0, stabilizer: int = 1, winners=None, count=None, decision=None, reward=None,
                       ws=None, stream=None):
    """f1 theta = +inf R-STDP chain (snn_rstdp_inf_sequence): images b0 .. b0 + N - 1 of the prepared batch
    ``prep``; lat_in uint8 [N, C, H, W] their (planar) layer input; w fp32 [F, C, KH, KW] updated in place.
    Returns (winners [N, 3], count [N], decision [N], reward [N])."""
    _req(lat_in, torch.uint8, "lat_in")
    _req(w, torch.float32, "w")
    N, C_, H, W = lat_in.shape
    F, _, KH, KW = w.shape
    dev = w.device
    win = winners if winners is not None else torch.empty((N, 3), dtype=torch.int32, device=dev)
    cnt = count if count is not None else torch.empty((N,), dtype=torch.int32, device=dev)
    dec = decision if decision is not None else torch.empty((N,), dtype=torch.int32, device=dev)
    rw = reward if reward is not None else torch.empty((N,), dtype=torch.float32, device=dev)
    n = int(lib().snn_rstdp_inf_workspace(C_, H, W, pad, F, KH, KW))
    buf = ws if ws is not None else _ws.get(n, dev, "rstdp_inf", stream)
    _check(lib().snn_rstdp_inf_sequence(_ptr(prep), int(b0), N, C_, H, W, pad, _ptr(lat_in), _ptr(w), F, KH, KW, T,
                                        _ptr(labels), int(n_classes), float(a_plus), float(a_minus), float(lb),
                                        float(ub), int(stabilizer), _ptr(win), _ptr(cnt), _ptr(dec), _ptr(rw),
                                        _ptr(buf), buf.numel(), _stream(stream)))
    return win, cnt, dec, rw


# ------------------------------------------------------------------------------------------ a4
def pool_out_hw(H, W, PH, PW, SH, SW, DH=0, DW=0, eq3=False):
    if eq3:  # Eq. 3 literally (snn_pool_ex SNN_POOL_EQ3)
        return (H + 2 * DH) // SH, (W + 2 * DW) // SW
    return (H + 2 * DH - PH) // SH + 1, (W + 2 * DW - PW) // SW + 1


POOL_EQ3, POOL_VFINAL, POOL_IN_NHWC, POOL_OUT_NHWC = 1, 2, 4, 8  # snn_pool_ex flags (f3 variants; layouts)


def pool(lat: torch.Tensor, v: Optional[torch.Tensor], window, stride=None, padding=(0, 0),
         lat_out=None, v_out=None, stream=None, flags: int = 0):
    _req(lat, torch.uint8, "lat")
    if v is not None:
        _req(v, torch.float32, "v")
    PH, PW = (window, window) if isinstance(window, int) else window
    SH, SW = (PH, PW) if stride is None else ((stride, stride) if isinstance(stride, int) else stride)
    DH, DW = (padding, padding) if isinstance(padding, int) else padding
    if flags & POOL_IN_NHWC:
        B, H, W, F = lat.shape
    else:
        B, F, H, W = lat.shape
    Ho, Wo = (max(d, 0) for d in pool_out_hw(H, W, PH, PW, SH, SW, DH, DW, bool(flags & POOL_EQ3)))
    oshape = (B, Ho, Wo, F) if flags & POOL_OUT_NHWC else (B, F, Ho, Wo)
    lo = lat_out if lat_out is not None else torch.empty(oshape, dtype=torch.uint8, device=lat.device)
    vo = None
    if v is not None:
        vo = v_out if v_out is not None else torch.empty(oshape, dtype=torch.float32, device=lat.device)
    if flags:
        _check(lib().snn_pool_ex(_ptr(lat), _ptr(v), B, F, H, W, PH, PW, SH, SW, DH, DW, flags, _ptr(lo), _ptr(vo),
                                 _stream(stream)))
    else:
        _check(lib().snn_pool(_ptr(lat), _ptr(v), B, F, H, W, PH, PW, SH, SW, DH, DW, _ptr(lo), _ptr(vo),
                              _stream(stream)))
    return lo, vo


# ------------------------------------------------------------------------------------------ a5
def inhibit(lat: torch.Tensor, v: torch.Tensor, lat_out=None, v_out=None, winner_f=None, stream=None):
    _req(lat, torch.uint8, "lat")
    _req(v, torch.float32, "v")
    B, F, H, W = lat.shape
    lo = lat_out if lat_out is not None else torch.empty_like(lat)
    vo = v_out if v_out is not None else torch.empty_like(v)
    wf = winner_f if winner_f is not None else torch.empty((B, H, W), dtype=torch.int16, device=lat.device)
    _check(lib().snn_inhibit(_ptr(lat), _ptr(v), B, F, H, W, _ptr(lo), _ptr(vo), _ptr(wf), _stream(stream)))
    return lo, vo, wf


# ------------------------------------------------------------------------------------------ a6
def k_winners(lat: torch.Tensor, v: torch.Tensor, k: int, r: int, winners=None, count=None, ws=None, stream=None):
    _req(lat, torch.uint8, "lat")
    _req(v, torch.float32, "v")
    B, F, H, W = lat.shape
    win = winners if winners is not None else torch.empty((B, k, 3), dtype=torch.int32, device=lat.device)
    cnt = count if count is not None else torch.empty((B,), dtype=torch.int32, device=lat.device)
    n = int(lib().snn_k_winners_workspace(B, F, H, W))
    buf = ws if ws is not None else _ws.get(n, lat.device, "kwta", stream)
    _check(lib().snn_k_winners(_ptr(lat), _ptr(v), B, F, H, W, k, r, _ptr(win), _ptr(cnt), _ptr(buf), buf.numel(),
                               _stream(stream)))
    return win, cnt


# ------------------------------------------------------------------------------------------ a7
def stdp_update(w: torch.Tensor, lat_in: torch.Tensor, pad: int, lat_out: torch.Tensor, winners: torch.Tensor,
                count: torch.Tensor, a_plus: float, a_minus: float, lb: float = 0.0, ub: float = 1.0,
                stabilizer: int = 1, reward: Optional[torch.Tensor] = None, stream=None,
                f_offset: Optional[int] = None) -> torch.Tensor:
    """In-place update of w [F, C, KH, KW] for one image: lat_in [C, H, W], lat_out [F, Ho, Wo],
    winners [k, 3], count [1] (device), reward float32 [1] (device, +1 / -1 / 0) or None (= +1)."""
    _req(w, torch.float32, "w")
    _req(lat_in, torch.uint8, "lat_in")
    _req(lat_out, torch.uint8, "lat_out")
    _req(winners, torch.int32, "winners")
    _req(count, torch.int32, "count")
    if reward is not None:
        _req(reward, torch.float32, "reward")
    F, C_, KH, KW = w.shape
    _, H, W = lat_in.shape
    _, Ho, Wo = lat_out.shape
    k = winners.shape[-2]
    if f_offset is not None:  # f4: w holds the features [f_offset, f_offset + F) of the layer
        _check(lib().snn_stdp_update_shard(_ptr(w), F, int(f_offset), C_, KH, KW, _ptr(lat_in), H, W, pad,
                                           _ptr(lat_out), Ho, Wo, _ptr(winners), _ptr(count), k, float(a_plus),
                                           float(a_minus), float(lb), float(ub), int(stabilizer), _ptr(reward),
                                           _stream(stream)))
        return w
    _check(lib().snn_stdp_update(_ptr(w), F, C_, KH, KW, _ptr(lat_in), H, W, pad, _ptr(lat_out), Ho, Wo,
                                 _ptr(winners), _ptr(count), k, float(a_plus), float(a_minus), float(lb), float(ub),
                                 int(stabilizer), _ptr(reward), _stream(stream)))
    return w


# ------------------------------------------------------------------------------------------ f4
KEY_NONE = (1 << 63) - 1  # SNN_KEY_NONE


def position_keys(lat: torch.Tensor, v: torch.Tensor, f_offset: int = 0, out=None, stream=None) -> torch.Tensor:
    """lat/v [B, F, H, W] of the rank's features -> int64 [B, H, W] min packed key (snn_position_keys)."""
    _req(lat, torch.uint8, "lat")
    _req(v, torch.float32, "v")
    B, F, H, W = lat.shape
    keys = out if out is not None else torch.empty((B, H, W), dtype=torch.int64, device=lat.device)
    _req(keys, torch.int64, "keys")
    _check(lib().snn_position_keys(_ptr(lat), _ptr(v), B, F, H, W, int(f_offset), _ptr(keys), _stream(stream)))
    return keys


def k_winners_keys(keys: torch.Tensor, F: int, k: int, r: int, winners=None, count=None, ws=None, stream=None):
    """k-WTA on the inhibited map given by reduced position keys [B, H, W] (snn_k_winners_keys)."""
    _req(keys, torch.int64, "keys")
    B, H, W = keys.shape
    win = winners if winners is not None else torch.empty((B, k, 3), dtype=torch.int32, device=keys.device)
    cnt = count if count is not None else torch.empty((B,), dtype=torch.int32, device=keys.device)
    n = int(lib().snn_k_winners_keys_workspace(B, H, W))
    buf = ws if ws is not None else _ws.get(n, keys.device, "kwta_keys", stream)
    _check(lib().snn_k_winners_keys(_ptr(keys), B, int(F), H, W, k, r, _ptr(win), _ptr(cnt), _ptr(buf), buf.numel(),
                                    _stream(stream)))
    return win, cnt


def decide(winners: torch.Tensor, count: torch.Tensor, F: int, n_classes: int, labels: Optional[torch.Tensor] = None,
           decision=None, reward=None, stream=None):
    _req(winners, torch.int32, "winners")
    _req(count, torch.int32, "count")
    B, k, _ = winners.shape
    d = decision if decision is not None else torch.empty((B,), dtype=torch.int32, device=winners.device)
    rw = reward if reward is not None else torch.empty((B,), dtype=torch.float32, device=winners.device)
    _check(lib().snn_decide(_ptr(winners), _ptr(count), B, k, F, n_classes, _ptr(labels), _ptr(d), _ptr(rw),
                            _stream(stream)))
    return d, rw


def count_events(lat_in: torch.Tensor, F: int, KH: int, KW: int, pad: int, T: int,
                 lat_out: Optional[torch.Tensor] = None, stream=None) -> Tuple[int, int]:
    """(paper-definition synaptic events, necessary events) of one conv layer (snn_count_events)."""
    _req(lat_in, torch.uint8, "lat_in")
    B, C_, H, W = lat_in.shape
    out = torch.zeros(2, dtype=torch.int64, device=lat_in.device)
    _check(lib().snn_count_events(_ptr(lat_in), B, C_, H, W, pad, F, KH, KW, T, _ptr(lat_out), _ptr(out),
                                  _stream(stream)))
    o = out.cpu().tolist()
    return int(o[0]), int(o[1])


def conv_fire_plan(B: int, Cin: int, H: int, W: int, pad: int, F: int, KH: int, KW: int, T: int,
                   theta: float) -> dict:
    """What one conv_fire call launches (snn_conv_fire_plan): path, kernel launches, list chunks."""
    path, launches, chunks = C.c_int(), C.c_int(), C.c_int()
    _check(lib().snn_conv_fire_plan(B, Cin, H, W, pad, F, KH, KW, T, theta, C.byref(path), C.byref(launches),
                                    C.byref(chunks)))
    names = {0: "walk_fused", 1: "walk_presorted", 2: "tc_inf", 3: "tct", 4: "ref", 5: "walk_presorted_global"}
    return {"path": names[path.value], "launches": launches.value, "chunks": chunks.value}


def stdp_sequence(lat_in: torch.Tensor, w: torch.Tensor, pad: int, T: int, theta: float, k: int, r: int,
                  a_plus: float, a_minus: float, lb: float = 0.0, ub: float = 1.0, stabilizer: int = 1,
                  winners: Optional[torch.Tensor] = None, count: Optional[torch.Tensor] = None,
                  snapshots: Optional[torch.Tensor] = None, snap_every: int = 0, ws: Optional[torch.Tensor] = None,
                  stream=None):
    """N sequential conv+fire -> inhibit -> k-WTA -> STDP steps in one persistent kernel (w in place)."""
    _req(lat_in, torch.uint8, "lat_in")
    _req(w, torch.float32, "w")
    N, Cin, H, W = lat_in.shape
    F, _, KH, KW = w.shape
    dev = lat_in.device
    if winners is None:
        winners = torch.empty((N, k, 3), dtype=torch.int32, device=dev)
    if count is None:
        count = torch.empty((N,), dtype=torch.int32, device=dev)
    if ws is None:
        n = int(lib().snn_stdp_sequence_workspace(N, Cin, H, W, pad, F, KH, KW, T, k))
        if n == 0:
            raise SNNError(SNN_ESHAPE, "snn_stdp_sequence: layer not supported")
        ws = torch.empty(n, dtype=torch.uint8, device=dev)
    _check(lib().snn_stdp_sequence(_ptr(lat_in), N, Cin, H, W, pad, _ptr(w), F, KH, KW, T, theta, k, r, a_plus,
                                   a_minus, lb, ub, stabilizer, _ptr(winners), _ptr(count), _ptr(snapshots),
                                   snap_every, _ptr(ws), ws.numel(), _stream(stream)))
    return winners, count


def launch_count() -> int:
    return int(lib().snn_launch_count())


def sync_status(stream=None) -> None:
    _check(lib().snn_sync_status(_stream(stream)))


def version() -> int:
    return int(lib().snn_version())
