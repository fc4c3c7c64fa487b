"""CPU oracle for the spike-wave hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1903_02440_b200``) never imports it and shares no code with it.

The arithmetic lives in ``snn_oracle.c`` (plain loops, one function per paper
step, each citing PAPER.md).  This module compiles it with gcc on first use and
wraps it with numpy marshalling only.  Every function is pinned by
``tests/test_oracle_*.py`` against worked examples, closed forms, brute force
and library routines.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import threading

import numpy as np

NO_SPIKE = 255          # P:51 "infinity stands for no spike" (oracle's own constant)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "snn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile snn_oracle.c -> liboracle.so (gcc, no FMA contraction, OpenMP over images)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            p = C.c_void_p
            i64, i32, f32 = C.c_int64, C.c_int, C.c_float
            sig = {
                "orc_pool_ex": (None, [p, p, i64, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, p, p]),
                "orc_encode_bins": (None, [p, i64, i64, i32, i32, p]),
                "orc_filter_bank": (None, [p, i64, i32, i32, p, i32, i32, i32, C.c_double, i32, p]),
                "orc_local_norm": (None, [p, i64, i32, i32, i32, i32, C.c_double, p]),
                "orc_lateral_inhibition": (None, [p, i64, i32, i32, i32, p, i32, p]),
                "orc_encode": (None, [p, i64, i64, i32, p]),
                "orc_expand": (None, [p, i64, i64, i32, p]),
                "orc_potentials": (None, [p, i32, i32, i32, i32, p, i32, i32, i32, i32, p]),
                "orc_potentials_brute": (None, [p, i32, i32, i32, i32, p, i32, i32, i32, i32, p]),
                "orc_fire": (None, [p, i32, i64, f32, i32, p, p]),
                "orc_conv_fire": (None, [p, i64, i32, i32, i32, i32, p, i32, i32, i32, i32, f32, i32, p, p]),
                "orc_conv_fire_sample": (None, [p, i32, i32, i32, i32, p, i32, i32, i32, i32, f32, i32,
                                                p, i64, p, p, p]),
                "orc_events": (i64, [p, i64, i32, i32, i32, i32, i32, i32, i32]),
                "orc_pool": (None, [p, p, i64, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, p, p]),
                "orc_inhibit": (None, [p, p, i64, i32, i32, i32, p, p, p]),
                "orc_k_winners_batch": (None, [p, p, i64, i32, i32, i32, i32, i32, p, p]),
                "orc_stdp": (None, [p, i32, i32, i32, i32, p, i32, i32, i32, p, i32, i32, p, i32,
                                    f32, f32, f32, f32, i32, i32]),
                "orc_decide": (i32, [p, i32, i32, i32, i32, C.POINTER(C.c_int)]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def set_threads(n: int) -> None:
    os.environ["OMP_NUM_THREADS"] = str(n)


# ----------------------------------------------------------------------------- a1
def encode(x: np.ndarray, T: int, bins: int = 0) -> np.ndarray:
    """x fp32 [B, C, H, W] (or [B, n]) -> lat uint8 same shape; bins = bin-size rule (orc_encode_bins)."""
    x = _c(x, np.float32)
    B = x.shape[0]
    n = int(np.prod(x.shape[1:])) if x.ndim > 1 else 0
    lat = np.empty(x.shape, dtype=np.uint8)
    lib().orc_encode_bins(_ptr(x), B, n, T, int(bins), _ptr(lat))
    return lat


def expand(lat: np.ndarray, T: int) -> np.ndarray:
    """lat uint8 [B, ...] -> wave fp32 [B, T, ...] (Eq. 1)."""
    lat = _c(lat, np.uint8)
    B = lat.shape[0]
    n = int(np.prod(lat.shape[1:]))
    wave = np.empty((B, T) + lat.shape[1:], dtype=np.float32)
    lib().orc_expand(_ptr(lat), B, n, T, _ptr(wave))
    return wave


# ----------------------------------------------------------------------------- a2/a3
def out_hw(H: int, W: int, KH: int, KW: int, pad: int):
    """Eq. 2 on the padded input."""
    return H + 2 * pad - KH + 1, W + 2 * pad - KW + 1


def potentials(lat_in: np.ndarray, w: np.ndarray, pad: int, T: int, brute: bool = False) -> np.ndarray:
    """One image: lat_in uint8 [C, H, W], w fp32 [F, C, KH, KW] -> P fp64 [T, F, Ho, Wo]."""
    lat_in = _c(lat_in, np.uint8)
    w = _c(w, np.float32)
    Cc, H, W = lat_in.shape
    F, Cw, KH, KW = w.shape
    assert Cw == Cc
    Ho, Wo = out_hw(H, W, KH, KW, pad)
    P = np.empty((T, F, Ho, Wo), dtype=np.float64)
    fn = lib().orc_potentials_brute if brute else lib().orc_potentials
    fn(_ptr(lat_in), Cc, H, W, pad, _ptr(w), F, KH, KW, T, _ptr(P))
    return P


def fire(P: np.ndarray, theta: float):
    """P fp64 [T, ...] -> (lat uint8 [...], v fp32 [...]).  theta = inf => Eq. 5."""
    P = _c(P, np.float64)
    T = P.shape[0]
    n = int(np.prod(P.shape[1:]))
    lat = np.empty(P.shape[1:], dtype=np.uint8)
    v = np.empty(P.shape[1:], dtype=np.float32)
    inf = math.isinf(theta)
    lib().orc_fire(_ptr(P), T, n, 0.0 if inf else float(theta), int(inf), _ptr(lat), _ptr(v))
    return lat, v


def conv_fire(lat_in: np.ndarray, w: np.ndarray, pad: int, T: int, theta: float):
    """Batch: lat_in uint8 [B, C, H, W] -> (lat uint8 [B, F, Ho, Wo], v fp32 [B, F, Ho, Wo])."""
    lat_in = _c(lat_in, np.uint8)
    w = _c(w, np.float32)
    B, Cc, H, W = lat_in.shape
    F, Cw, KH, KW = w.shape
    assert Cw == Cc
    Ho, Wo = out_hw(H, W, KH, KW, pad)
    lat = np.empty((B, F, Ho, Wo), dtype=np.uint8)
    v = np.empty((B, F, Ho, Wo), dtype=np.float32)
    inf = math.isinf(theta)
    lib().orc_conv_fire(_ptr(lat_in), B, Cc, H, W, pad, _ptr(w), F, KH, KW, T,
                        0.0 if inf else float(theta), int(inf), _ptr(lat), _ptr(v))
    return lat, v


def conv_fire_sample(lat_in: np.ndarray, w: np.ndarray, pad: int, T: int, theta: float,
                     neurons: np.ndarray, want_p: bool = False):
    """Sampled neurons (flat indices into [B, F, Ho, Wo]) -> (lat, v[, P fp64 [n, T]])."""
    lat_in = _c(lat_in, np.uint8)
    w = _c(w, np.float32)
    neurons = _c(neurons, np.int64)
    B, Cc, H, W = lat_in.shape
    F, _, KH, KW = w.shape
    n = neurons.shape[0]
    lat = np.empty(n, dtype=np.uint8)
    v = np.empty(n, dtype=np.float32)
    P = np.empty((n, T), dtype=np.float64) if want_p else None
    inf = math.isinf(theta)
    lib().orc_conv_fire_sample(_ptr(lat_in), Cc, H, W, pad, _ptr(w), F, KH, KW, T,
                               0.0 if inf else float(theta), int(inf), _ptr(neurons), n,
                               _ptr(lat), _ptr(v), _ptr(P))
    return (lat, v, P) if want_p else (lat, v)


def events(lat_in: np.ndarray, F: int, KH: int, KW: int, pad: int) -> int:
    lat_in = _c(lat_in, np.uint8)
    B, Cc, H, W = lat_in.shape
    return int(lib().orc_events(_ptr(lat_in), B, Cc, H, W, pad, F, KH, KW))


# ----------------------------------------------------------------------------- a4
def pool_out_hw(H, W, PH, PW, SH, SW, DH=0, DW=0, eq3=False):
    """Reading R10: windows fully inside the padded input; eq3: Eq. 3 literally (f3 variant)."""
    if eq3:
        return (H + 2 * DH) // SH, (W + 2 * DW) // SW
    return (H + 2 * DH - PH) // SH + 1, (W + 2 * DW - PW) // SW + 1


def pool(lat: np.ndarray, v, PH, PW, SH, SW, DH=0, DW=0, T=254, eq3=False, vfinal=False):
    lat = _c(lat, np.uint8)
    B, F, H, W = lat.shape
    v = None if v is None else _c(v, np.float32)
    Ho, Wo = pool_out_hw(H, W, PH, PW, SH, SW, DH, DW, eq3)
    lo = np.empty((B, F, Ho, Wo), dtype=np.uint8)
    vo = np.empty((B, F, Ho, Wo), dtype=np.float32) if v is not None else None
    lib().orc_pool_ex(_ptr(lat), _ptr(v), B, F, H, W, PH, PW, SH, SW, DH, DW, T, int(eq3), int(vfinal),
                      _ptr(lo), _ptr(vo))
    return lo, vo


# ----------------------------------------------------------------------------- a5
def inhibit(lat: np.ndarray, v: np.ndarray):
    lat = _c(lat, np.uint8)
    v = _c(v, np.float32)
    B, F, H, W = lat.shape
    lo = np.empty_like(lat)
    vo = np.empty_like(v)
    wf = np.empty((B, H, W), dtype=np.int16)
    lib().orc_inhibit(_ptr(lat), _ptr(v), B, F, H, W, _ptr(lo), _ptr(vo), _ptr(wf))
    return lo, vo, wf


# ----------------------------------------------------------------------------- a6
def k_winners(lat: np.ndarray, v: np.ndarray, k: int, r: int):
    """lat/v [B, F, H, W] -> (winners int32 [B, k, 3] (-1 padded), count int32 [B])."""
    lat = _c(lat, np.uint8)
    v = _c(v, np.float32)
    B, F, H, W = lat.shape
    win = np.empty((B, k, 3), dtype=np.int32)
    cnt = np.empty(B, dtype=np.int32)
    lib().orc_k_winners_batch(_ptr(lat), _ptr(v), B, F, H, W, k, r, _ptr(win), _ptr(cnt))
    return win, cnt


# ----------------------------------------------------------------------------- a7
def stdp(w: np.ndarray, lat_in: np.ndarray, pad: int, lat_out: np.ndarray, winners: np.ndarray,
         count: int, a_plus: float, a_minus: float, lb: float = 0.0, ub: float = 1.0,
         stabilizer: int = 1, reward: int = 1) -> np.ndarray:
    """One image.  w fp32 [F, C, KH, KW] is returned updated (copy)."""
    w = np.array(w, dtype=np.float32, order="C", copy=True)
    lat_in = _c(lat_in, np.uint8)
    lat_out = _c(lat_out, np.uint8)
    winners = _c(winners, np.int32).reshape(-1, 3)
    F, Cc, KH, KW = w.shape
    _, H, W = lat_in.shape
    _, Ho, Wo = lat_out.shape
    lib().orc_stdp(_ptr(w), F, Cc, KH, KW, _ptr(lat_in), H, W, pad, _ptr(lat_out), Ho, Wo,
                   _ptr(winners), int(count), float(a_plus), float(a_minus), float(lb), float(ub),
                   int(stabilizer), int(reward))
    return w


def decide(winners: np.ndarray, count: int, F: int, n_classes: int, label: int):
    winners = _c(winners, np.int32).reshape(-1, 3)
    d = C.c_int(0)
    rw = lib().orc_decide(_ptr(winners), int(count), F, n_classes, int(label), C.byref(d))
    return int(d.value), int(rw)


# ------------------------------------------------------------------------------ f2 front end
def filter_bank(img: np.ndarray, kernels: np.ndarray, pad: int, mode: int = 0,
                threshold: float = -math.inf) -> np.ndarray:
    """[B,H,W] fp64 images * [K,S,S] fp64 kernels -> fp32 [B,Kout,Ho,Wo] (R33; mode 0 thresholded,
    1 DoG on/off split, 2 rectified)."""
    img = np.ascontiguousarray(img, dtype=np.float64)
    ker = np.ascontiguousarray(kernels, dtype=np.float64)
    B, H, W = img.shape
    K, S, _ = ker.shape
    Ho, Wo = H + 2 * pad - S + 1, W + 2 * pad - S + 1
    out = np.zeros((B, 2 * K if mode == 1 else K, Ho, Wo), dtype=np.float32)
    lib().orc_filter_bank(_ptr(img), B, H, W, _ptr(ker), K, S, pad, float(threshold), mode, _ptr(out))
    return out


def local_norm(x: np.ndarray, radius: int, eps: float = 1e-12) -> np.ndarray:
    """x / max(regional mean, eps), border windows truncated (R34)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    B, Cc, H, W = x.shape
    out = np.empty_like(x)
    lib().orc_local_norm(_ptr(x), B, Cc, H, W, radius, float(eps), _ptr(out))
    return out


def lateral_inhibition(x: np.ndarray, factors) -> np.ndarray:
    """Intensity lateral inhibition, SPEC's descending-intensity sweep (R35)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    f = np.ascontiguousarray(np.asarray(factors, dtype=np.float32))
    B, Cc, H, W = x.shape
    out = np.empty_like(x)
    lib().orc_lateral_inhibition(_ptr(x), B, Cc, H, W, _ptr(f), len(f), _ptr(out))
    return out
