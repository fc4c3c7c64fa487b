// walk_dev.cuh -- device code of the delta walk shared by conv_walk.cu (the conv+fire kernels) and
// seq_train.cu (the persistent per-image plasticity chain): list layout constants, the receptive-field
// counting sort (K2), the monotone block test (K3) and the walk of one sorted list.  Product code.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace snn {

constexpr int kWalkSmemLimit = 227 * 1024;
constexpr size_t kListChunkBytes = size_t(512) << 20;  // sorted lists per chunk (measured: fewer, larger chunks win;
                                                        // the lists stream from HBM either way)
constexpr int kIt = 16;                               // list entries per walk iteration (lists padded to this)
constexpr int kListSlack = 2048;
// entries a sorted list can take: R spiking inputs, up to 3 pads per bucket, the tail padding and a
// partial last block's entry over-read (never gathered)
__host__ __device__ constexpr int list_cap(int R, int T) { return R + 3 * T + 2 * kIt; }
#ifndef SNN_SORT_UNROLL
#define SNN_SORT_UNROLL 4  // receptive-field entries per lane whose latency loads are in flight together
#endif
#ifndef SNN_SORT_BATCH
#define SNN_SORT_BATCH 0   // 1: each lane's latencies loaded in batches of kSortUnroll before their updates
#endif
constexpr int kSortUnroll = SNN_SORT_UNROLL;                      // bytes read past the last record (prefetch)

struct WalkArgs {
  const uint8_t* lat_in;
  int B, C, H, W, pad;
  int F, KH, KW, T, Ho, Wo, R;
  const uint32_t* wq;  // [n_groups][R+1][FGS]
  int64_t thr;        // threshold in units of 2^-31: floor(theta * 2^31) (saturated)
  int64_t thr28;      // the same in units of 2^-28 (walks of S28 weight slices)
  uint8_t* lat_out;
  float* v_out;
  int off_eoff, off_ekk, off_warps, warp_bytes, pos_bytes;
  int cnt_off, start_off, list_off;
  int row_bytes;      // bytes per weight row of the walk's slice (FGS * 4): list entries are row * row_bytes
  // presorted lists: record of position p (chunk-relative) at lists + (p - p0) * rec bytes
  unsigned char* lists;
  int rec, hdr;       // bytes per record; bytes of its header (T+1 u16 bucket starts, 16-aligned)
  int64_t p0, np;     // chunk of positions [p0, p0 + np)
  int* err;           // device error word
  int npre, buf_bytes; // PRE: list entries prefetched per position (one bulk copy), bytes of one buffer
  // sort from a per-warp shared-memory patch of the input (the union of the warp's PPW receptive fields
  // when its positions share an output row): C x KH x patch_w latencies, patch_w = KW + PPW - 1;
  // patch_n = 0 disables it.  Tables: ptab (patch index -> input offset), pkk (ky << 8 | kx),
  // eoffp (receptive-field entry -> patch index); the patch sits at warp base + patch_off.
  int patch_w, patch_n, patch_off, off_ptab, off_pkk, off_eoffp;
  // fused schedule: the fp32 weights [F][R], converted to fixed point while staged into shared memory
  // (no separate weight-prep launch); nullptr = copy the prepared wq
  const float* wf32;
  int nhwc;           // output layout: 0 = [B, F, Ho, Wo], 1 = [B, Ho, Wo, F] (SNN_CONV_OUT_NHWC)
  const int* kstar;   // nullable: K* (kstar_kernel) -- any K* spiking inputs fire every feature, so a
                      // sorted list can end with the first bucket that brings its count to K* (K2b)
  const int* kmin;    // nullable: word 1 of the K* pair = INT_MAX - kmin, kmin = the fewest spiking inputs that can
                      // bring ANY feature above the threshold (kstar_kernel); buckets that end below kmin
                      // entries are added without a threshold test (K2e)
  int pad_unit;       // sorted buckets padded to a multiple of this many entries: 4 (bucket walk) or 2 (K3 blocks)
  int in_nhwc;        // input layout [B, H, W, C] (SNN_CONV_IN_NHWC): receptive-field entries are then
                      // ordered (ky, kx, c) -- e = (ky KW + kx) C + c -- and so are the weight rows
  // row tiles (K7, walk_rows): a warp sorts the input halo of nx consecutive output positions of one
  // output row once, by (spike time, halo column); nseg tiles per output row
  int nx, nseg;
  int rows_g;         // K7c: buckets per threshold test of the row-tile walk (1, 2)
  int pool2, pool_off; // SNN_CONV_POOL2: 2 x 2 / stride 2 latency pooling fused into the row-tile walk
};

static inline int al16(int x) { return (x + 15) & ~15; }

template <int FPL> struct WalkVec;
template <> struct WalkVec<1> { typedef uint32_t T; };
template <> struct WalkVec<2> { typedef uint2 T; };
template <> struct WalkVec<4> { typedef uint4 T; };

template <int FPL>
__device__ __forceinline__ void wgather(const unsigned char* p, uint32_t (&o)[FPL]) {
  typedef typename WalkVec<FPL>::T V;
  const V v = *reinterpret_cast<const V*>(p);
  if constexpr (FPL == 1) { o[0] = v; }
  else if constexpr (FPL == 2) { o[0] = v.x; o[1] = v.y; }
  else { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
}

// The same gather from a 32-bit shared-window address (lane base + row offset): one LDS, no generic
// address arithmetic.  The weights do not change during a walk, so the load needs no ordering.
template <int FPL>
__device__ __forceinline__ void wgather_s(uint32_t a, uint32_t (&o)[FPL]) {
  if constexpr (FPL == 1) {
    asm("ld.shared.u32 %0, [%1];" : "=r"(o[0]) : "r"(a));
  } else if constexpr (FPL == 2) {
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(o[0]), "=r"(o[1]) : "r"(a));
  } else {
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "r"(a));
  }
}

// Where a walk gathers its weight rows from: the CTA's shared-memory slice (a 32-bit shared-window
// base, the default) or, for receptive fields too large for any shared-memory slice, the prepared
// fixed-point slice in global memory (L2-resident; GW walks, see conv_walk.cu).
struct WSrcS {
  uint32_t b;
  template <int FPL> __device__ __forceinline__ void g(uint32_t off, uint32_t (&o)[FPL]) const { wgather_s<FPL>(b + off, o); }
};
struct WSrcG {
  const unsigned char* b;
  template <int FPL> __device__ __forceinline__ void g(uint32_t off, uint32_t (&o)[FPL]) const {
    typedef typename WalkVec<FPL>::T V;
    const V v = __ldg(reinterpret_cast<const V*>(b + off));
    if constexpr (FPL == 1) { o[0] = v; }
    else if constexpr (FPL == 2) { o[0] = v.x; o[1] = v.y; }
    else { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  }
};

__device__ __forceinline__ uint8_t rf_lat(const WalkArgs& a, const int32_t* eoff, const uint16_t* ekk,
                                          const uint8_t* in, bool interior, int y0, int x0, int e) {
  if (interior) return in[eoff[e]];
  const int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
  const bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
  return ok ? in[eoff[e]] : kNoSpike;
}

// Counting sort of one position's receptive field by a group of LPP lanes into (start, list).
// Pass 1 counts the spiking inputs of each bucket with shared-memory atomics (independent, no
// read-modify-write chains in the lane); the counts are scanned (each bucket padded to a multiple of
// 4 entries with the zero-weight row R, so every bucket starts on a 16-byte boundary) into the header:
// start[0] = 0 and start[t + 1] = (padded end of bucket t) | (its pad count, 0..3, in the low 2 bits);
// pass 2 re-reads the latencies (L1-resident) and takes each entry's slot with an atomic on the
// bucket's running position.  Entries are weight-row byte offsets e * row_bytes; the tail is padded
// to a whole walk iteration.  The order inside a bucket is whatever the atomics gave: it does
// not change any result (the sum at a bucket end is exact and order-free).
template <int LPP, bool KM = false, class Lat>
__device__ __forceinline__ void rf_sort_group(const WalkArgs& a, bool pv, int gl, uint32_t* cnt, uint16_t* start,
                                              uint32_t* list, Lat lat_of) {
  const int R = a.R, T = a.T;
  const uint32_t rb = uint32_t(a.row_bytes);
  for (int t = gl; t < T; t += LPP) cnt[t] = 0;
  __syncwarp();
  if (pv) {
#if SNN_SORT_BATCH
    // latencies loaded in batches before their updates (the shared-memory atomics would otherwise order
    // each entry's table lookup and dependent load behind the previous entry's atomic)
    for (int e0 = gl; e0 < R; e0 += LPP * kSortUnroll) {
      int lb[kSortUnroll];
#pragma unroll
      for (int k = 0; k < kSortUnroll; ++k) lb[k] = e0 + k * LPP < R ? lat_of(e0 + k * LPP) : int(kNoSpike);
#pragma unroll
      for (int k = 0; k < kSortUnroll; ++k)
        if (lb[k] < T) atomicAdd(&cnt[lb[k]], 1u);
    }
#else
#pragma unroll kSortUnroll
    for (int e = gl; e < R; e += LPP) {
      const int l = lat_of(e);
      if (l < T) atomicAdd(&cnt[l], 1u);
    }
#endif
  }
  __syncwarp();
  // K2b: the last bucket kept, tcut = the first bucket whose running count reaches K* (every feature
  // has fired by its end, see kstar_kernel); later buckets are neither placed nor walked
  int tcut = T - 1;
  if (a.kstar) {
    const int ks = *a.kstar;
    if (ks < R) {
      int carry_r = 0;
      bool found = false;
      for (int tb = 0; tb < T; tb += LPP) {
        const int t = tb + gl;
        int inc = t < T ? int(cnt[t]) : 0;
#pragma unroll
        for (int o = 1; o < LPP; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, inc, o, LPP);
          if (gl >= o) inc += v;
        }
        const bool reach = t < T && carry_r + inc >= ks;
        const unsigned m = __ballot_sync(0xffffffffu, reach);
        const unsigned gm = (LPP == 32) ? m : (m >> ((threadIdx.x & 31) / LPP * LPP)) & ((1u << LPP) - 1u);
        if (!found && gm) { tcut = tb + __ffs(gm) - 1; found = true; }
        carry_r += __shfl_sync(0xffffffffu, inc, LPP - 1, LPP);
      }
    }
  }
  // K2e: with the kmin bound the walk adds the buckets before t0 -- the first bucket whose running count
  // reaches kmin -- as one run together with bucket t0, so those buckets need no pads: they are laid out
  // back to back (their header words hold the end rounded DOWN to 4 entries, which stays below kmin, pad
  // bits 0) and bucket t0 is padded so that its END falls on a 4-entry boundary.  cum0 = entries before t0
  // (KM: only the presorted sort kernel compiles this in -- the fused kernels never get the bound)
  int t0 = -1, cum0 = 0;
  if (KM && a.kmin && a.pad_unit == 4) {
    const int km = 0x7FFFFFFF - *a.kmin, need = km > 1 ? km : 1;
    t0 = 0x7FFFFFFF;
    int carry_r = 0;
    for (int tb = 0; tb < T; tb += LPP) {
      const int t = tb + gl;
      const int tot = (t < T && t <= tcut) ? int(cnt[t]) : 0;
      int inc = tot;
#pragma unroll
      for (int o = 1; o < LPP; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o, LPP);
        if (gl >= o) inc += v;
      }
      const unsigned m = __ballot_sync(0xffffffffu, t < T && carry_r + inc >= need);
      const unsigned gm = (LPP == 32) ? m : (m >> ((threadIdx.x & 31) / LPP * LPP)) & ((1u << LPP) - 1u);
      const int src = gm ? __ffs(gm) - 1 : 0;
      const int before = carry_r + __shfl_sync(0xffffffffu, inc - tot, src, LPP);
      if (t0 == 0x7FFFFFFF && gm) { t0 = tb + src; cum0 = before; }
      carry_r += __shfl_sync(0xffffffffu, inc, LPP - 1, LPP);
    }
  }
  int carry = 0;
  if (gl == 0) start[0] = 0;
  for (int tb = 0; tb < T; tb += LPP) {
    const int t = tb + gl;
    const int tot = t <= tcut ? int(cnt[t]) : 0;
    int padded = (tot + a.pad_unit - 1) & -a.pad_unit;  // 4: buckets 16-byte aligned (bucket walk); 2: pairs
    if (t < t0) padded = tot;
    else if (t == t0) padded = tot + ((-(cum0 + tot)) & 3);
    int inc = padded;
#pragma unroll
    for (int o = 1; o < LPP; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o, LPP);
      if (gl >= o) inc += v;
    }
    const int st = carry + inc - padded;
    if (t < T) {
      start[t + 1] = t < t0 ? uint16_t((st + tot) & ~3)         // K2e: an unpadded bucket of the test-free prefix
                            : uint16_t((st + padded) | (padded - tot));  // padded end | this bucket's pad count
      cnt[t] = uint32_t(st);                                    // pass 2: running slot of the bucket
      for (int k = tot; k < padded; ++k) list[st + k] = uint32_t(R) * rb;  // pads: the zero-weight row
    }
    carry += __shfl_sync(0xffffffffu, inc, LPP - 1, LPP);
  }
  __syncwarp();
  if (pv) {
#if SNN_SORT_BATCH
    for (int e0 = gl; e0 < R; e0 += LPP * kSortUnroll) {
      int lb[kSortUnroll];
#pragma unroll
      for (int k = 0; k < kSortUnroll; ++k) lb[k] = e0 + k * LPP < R ? lat_of(e0 + k * LPP) : int(kNoSpike);
#pragma unroll
      for (int k = 0; k < kSortUnroll; ++k)
        if (lb[k] <= tcut) list[atomicAdd(&cnt[lb[k]], 1u)] = uint32_t(e0 + k * LPP) * rb;
    }
#else
#pragma unroll kSortUnroll
    for (int e = gl; e < R; e += LPP) {
      const int l = lat_of(e);
      if (l <= tcut) {
        const uint32_t slot = atomicAdd(&cnt[l], 1u);
        SNN_DCHECK(slot < uint32_t(list_cap(R, T)));
        list[slot] = uint32_t(e) * rb;
      }
    }
#endif
  }
  {  // pad the tail to a whole walk iteration with the zero-weight row R
    const int n = carry;
    for (int k = n + gl; k < ((n + kIt - 1) & ~(kIt - 1)); k += LPP) list[k] = uint32_t(R) * rb;
  }
  __syncwarp();
}

// Sort the receptive field of each of the warp's PPW consecutive positions (group grp = position
// q0 + grp).  When the warp's valid positions share an output row, the union of their receptive
// fields is first staged once into the warp's shared-memory patch (one coalesced-ish byte gather,
// bounds checked once per patch element); both sort passes then read latencies from the patch.
// Otherwise (a warp straddling a row end) each group reads its latencies from global memory.
template <int PPW, bool KM = false>
__device__ __forceinline__ void rf_sort_warp(const WalkArgs& a, const unsigned char* tabs, unsigned char* wbase,
                                             int64_t q0, int lane, int grp, int gl, bool pv, uint32_t* cnt,
                                             uint16_t* start, uint32_t* list) {
  constexpr int LPP = 32 / PPW;
  const int HoWo = a.Ho * a.Wo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  const int64_t qlast = (q0 + PPW - 1 < a.np ? q0 + PPW - 1 : a.np - 1);
  const int pf = int(a.p0 + q0), pl = int(a.p0 + qlast);
  if (a.patch_n > 0 && pf / a.Wo == pl / a.Wo) {  // warp-uniform
    const int32_t* ptab = reinterpret_cast<const int32_t*>(tabs + a.off_ptab);
    const uint16_t* pkk = reinterpret_cast<const uint16_t*>(tabs + a.off_pkk);
    const uint16_t* eoffp = reinterpret_cast<const uint16_t*>(tabs + a.off_eoffp);
    uint8_t* patch = wbase + a.patch_off;
    const int b = pf / HoWo, rem = pf - b * HoWo, y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in0 = a.lat_in + int64_t(b) * CHW + (int64_t(y0) * a.W + x0) * (a.in_nhwc ? a.C : 1);
    const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.patch_w <= a.W;
    if (interior) {
      for (int i = lane; i < a.patch_n; i += 32) patch[i] = __ldg(in0 + ptab[i]);
    } else {
      for (int i = lane; i < a.patch_n; i += 32) {
        const int kk = pkk[i], yy = y0 + (kk >> 8), xx = x0 + (kk & 0xFF);
        patch[i] = (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W) ? __ldg(in0 + ptab[i]) : kNoSpike;
      }
    }
    __syncwarp();
    const uint8_t* pg = patch + grp * (a.in_nhwc ? a.C : 1);  // the group's position is grp columns right
    rf_sort_group<LPP, KM>(a, pv, gl, cnt, start, list, [&](int e) { return int(pg[eoffp[e]]); });
  } else {
    const int32_t* eoff = reinterpret_cast<const int32_t*>(tabs + a.off_eoff);
    const uint16_t* ekk = reinterpret_cast<const uint16_t*>(tabs + a.off_ekk);
    const int p = int(a.p0 + q0 + grp);
    const int b = pv ? p / HoWo : 0;
    const int rem = pv ? p - b * HoWo : 0;
    const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in = a.lat_in + int64_t(b) * CHW + (int64_t(y0) * a.W + x0) * (a.in_nhwc ? a.C : 1);
    const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;
    if (PPW == 1 && interior)  // no bounds tests: the loads of an unrolled group issue back to back
      rf_sort_group<LPP, KM>(a, pv, gl, cnt, start, list, [&](int e) { return int(__ldg(in + eoff[e])); });
    else  // (PPW > 1 only reaches here for a warp straddling a row end: one lambda keeps its code small)
      rf_sort_group<LPP, KM>(a, pv, gl, cnt, start, list,
                         [&](int e) { return int(rf_lat(a, eoff, ekk, in, interior, y0, x0, e)); });
  }
}

__device__ __forceinline__ void rf_tables(const WalkArgs& a, unsigned char* tabs) {
  int32_t* eoff = reinterpret_cast<int32_t*>(tabs + a.off_eoff);
  uint16_t* ekk = reinterpret_cast<uint16_t*>(tabs + a.off_ekk);
  const int KK = a.KH * a.KW;
  for (int e = threadIdx.x; e < a.R; e += blockDim.x) {
    int c, ky, kx;
    if (a.in_nhwc) {  // e = (ky KW + kx) C + c
      const int kk = e / a.C;
      c = e - kk * a.C; ky = kk / a.KW; kx = kk - ky * a.KW;
      eoff[e] = (ky * a.W + kx) * a.C + c;
      if (a.patch_n > 0)
        reinterpret_cast<uint16_t*>(tabs + a.off_eoffp)[e] = uint16_t((ky * a.patch_w + kx) * a.C + c);
    } else {          // e = (c KH + ky) KW + kx
      c = e / KK;
      const int r = e - c * KK;
      ky = r / a.KW; kx = r - ky * a.KW;
      eoff[e] = c * a.H * a.W + ky * a.W + kx;
      if (a.patch_n > 0)
        reinterpret_cast<uint16_t*>(tabs + a.off_eoffp)[e] = uint16_t((c * a.KH + ky) * a.patch_w + kx);
    }
    ekk[e] = uint16_t((ky << 8) | kx);
  }
  const int PK = a.KH * a.patch_w;
  for (int i = threadIdx.x; i < a.patch_n; i += blockDim.x) {
    int c, ky, kx;
    if (a.in_nhwc) {
      const int kk = i / a.C;
      c = i - kk * a.C; ky = kk / a.patch_w; kx = kk - ky * a.patch_w;
      reinterpret_cast<int32_t*>(tabs + a.off_ptab)[i] = (ky * a.W + kx) * a.C + c;
    } else {
      c = i / PK;
      const int r = i - c * PK;
      ky = r / a.patch_w; kx = r - ky * a.patch_w;
      reinterpret_cast<int32_t*>(tabs + a.off_ptab)[i] = c * a.H * a.W + ky * a.W + kx;
    }
    reinterpret_cast<uint16_t*>(tabs + a.off_pkk)[i] = uint16_t((ky << 8) | kx);
  }
}

// ------------------------------------------------------------------------------------- walk
template <int FPL, bool PRE> struct WalkThreads { static constexpr int v = FPL == 4 ? 768 : 1024; };

// Accumulator of a fired (or padding) feature: INT64_MIN, so no later sum along the list (at most
// R * 2^31 < 2^44) can bring it back above a threshold, and "fired" needs no separate mask.
constexpr uint64_t kFiredAcc = 0x8000000000000000ull;

// Fixed-point scale of a walk: S28 = weights in units of 2^-28 (every weight of the slice is 0 or a
// multiple of 2^-28 in [0, 1], i.e. w = 0 or w >= 2^-5 for fp32), else units of 2^-31 (N1).
// At 2^-28 the sum of any 8 weights is < 2^31, so a block sums in 32 bits exactly (K3b).
template <bool S28>
__device__ __forceinline__ float fixed_to_float_s(int64_t acc) {
  if constexpr (S28) return __ll2float_rn(acc) * 3.7252902984619140625e-09f;  // 2^-28, exact scaling
  else return fixed_to_float(acc);
}

// Fire every unfired feature whose potential at the end of bucket t exceeds the threshold.
template <int FPL, bool S28>
__device__ __forceinline__ void fire_at(uint64_t (&acc)[FPL], int64_t thr, int t, uint32_t& lo, float (&vo)[FPL]) {
#pragma unroll
  for (int j = 0; j < FPL; ++j) {
    if (int64_t(acc[j]) > thr) {
      lo = (lo & ~(0xFFu << (8 * j))) | (uint32_t(t) << (8 * j));
      vo[j] = fixed_to_float_s<S28>(int64_t(acc[j]));
      acc[j] = kFiredAcc;
    }
  }
}

// NB consecutive entries of one bucket: gather each lane's FPL weights per entry (one conflict-free
// LDS.32/64/128) and add them to the exact accumulators.  S28: every (up to) 8 weights are summed in
// 32 bits (exact, < 2^31) before the 64-bit add (K3b).  Pad entries (the zero-weight row) add 0.
template <int FPL, bool S28, int NB, class WS>
__device__ __forceinline__ void walk_gather_add(const WS& wls, const uint32_t (&off)[NB], uint64_t (&acc)[FPL]) {
  uint32_t wv[NB][FPL];
#pragma unroll
  for (int k = 0; k < NB; ++k) wls.template g<FPL>(off[k], wv[k]);
#pragma unroll
  for (int j = 0; j < FPL; ++j) {
    uint64_t t = acc[j];
    if constexpr (S28) {
#pragma unroll
      for (int h = 0; h < NB; h += 8) {
        if constexpr (NB >= 8)
          t += ((wv[h][j] + wv[h + 1][j]) + (wv[h + 2][j] + wv[h + 3][j])) +
               ((wv[h + 4][j] + wv[h + 5][j]) + (wv[h + 6][j] + wv[h + 7][j]));
        else
          t += (wv[h][j] + wv[h + 1][j]) + (wv[h + 2][j] + wv[h + 3][j]);
      }
    } else {
#pragma unroll
      for (int h = 0; h < NB; h += 2) t += uint64_t(wv[h][j]) + wv[h + 1][j];
    }
    acc[j] = t;
  }
}

// ---------------------------------------------------------------- walk in blocks across buckets (K3)
// For layers whose buckets are small (a few entries: R / T below ~8, e.g. C1, C4's first layer) the
// bucket-by-bucket walk below would pay its per-bucket test, vote and padding for 2-3 entries; this
// walk streams the list in fixed blocks instead.  The bucket ends inside a block are known to the
// whole group beforehand (endm: bit m = a bucket ends after pair m, its index in byte m of tpk); each
// lane sums its features' weights for the block exactly; if no unfired feature then exceeds the
// threshold no test inside the block could fire (potentials only grow along the list) and the block is
// taken whole; otherwise the lane re-adds it pair by pair and tests at every bucket end (K3).
// Sorted with pad unit 2: header word = padded end | pad count (bit 0).
template <int FPL, bool S28, int NB, class WS>
__device__ __forceinline__ void walk_block_k3(const WS& wls, const uint32_t (&off)[NB], unsigned endm, uint64_t tpk,
                                           int64_t thr, uint64_t (&acc)[FPL], uint32_t& lo, float (&vo)[FPL]) {
  uint32_t wv[NB][FPL];
#pragma unroll
  for (int k = 0; k < NB; ++k) wls.template g<FPL>(off[k], wv[k]);
  uint64_t s[FPL];
  bool hit = false;
#pragma unroll
  for (int j = 0; j < FPL; ++j) {
    if constexpr (S28) {
      uint64_t t = acc[j];
#pragma unroll
      for (int h = 0; h < NB; h += 8) {
        const uint32_t b = ((wv[h][j] + wv[h + 1][j]) + (wv[h + 2][j] + wv[h + 3][j])) +
                           ((wv[h + 4][j] + wv[h + 5][j]) + (wv[h + 6][j] + wv[h + 7][j]));
        t += b;
      }
      s[j] = t;
    } else {
      uint64_t t = acc[j];
#pragma unroll
      for (int h = 0; h < NB; h += 2) t += uint64_t(wv[h][j]) + wv[h + 1][j];
      s[j] = t;
    }
    hit |= int64_t(s[j]) > thr;
  }
  constexpr unsigned kInner = (1u << (NB / 2 - 1)) - 1u;  // bucket ends strictly inside the block
  if (hit && endm) {
    if (endm & kInner) {  // pair by pair
#pragma unroll
      for (int m = 0; m < NB / 2; ++m) {
#pragma unroll
        for (int j = 0; j < FPL; ++j) {
          if constexpr (S28) acc[j] += uint32_t(wv[2 * m][j] + wv[2 * m + 1][j]);
          else acc[j] += uint64_t(wv[2 * m][j]) + wv[2 * m + 1][j];
        }
        if (endm >> m & 1) fire_at<FPL, S28>(acc, thr, int((tpk >> (8 * m)) & 0xFFu), lo, vo);
      }
      return;
    }
    // the only bucket end is the block end
#pragma unroll
    for (int j = 0; j < FPL; ++j) acc[j] = s[j];
    fire_at<FPL, S28>(acc, thr, int((tpk >> (8 * (NB / 2 - 1))) & 0xFFu), lo, vo);
    return;
  }
#pragma unroll
  for (int j = 0; j < FPL; ++j) acc[j] = s[j];
}

// Walk one position's sorted list (K2/K3) for the FPL features of this lane; group-uniform control,
// full-warp votes only.  start: T+1 bucket starts; entries come from shared memory (sent for PRE,
// list otherwise) or, for PRE past the prefetched npre entries, from global memory (ent).  thr is
// the threshold in the walk's fixed-point units (S28: 2^-28, else 2^-31).
template <int FPL, int PPW, bool PRE, bool S28, bool GW>
__device__ __forceinline__ void walk_list_blocks(const WalkArgs& a, const unsigned char* wl, const uint16_t* start,
                                          const unsigned char* sent, const unsigned char* ent, const uint32_t* list,
                                          bool pv, unsigned valid, unsigned gmask, uint32_t& lo, float (&vo)[FPL]) {
  const int T = a.T;
  const int64_t thr = S28 ? a.thr28 : a.thr;
  // the lane's weight base: a shared-window address, opaque so it stays in a register (GW: global)
  typename std::conditional<GW, WSrcG, WSrcS>::type wls;
  if constexpr (GW) wls.b = wl;
  else asm volatile("mov.u32 %0, %1;" : "=r"(wls.b) : "r"(smem_u32(wl)));
    uint64_t acc[FPL];
    lo = 0xFFFFFFFFu;  // byte j = lat of feature j (255 = no spike)
#pragma unroll
    for (int j = 0; j < FPL; ++j) { acc[j] = (valid >> j & 1) ? 0ull : kFiredAcc; vo[j] = 0.0f; }
    const int total = pv ? int(start[T] & ~1u) : 0;  // padded end of the list
    if (pv && int(start[1]) == 0 && int64_t(0) > thr) {  // empty bucket 0: P[0] = 0 > a negative threshold
#pragma unroll
      for (int j = 0; j < FPL; ++j)
        if (int64_t(acc[j]) >= 0) { lo &= ~(0xFFu << (8 * j)); acc[j] = kFiredAcc; }
    }
    bool done = !pv || total == 0;  // group-uniform, like every later update of done
    auto alive = [&]() {  // an unfired valid feature remains in this lane
      bool al = false;
#pragma unroll
      for (int j = 0; j < FPL; ++j) al |= int64_t(acc[j]) >= 0;
      return al;
    };
    {
      const unsigned nd = __ballot_sync(0xffffffffu, alive());
      if ((nd & gmask) == 0) done = true;  // all features of the group fired (or are padding)
    }
    int i = 0, it = 0;
    // the first non-empty bucket (leading empty ones were handled above): the group's lanes test LPP
    // buckets per vote (no serial chain of dependent header loads); a uniform trip count keeps every
    // group's lanes in the full-warp ballots
    constexpr int LPP = 32 / PPW;
    const int gl = int(threadIdx.x & 31) % LPP;
    int t = T;
    for (int tb = 0; tb < T; tb += LPP) {
      const int tt = tb + gl;
      const bool ne = pv && tt < T && int(start[tt + 1]) != 0;
      const unsigned m = (__ballot_sync(0xffffffffu, ne) & gmask) >> (gmask == 0xffffffffu ? 0 : __ffs(gmask) - 1);
      if (t == T && m) t = tb + __ffs(m) - 1;
    }
    int bend = t < T ? int(start[t + 1] & ~1u) : 0x7FFFFFFF;  // (padded) end of the current non-empty bucket t
    int guard = (total + kIt - 1) / kIt + 2;  // iterations this group can take (a bug trap, never hit)
    uint32_t ebase;  // shared-window address of the entries (computed once, kept in a register)
    asm volatile("mov.u32 %0, %1;" : "=r"(ebase)
                 : "r"(smem_u32(PRE ? static_cast<const void*>(sent) : static_cast<const void*>(list))));
    // Every vote below is a full-warp ballot at a converged point; done is group-uniform.
    while (true) {
      if (__ballot_sync(0xffffffffu, !done) == 0) break;
      uint4 cur[4];  // this iteration's 16 entries: shared memory (PRE past npre: global memory)
      if (PRE && it * kIt >= a.npre) {
        const uint4* g4 = reinterpret_cast<const uint4*>(ent + it * kIt * 4);
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = __ldg(g4 + u);
      } else {
        const uint32_t sa = ebase + uint32_t(it * kIt * 4);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(cur[u].x), "=r"(cur[u].y), "=r"(cur[u].z), "=r"(cur[u].w)
                       : "r"(sa + 16 * u));
      }
      // blocks of NB entries: 16 for FPL <= 2 (one bookkeeping / vote / threshold test per 16 gathers),
      // 8 for FPL = 4 (register budget: 4 registers per gathered entry)
      constexpr int NB = FPL == 4 ? 8 : 16;
      const uint32_t offs[16] = {cur[0].x, cur[0].y, cur[0].z, cur[0].w, cur[1].x, cur[1].y, cur[1].z, cur[1].w,
                                 cur[2].x, cur[2].y, cur[2].z, cur[2].w, cur[3].x, cur[3].y, cur[3].z, cur[3].w};
#pragma unroll
      for (int h = 0; h < 16 / NB; ++h) {
        if (!done) {
          // group-uniform: bucket ends inside this block (pair m ends bucket t_m)
          unsigned endm = 0;
          uint64_t tpk = 0;
          i += NB;
          while (bend <= i) {
            const int m = ((bend - (i - NB)) >> 1) - 1;
            endm |= 1u << m;
            tpk |= uint64_t(t) << (8 * m);
            ++t;
            while (t < T && int(start[t + 1] & ~1u) == bend) ++t;  // empty buckets add nothing
            bend = t < T ? int(start[t + 1] & ~1u) : 0x7FFFFFFF;
          }
          uint32_t off[NB];
#pragma unroll
          for (int k = 0; k < NB; ++k) off[k] = offs[h * NB + k];
          walk_block_k3<FPL, S28, NB>(wls, off, endm, tpk, thr, acc, lo, vo);
        }
        const unsigned nf = __ballot_sync(0xffffffffu, !done && alive());
        if (!done && ((nf & gmask) == 0 || i >= total)) done = true;
      }
      ++it;
      if (!done && --guard < 0) {
        flag_error(a.err, kErrInternal);
        done = true;
      }
    }
}


// Walk one position's sorted list (K2/K3) for the FPL features of this lane, bucket by bucket: a
// bucket's entries are added in blocks of NB (no test inside a bucket -- the potential is only
// defined per time step), then every unfired feature is tested once at the bucket end (exact:
// lat = t, v = P[t]); the group stops when all its features fired.  Control is group-uniform and every
// vote / shuffle is group-masked, so groups of a warp (PPW > 1) may diverge.  start: the header
// (start[t + 1] = padded end of bucket t | its pad count); entries come from shared memory (sent for
// PRE, list otherwise) or, for PRE past the prefetched npre entries, from global memory (ent).  thr
// is the threshold in the walk's fixed-point units (S28: 2^-28, else 2^-31).
template <int FPL, int PPW, bool PRE, bool S28 = false, bool BW = true, bool GW = false>
__device__ __forceinline__ void walk_list(const WalkArgs& a, const unsigned char* wl, const uint16_t* start,
                                          const unsigned char* sent, const unsigned char* ent, const uint32_t* list,
                                          bool pv, unsigned valid, unsigned gmask, uint32_t& lo, float (&vo)[FPL],
                                          int need = 1) {
  if constexpr (!BW) {
    walk_list_blocks<FPL, PPW, PRE, S28, GW>(a, wl, start, sent, ent, list, pv, valid, gmask, lo, vo);
    return;
  }
  constexpr int NB = FPL == 4 ? 8 : 16;  // register budget: FPL registers per gathered entry
  constexpr int LPP = 32 / PPW;
  const int T = a.T;
  const int64_t thr = S28 ? a.thr28 : a.thr;
  // the lane's weight base: a shared-window address, opaque so it stays in a register (GW: global)
  typename std::conditional<GW, WSrcG, WSrcS>::type wls;
  if constexpr (GW) wls.b = wl;
  else asm volatile("mov.u32 %0, %1;" : "=r"(wls.b) : "r"(smem_u32(wl)));
  uint32_t ebase;  // shared-window address of the entries
  asm volatile("mov.u32 %0, %1;" : "=r"(ebase)
               : "r"(smem_u32(PRE ? static_cast<const void*>(sent) : static_cast<const void*>(list))));
  uint64_t acc[FPL];
  lo = 0xFFFFFFFFu;  // byte j = lat of feature j (255 = no spike)
#pragma unroll
  for (int j = 0; j < FPL; ++j) { acc[j] = (valid >> j & 1) ? 0ull : kFiredAcc; vo[j] = 0.0f; }
  if (!pv) return;                       // group-uniform
  auto alive = [&]() {
    bool al = false;
#pragma unroll
    for (int j = 0; j < FPL; ++j) al |= int64_t(acc[j]) >= 0;
    return al;
  };
  if (int(start[1]) == 0 && int64_t(0) > thr) {  // empty bucket 0: P[0] = 0 > a negative threshold
#pragma unroll
    for (int j = 0; j < FPL; ++j)
      if (int64_t(acc[j]) >= 0) { lo &= ~(0xFFu << (8 * j)); acc[j] = kFiredAcc; }
  }
  if (__ballot_sync(gmask, alive()) == 0) return;
  // the first bucket that can fire a feature: the first one whose padded end reaches kmin entries (K2e; no
  // feature crosses the threshold with fewer than kmin inputs, and a padded end bounds the real count from
  // above; need = max(kmin, 1), read once per kernel by the caller); without the bound (need = 1) the first
  // non-empty bucket.  The group's lanes test LPP buckets per vote
  const int gl = int(threadIdx.x & 31) % LPP;
  int t = T;
  for (int tb = 0; tb < T && t == T; tb += LPP) {
    const int tt = tb + gl;
    const unsigned m = __ballot_sync(gmask, tt < T && int(start[tt + 1] & ~3u) >= need) & gmask;
    if (m) t = tb + __ffs(m >> (__ffs(gmask) - 1)) - 1;
  }
  int b0 = 0;                            // the first run walked is [0, end of bucket t): the earlier buckets (empty,
                                         // or below kmin entries: no test needed, pads add 0) together with bucket t
  // header words through a 32-bit shared-window address kept in a register (start[t + 2] = hdr + 2 t + 4)
  uint32_t hdr_a;
  asm volatile("mov.u32 %0, %1;" : "=r"(hdr_a) : "r"(smem_u32(start)));
  auto hdr_word = [&](int i) {
    uint16_t h;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(hdr_a + uint32_t(2 * i)));
    return uint32_t(h);
  };
  // entries k.. of the list from shared memory (every entry of a bucket below npre), 4 per LDS.128
  auto load_sm = [&](int k, auto& off) {
    constexpr int M = sizeof(off) / sizeof(off[0]);
#pragma unroll
    for (int q = 0; q < M / 4; ++q) {
      uint4 c;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "r"(ebase + uint32_t((k + 4 * q) * 4)));
      off[4 * q] = c.x; off[4 * q + 1] = c.y; off[4 * q + 2] = c.z; off[4 * q + 3] = c.w;
#ifdef SNN_CHECKED
      for (int u = 0; u < 4; ++u)
        SNN_DCHECK(off[4 * q + u] <= uint32_t(a.R) * uint32_t(a.row_bytes) && off[4 * q + u] % uint32_t(a.row_bytes) == 0);
#endif
    }
  };
  // PRE, past the prefetched npre entries (a long walk): 16-byte groups from global memory
  auto load_gl = [&](int k, auto& off) {
    constexpr int M = sizeof(off) / sizeof(off[0]);
#pragma unroll
    for (int q = 0; q < M / 4; ++q) {
      const int e4 = k + 4 * q;
      uint4 c;
      if (e4 >= a.npre) {
        c = __ldg(reinterpret_cast<const uint4*>(ent + e4 * 4));
      } else {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "r"(ebase + uint32_t(e4 * 4)));
      }
      off[4 * q] = c.x; off[4 * q + 1] = c.y; off[4 * q + 2] = c.z; off[4 * q + 3] = c.w;
    }
  };
  // the padded bucket [b0, b1) (a multiple of 4 entries; its 0-3 pads gather the zero row) in blocks of
  // NB, then at most one block of 8 (NB = 16) and one of 4: no per-entry predicates
  auto add_bucket = [&](int b0_, int b1_, auto load_off) {
    int k = b0_;
    if constexpr (NB == 16) {
      for (; k + 16 <= b1_; k += 16) {
        uint32_t off[16];
        load_off(k, off);
        walk_gather_add<FPL, S28, 16>(wls, off, acc);
      }
    }
    if (k + 8 <= b1_) {
      uint32_t off[8];
      load_off(k, off);
      walk_gather_add<FPL, S28, 8>(wls, off, acc);
      k += 8;
      if constexpr (NB == 8) {
        for (; k + 8 <= b1_; k += 8) {
          uint32_t off2[8];
          load_off(k, off2);
          walk_gather_add<FPL, S28, 8>(wls, off2, acc);
        }
      }
    }
    if (k < b1_) {
      uint32_t off[4];
      load_off(k, off);
      walk_gather_add<FPL, S28, 4>(wls, off, acc);
    }
  };
  const int nsm = PRE ? a.npre : 0x7FFFFFFF;  // entries below nsm are in shared memory
  uint32_t wnext = t < T ? hdr_word(t + 1) : 0;
#pragma unroll 1
  for (; t < T; ++t) {
    const uint32_t w1 = wnext;
    if (t + 1 < T) wnext = hdr_word(t + 2);  // the next header word in flight while this bucket is walked
    const int b1 = int(w1 & ~3u), n = b1 - b0 - int(w1 & 3u);
    if (n > 0) {
      if (!PRE || b1 <= nsm) add_bucket(b0, b1, load_sm);  // the common case: no global-memory code
      else add_bucket(b0, b1, load_gl);
      // the exact test at the bucket end; the conversions only in the (rare) bucket where one fires
      bool any = false;
#pragma unroll
      for (int j = 0; j < FPL; ++j) any |= int64_t(acc[j]) > thr;
      // only a bucket in which some lane fired can end the group's walk: vote on liveness only then
      if (__any_sync(gmask, any)) {
        if (any) fire_at<FPL, S28>(acc, thr, t, lo, vo);
        if (__ballot_sync(gmask, alive()) == 0) break;
      }
    }
    b0 = b1;
  }
}

// Walk PPW > 1 positions' sorted lists in lockstep (K3c; the fused schedule of small-receptive-field
// layers, e.g. C2's first layer and C4's first layer, whose buckets hold a few entries each).  Every
// lane runs the same bucket loop t = 0..T-1: a group gathers its own bucket's entries, the warp iterates
// to the largest bucket of its groups (a shorter bucket's lanes gather the zero-weight row R), so control
// never diverges between the groups of a warp; the exact test at each bucket end as in walk_list
// (lat = t, v = P[t]).  Lists sorted with pad unit 1 (start[t + 1] = the end of bucket t, no pads).  S28:
// up to 14 weights are summed in 32 bits (< 2^32) before the 64-bit add.  A group whose features have
// all fired stops gathering; the warp stops when every group has.
template <int FPL, int PPW, bool S28>
__device__ __forceinline__ void walk_list_lockstep(const WalkArgs& a, const unsigned char* wl, const uint16_t* start,
                                                   const uint32_t* list, bool pv, unsigned valid, uint32_t& lo,
                                                   float (&vo)[FPL]) {
  const int T = a.T;
  const int64_t thr = S28 ? a.thr28 : a.thr;
  WSrcS wls;
  asm volatile("mov.u32 %0, %1;" : "=r"(wls.b) : "r"(smem_u32(wl)));
  const uint32_t zrow = uint32_t(a.R) * uint32_t(a.row_bytes);  // the zero-weight row
  uint64_t acc[FPL];
  lo = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < FPL; ++j) { acc[j] = (pv && (valid >> j & 1)) ? 0ull : kFiredAcc; vo[j] = 0.0f; }
  auto alive = [&]() {
    bool al = false;
#pragma unroll
    for (int j = 0; j < FPL; ++j) al |= int64_t(acc[j]) >= 0;
    return al;
  };
  // a group is alive while one of its lanes has an unfired feature (group-uniform via the group's ballot)
  constexpr int LPP = 32 / PPW;
  const int grp = int(threadIdx.x & 31) / LPP;
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1u) << (grp * LPP));
  bool galive = (__ballot_sync(0xffffffffu, alive()) & gmask) != 0;
  if (!__any_sync(0xffffffffu, galive)) return;
  uint32_t lbase;  // the group's list as a shared-window address
  asm volatile("mov.u32 %0, %1;" : "=r"(lbase) : "r"(smem_u32(list)));
  int b0 = 0;
#pragma unroll 1
  for (int t = 0; t < T; ++t) {
    const int b1 = pv ? int(start[t + 1]) : 0;
    const int n = galive ? b1 - b0 : 0;
    const int nmax = __reduce_max_sync(0xffffffffu, n);
    for (int c0 = 0; c0 < nmax; c0 += 14) {  // chunks of <= 14 entries (32-bit partial sums, S28)
      const int c1 = min(nmax, c0 + 14);
      uint32_t part[FPL];
#pragma unroll
      for (int j = 0; j < FPL; ++j) part[j] = 0;
      for (int k = c0; k < c1; k += 2) {
        uint32_t off[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t e = zrow;
          if (k + u < n) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(lbase + uint32_t((b0 + k + u) * 4)));
          SNN_DCHECK(e <= zrow && e % uint32_t(a.row_bytes) == 0);
          off[u] = e;
        }
        uint32_t w0[FPL], w1[FPL];
        wls.template g<FPL>(off[0], w0);
        wls.template g<FPL>(off[1], w1);
#pragma unroll
        for (int j = 0; j < FPL; ++j) {
          if constexpr (S28) part[j] += w0[j] + w1[j];
          else acc[j] += uint64_t(w0[j]) + w1[j];
        }
      }
      if constexpr (S28) {
#pragma unroll
        for (int j = 0; j < FPL; ++j) acc[j] += part[j];
      }
    }
    if (n > 0 || t == 0) {  // the exact test at the end of bucket t (t = 0: a negative threshold)
      bool any = false;
#pragma unroll
      for (int j = 0; j < FPL; ++j) any |= int64_t(acc[j]) > thr;
      if (any) fire_at<FPL, S28>(acc, thr, t, lo, vo);
    }
    if (__any_sync(0xffffffffu, n > 0 || t == 0)) {
      galive = (__ballot_sync(0xffffffffu, alive()) & gmask) != 0;
      if (!__any_sync(0xffffffffu, galive)) break;
    }
    b0 = b1;
  }
}

// ------------------------------------------------------------------------------------- K7 row tiles
// Walk of one position's buckets from a row tile's (t, column) sorted halo list (walk_rows): the same
// lockstep loop as walk_list_lockstep (PPW positions per warp, a group gathers its own bucket, the warp
// iterates to the largest; exact test at each bucket end, lat = t, v = P[t]), but bucket t of the
// group's position is the contiguous list range [base[t ncol], base[t ncol + KW]) -- the entries of the
// KW halo columns its receptive field covers -- and the entries are u16 weight-row byte offsets
// relative to the tile's first position, so the group's gather base is shifted by its column
// (wgb = slice - xr C row_bytes) and its zero-weight row is zrow = (R + xr C) row_bytes.
template <int FPL, int PPW, bool S28, int G>
__device__ __forceinline__ void walk_rows_lockstep(const WalkArgs& a, uint32_t wgb, uint32_t zrow, const uint16_t* base,
                                                   int ncol, uint32_t lbase, bool pv, unsigned valid, uint32_t& lo,
                                                   float (&vo)[FPL]) {
  const int T = a.T, KW = a.KW;
  const int64_t thr = S28 ? a.thr28 : a.thr;
  WSrcS wls;
  wls.b = wgb;
  uint64_t acc[FPL];
  lo = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < FPL; ++j) { acc[j] = (pv && (valid >> j & 1)) ? 0ull : kFiredAcc; vo[j] = 0.0f; }
  auto alive = [&]() {
    bool al = false;
#pragma unroll
    for (int j = 0; j < FPL; ++j) al |= int64_t(acc[j]) >= 0;
    return al;
  };
  constexpr int LPP = 32 / PPW;
  const int grp = int(threadIdx.x & 31) / LPP;
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1u) << (grp * LPP));
  bool galive = (__ballot_sync(0xffffffffu, alive()) & gmask) != 0;
  if (!__any_sync(0xffffffffu, galive)) return;
  // gather-add of entries [k0, k1) of the lockstep bucket (b0, n) into 32-bit (S28) or 64-bit sums
  auto gather = [&](int b0, int n, int k0, int k1, uint32_t (&part)[FPL]) {
    for (int k = k0; k < k1; k += 2) {
      uint32_t off[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        uint32_t e = zrow;
        if (k + u < n) {
          uint16_t h;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(lbase + uint32_t((b0 + k + u) * 2)));
          e = h;
        }
        off[u] = e;
      }
      uint32_t w0[FPL], w1[FPL];
      wls.template g<FPL>(off[0], w0);
      wls.template g<FPL>(off[1], w1);
#pragma unroll
      for (int j = 0; j < FPL; ++j) {
        if constexpr (S28) part[j] += w0[j] + w1[j];
        else acc[j] += uint64_t(w0[j]) + w1[j];
      }
    }
  };
  const uint16_t* bt = base;
#pragma unroll 1
  for (int t0 = 0; t0 < T; t0 += G, bt += G * ncol) {
    int b0[G], n[G], tot = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      b0[i] = 0; n[i] = 0;
      if (pv && galive && t0 + i < T) { b0[i] = int(bt[i * ncol]); n[i] = int(bt[i * ncol + KW]) - b0[i]; }
      tot += n[i];
    }
    bool fired = false;
    if (S28 && G > 1 && __reduce_max_sync(0xffffffffu, tot) <= 14) {
      // K7c block of G buckets: sums in 32 bits with a snapshot at every bucket end, ONE threshold test at
      // the block end (the potential is monotone: no feature crosses inside the block unless it is above
      // the threshold at its end); a crossing feature takes the first bucket end above (exact lat, v)
      uint32_t part[FPL], snap[G][FPL];
#pragma unroll
      for (int j = 0; j < FPL; ++j) part[j] = 0;
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int nmax = __reduce_max_sync(0xffffffffu, n[i]);
        gather(b0[i], n[i], 0, nmax, part);
#pragma unroll
        for (int j = 0; j < FPL; ++j) snap[i][j] = part[j];
      }
      bool any = false;
#pragma unroll
      for (int j = 0; j < FPL; ++j) any |= int64_t(acc[j] + part[j]) > thr;
      if (any) {
#pragma unroll
        for (int j = 0; j < FPL; ++j) {
          if (int64_t(acc[j] + part[j]) > thr) {
            int fi = G - 1;
#pragma unroll
            for (int i = G - 2; i >= 0; --i)
              if (int64_t(acc[j] + snap[i][j]) > thr) fi = i;
            uint32_t sv = snap[0][j];
#pragma unroll
            for (int i = 1; i < G; ++i) if (fi == i) sv = snap[i][j];
            lo = (lo & ~(0xFFu << (8 * j))) | (uint32_t(t0 + fi) << (8 * j));
            vo[j] = fixed_to_float_s<S28>(int64_t(acc[j] + sv));
            acc[j] = kFiredAcc;
          } else {
            acc[j] += part[j];
          }
        }
        fired = true;
      } else {
#pragma unroll
        for (int j = 0; j < FPL; ++j) acc[j] += part[j];
      }
    } else {
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int t = t0 + i;
        const int nmax = __reduce_max_sync(0xffffffffu, n[i]);
        for (int c0 = 0; c0 < nmax; c0 += 14) {  // chunks of <= 14 entries (32-bit partial sums, S28)
          uint32_t part[FPL];
#pragma unroll
          for (int j = 0; j < FPL; ++j) part[j] = 0;
          gather(b0[i], n[i], c0, min(nmax, c0 + 14), part);
          if constexpr (S28) {
#pragma unroll
            for (int j = 0; j < FPL; ++j) acc[j] += part[j];
          }
        }
        if ((n[i] > 0 || t == 0) && t < T) {  // the exact test at the end of bucket t (t = 0: a negative threshold)
          bool any = false;
#pragma unroll
          for (int j = 0; j < FPL; ++j) any |= int64_t(acc[j]) > thr;
          if (any) { fire_at<FPL, S28>(acc, thr, t, lo, vo); fired = true; }
        }
      }
    }
    if (__any_sync(0xffffffffu, fired)) {  // liveness changes only where a feature fired
      galive = (__ballot_sync(0xffffffffu, alive()) & gmask) != 0;
      if (!__any_sync(0xffffffffu, galive)) break;
    }
  }
}

// Counting sort of one row tile's input halo (output row y of image b, output columns x0 .. x0+nxs-1;
// channels-last input): KH halo rows of ncol = nxs + KW - 1 columns x C channels, each a contiguous
// run of ncol C bytes.  Buckets are (t, column) in t-major order, so for every t the entries of KW
// consecutive columns -- one position's receptive field at time t -- are one contiguous range.  Pass 1
// counts with shared-memory atomics, a warp scan turns the counts into bucket bases (u16; base[nb] = the
// total), pass 2 re-reads the latencies (L1) and places each spiking input's weight-row byte offset
// (ky KW C + j) row_bytes -- j = column C + c inside the halo row -- relative to the tile's first
// position; position xr reads row (ky KW + col - xr) C + c = that minus xr C, the (ky, kx, c) order of
// the channels-last weight rows.  Every halo input is sorted once for the tile's nxs positions instead
// of once per position (KH KW C entries each).
__device__ __forceinline__ void rows_sort(const WalkArgs& a, int b, int y, int x0, int ncol, const uint8_t* colof,
                                          uint32_t* cnt, uint16_t* base, uint16_t* list, int lane) {
  const int T = a.T, C = a.C, KW = a.KW;
  const int nb = T * ncol;
  for (int i = lane; i < nb; i += 32) cnt[i] = 0;
  __syncwarp();
  const int ix0 = x0 - a.pad;
  const int jlo = max(0, -ix0) * C, jhi = min(ncol, a.W - ix0) * C;  // the halo columns inside the input
  for (int ky = 0; ky < a.KH; ++ky) {
    const int iy = y - a.pad + ky;
    if (iy < 0 || iy >= a.H) continue;  // warp-uniform
    const uint8_t* rowp = a.lat_in + ((int64_t(b) * a.H + iy) * a.W + ix0) * C;
#pragma unroll 4
    for (int j = jlo + lane; j < jhi; j += 32) {
      const int l = __ldg(rowp + j);
      if (l < T) atomicAdd(&cnt[l * ncol + colof[j]], 1u);
    }
  }
  __syncwarp();
  const int per = (nb + 31) >> 5;
  const int k0 = min(nb, lane * per), k1 = min(nb, k0 + per);
  int sum = 0;
  for (int k = k0; k < k1; ++k) sum += int(cnt[k]);
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  int run = inc - sum;
  for (int k = k0; k < k1; ++k) {
    const int c = int(cnt[k]);
    base[k] = uint16_t(run);
    cnt[k] = uint32_t(run);
    run += c;
  }
  if (lane == 31) base[nb] = uint16_t(inc);
  __syncwarp();
  const uint32_t rb = uint32_t(a.row_bytes);
  for (int ky = 0; ky < a.KH; ++ky) {
    const int iy = y - a.pad + ky;
    if (iy < 0 || iy >= a.H) continue;
    const uint8_t* rowp = a.lat_in + ((int64_t(b) * a.H + iy) * a.W + ix0) * C;
    const uint32_t eb = uint32_t(ky * KW * C);
#pragma unroll 4
    for (int j = jlo + lane; j < jhi; j += 32) {
      const int l = __ldg(rowp + j);
      if (l < T) {
        const uint32_t slot = atomicAdd(&cnt[l * ncol + colof[j]], 1u);
        SNN_DCHECK(slot < uint32_t(a.KH * ncol * C));
        list[slot] = uint16_t((eb + uint32_t(j)) * rb);
      }
    }
  }
  __syncwarp();
}

}  // namespace snn
