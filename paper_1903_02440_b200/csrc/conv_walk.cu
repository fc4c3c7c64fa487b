// conv_walk.cu -- the throughput finite-threshold conv+fire path (a2 + a3; Eq. 2, P:122;
// DESIGN.md R3-R8, N1, K2).  Same arithmetic as conv_fire_kernel (the validation-mode kernel kept
// in conv_fire.cu for pot_out), organised for throughput:
//
//  * Receptive-field sort.  Each output position's C*KH*KW inputs are counting-sorted by spike time
//    (lane-private u16 counters per (bucket, lane), rows scanned with 16-byte loads, bucket starts by a
//    segmented warp scan; buckets padded to an even length with the zero-weight dummy row R).
//  * Walk.  PPW output positions per warp, LPP = 32/PPW lanes per position, FPL features per lane:
//    a group of LPP lanes covers FGS = LPP*FPL features of its position.  All groups advance in
//    lockstep, one pair of list entries per iteration: each lane gathers its FPL fixed-point weights
//    per input (one conflict-free LDS.64/128) and accumulates exactly in int64 (units of 2^-31); at
//    the end of every non-empty bucket it tests the threshold and records (lat, v); a group stops as
//    soon as all its features fired or its list is exhausted.
//  * Two schedules.  If the layer fits one feature group (weights of all F features in shared
//    memory), sort and walk are fused in one kernel (no list traffic).  Otherwise the sort runs ONCE
//    per position in rf_sort_kernel, which writes compact bucketed lists to a workspace chunk that
//    stays L2-resident, and conv_walk_kernel<PRE=true> streams them (16-byte prefetched loads) for
//    every feature group -- the sort is not repeated per group.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace snn {

int weight_prep_launch(const float* w, int F, int R, int FGS, int n_groups, uint32_t* wq, cudaStream_t s);

constexpr int kWalkSmemLimit = 227 * 1024;
constexpr size_t kListChunkBytes = size_t(48) << 20;  // sorted lists per chunk (L2-resident)

struct WalkArgs {
  const uint8_t* lat_in;
  int B, C, H, W, pad;
  int F, KH, KW, T, Ho, Wo, R;
  const uint32_t* wq;  // [n_groups][R+1][FGS]
  int64_t thr;
  uint8_t* lat_out;
  float* v_out;
  int off_eoff, off_ekk, off_warps, warp_bytes, pos_bytes;
  int cnt_off, start_off, size_off, list_off, row_words;
  // presorted lists: record of position p (chunk-relative) at lists + (p - p0) * rec (u16 units)
  uint16_t* lists;
  int rec, hdr;       // u16 per record; u16 of the header (bucket starts), multiple of 8
  int64_t p0, np;     // chunk of positions [p0, p0 + np)
};

static inline int al16(int x) { return (x + 15) & ~15; }

template <int FPL> struct WalkVec;
template <> struct WalkVec<1> { typedef uint32_t T; };
template <> struct WalkVec<2> { typedef uint2 T; };
template <> struct WalkVec<4> { typedef uint4 T; };

template <int FPL>
__device__ __forceinline__ void wgather(const uint32_t* p, uint32_t (&o)[FPL]) {
  typedef typename WalkVec<FPL>::T V;
  const V v = *reinterpret_cast<const V*>(p);
  if constexpr (FPL == 1) { o[0] = v; }
  else if constexpr (FPL == 2) { o[0] = v.x; o[1] = v.y; }
  else { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
}

__device__ __forceinline__ uint8_t rf_lat(const WalkArgs& a, const int32_t* eoff, const uint16_t* ekk,
                                          const uint8_t* in, bool interior, int y0, int x0, int e) {
  if (interior) return in[eoff[e]];
  const int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
  const bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
  return ok ? in[eoff[e]] : kNoSpike;
}

// Counting sort of one position's receptive field by a group of LPP lanes into (start, list).
template <int LPP>
__device__ __forceinline__ void rf_sort_group(const WalkArgs& a, const int32_t* eoff, const uint16_t* ekk, bool pv,
                                              const uint8_t* in, bool interior, int y0, int x0, int gl,
                                              uint16_t* cnt, uint16_t* start, uint16_t* bsize, uint16_t* list) {
  const int R = a.R, T = a.T, rw = a.row_words;
  for (int t = 0; t < T; ++t) cnt[t * rw * 2 + gl] = 0;
  __syncwarp();
  if (pv)
    for (int e = gl; e < R; e += LPP) {
      const uint8_t l = rf_lat(a, eoff, ekk, in, interior, y0, x0, e);
      if (l < T) cnt[l * rw * 2 + gl] += 1;
    }
  __syncwarp();
  int carry = 0;
  for (int tb = 0; tb < T; tb += LPP) {
    const int t = tb + gl;
    uint32_t words[LPP / 2];
    int tot = 0;
    if (t < T) {
      const uint32_t* row = reinterpret_cast<const uint32_t*>(cnt + t * rw * 2);
#pragma unroll
      for (int q = 0; q < LPP / 2; q += 4) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(row + q);
        words[q] = v4.x; words[q + 1] = v4.y; words[q + 2] = v4.z; words[q + 3] = v4.w;
      }
#pragma unroll
      for (int q = 0; q < LPP / 2; ++q) tot += int(words[q] & 0xFFFFu) + int(words[q] >> 16);
    }
    const int padded = tot + (tot & 1);
    int inc = padded;
#pragma unroll
    for (int o = 1; o < LPP; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o, LPP);
      if (gl >= o) inc += v;
    }
    const int st = carry + inc - padded;
    if (t < T) {
      start[t] = uint16_t(st);
      bsize[t] = uint16_t(tot);
      int run = st;
      uint32_t* row = reinterpret_cast<uint32_t*>(cnt + t * rw * 2);
#pragma unroll
      for (int q = 0; q < LPP / 2; ++q) {
        const int c0 = int(words[q] & 0xFFFFu), c1 = int(words[q] >> 16);
        words[q] = uint32_t(run) | (uint32_t(run + c0) << 16);
        run += c0 + c1;
      }
#pragma unroll
      for (int q = 0; q < LPP / 2; q += 4)
        *reinterpret_cast<uint4*>(row + q) = make_uint4(words[q], words[q + 1], words[q + 2], words[q + 3]);
    }
    carry += __shfl_sync(0xffffffffu, inc, LPP - 1, LPP);
  }
  if (gl == 0) start[T] = uint16_t(carry);
  __syncwarp();
  if (pv)
    for (int e = gl; e < R; e += LPP) {
      const uint8_t l = rf_lat(a, eoff, ekk, in, interior, y0, x0, e);
      if (l < T) {
        const int c = cnt[l * rw * 2 + gl];
        cnt[l * rw * 2 + gl] = uint16_t(c + 1);
        list[c] = uint16_t(e);
      }
    }
  for (int t = gl; t < T; t += LPP)
    if (bsize[t] & 1) list[start[t] + bsize[t]] = uint16_t(R);
  {  // pad the tail to a whole 8-entry block (the walk consumes blocks of 4 pairs)
    const int n = carry;
    for (int k = n + gl; k < ((n + 7) & ~7); k += LPP) list[k] = uint16_t(R);
  }
  __syncwarp();
}

__device__ __forceinline__ void rf_tables(const WalkArgs& a, int32_t* eoff, uint16_t* ekk) {
  const int KK = a.KH * a.KW;
  for (int e = threadIdx.x; e < a.R; e += blockDim.x) {
    const int c = e / KK, r = e - c * KK, ky = r / a.KW, kx = r - ky * a.KW;
    eoff[e] = c * a.H * a.W + ky * a.W + kx;
    ekk[e] = uint16_t((ky << 8) | kx);
  }
}

// ------------------------------------------------------------------------------------- sort only
template <int PPW>
__global__ void __launch_bounds__(512) rf_sort_kernel(const WalkArgs a) {
  constexpr int LPP = 32 / PPW;
  extern __shared__ __align__(16) unsigned char smem[];
  int32_t* eoff = reinterpret_cast<int32_t*>(smem + a.off_eoff);
  uint16_t* ekk = reinterpret_cast<uint16_t*>(smem + a.off_ekk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / LPP, gl = lane - grp * LPP;
  unsigned char* pb = smem + a.off_warps + warp * a.warp_bytes + grp * a.pos_bytes;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(pb + a.cnt_off);
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);
  uint16_t* bsize = reinterpret_cast<uint16_t*>(pb + a.size_off);
  uint16_t* list = reinterpret_cast<uint16_t*>(pb + a.list_off);
  rf_tables(a, eoff, ekk);
  __syncthreads();
  const int64_t HoWo = int64_t(a.Ho) * a.Wo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < a.np; wi += int64_t(gridDim.x) * nwarps) {
    const int64_t q = wi * PPW + grp;  // chunk-relative position
    const bool pv = q < a.np;
    const int p = int(a.p0 + q);
    const int b = pv ? p / int(HoWo) : 0;
    const int rem = pv ? p - b * int(HoWo) : 0;
    const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in = a.lat_in + int64_t(b) * CHW + int64_t(y0) * a.W + x0;
    const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;
    rf_sort_group<LPP>(a, eoff, ekk, pv, in, interior, y0, x0, gl, cnt, start, bsize, list);
    if (pv) {  // record = [header (T+1 starts, padded to hdr)][entries (start[T] of them)]
      uint16_t* rec = a.lists + q * a.rec;
      for (int t = gl; t <= a.T; t += LPP) rec[t] = start[t];
      const int n8 = (int(start[a.T]) + 7) >> 3;  // whole 8-entry blocks (tail padded with R)
      const uint4* src = reinterpret_cast<const uint4*>(list);
      uint4* dst = reinterpret_cast<uint4*>(rec + a.hdr);
      for (int k = gl; k < n8; k += LPP) dst[k] = src[k];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------- walk
template <int FPL> struct WalkThreads { static constexpr int v = FPL == 4 ? 768 : 1024; };

template <int FPL, int PPW, bool PRE>
__global__ void __launch_bounds__(WalkThreads<FPL>::v, 1) conv_walk_kernel(const WalkArgs a) {
  constexpr int LPP = 32 / PPW;
  constexpr int FGS = LPP * FPL;
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, T = a.T;
  const uint32_t* Ws = reinterpret_cast<const uint32_t*>(smem);
  int32_t* eoff = reinterpret_cast<int32_t*>(smem + a.off_eoff);
  uint16_t* ekk = reinterpret_cast<uint16_t*>(smem + a.off_ekk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / LPP, gl = lane - grp * LPP;
  unsigned char* pb = smem + a.off_warps + warp * a.warp_bytes + grp * a.pos_bytes;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(pb + a.cnt_off);
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);
  uint16_t* bsize = reinterpret_cast<uint16_t*>(pb + a.size_off);
  uint16_t* list = reinterpret_cast<uint16_t*>(pb + a.list_off);
  const int g = blockIdx.y;
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wq + int64_t(g) * (R + 1) * FGS);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const int n4 = (R + 1) * FGS / 4;
    for (int i = tid; i < n4; i += blockDim.x) dst[i] = src[i];
    if (!PRE) rf_tables(a, eoff, ekk);
  }
  __syncthreads();

  const int64_t HoWo = int64_t(a.Ho) * a.Wo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  const int fbase = g * FGS + gl * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < a.F) ? (1u << j) : 0u;
  constexpr unsigned kAll = (1u << FPL) - 1;
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1u) << (grp * LPP));
  const int64_t stride_w = int64_t(gridDim.x) * nwarps;

  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < a.np; wi += stride_w) {
    const int64_t q = wi * PPW + grp;
    const bool pv = q < a.np;
    const int p = int(a.p0 + q);  // npos < 2^31 (checked by the planner)
    const int b = pv ? p / int(HoWo) : 0;
    const int rem = pv ? p - b * int(HoWo) : 0;
    const uint16_t* rec = nullptr;
    if constexpr (PRE) {
      rec = a.lists + (pv ? q : 0) * a.rec;
      for (int t = gl; t <= T; t += LPP) start[t] = pv ? rec[t] : 0;
      __syncwarp();
    } else {
      const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
      const int y0 = y - a.pad, x0 = x - a.pad;
      const uint8_t* in = a.lat_in + int64_t(b) * CHW + int64_t(y0) * a.W + x0;
      const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;
      rf_sort_group<LPP>(a, eoff, ekk, pv, in, interior, y0, x0, gl, cnt, start, bsize, list);
    }

    uint64_t acc[FPL];
    uint8_t lo[FPL];
    float vo[FPL];
#pragma unroll
    for (int j = 0; j < FPL; ++j) { acc[j] = 0; lo[j] = kNoSpike; vo[j] = 0.0f; }
    unsigned fired = ~valid & kAll;
    const int total = pv ? int(start[T]) : 0;
    int i = 0, t = 0;
    int bend = start[1];
    if (bend == 0) {  // bucket 0 empty: P[0] = 0 may still exceed a negative threshold
      if (int64_t(0) > a.thr) {
#pragma unroll
        for (int j = 0; j < FPL; ++j)
          if (!(fired >> j & 1)) { fired |= 1u << j; lo[j] = 0; vo[j] = 0.0f; }
      }
      while (t < T && int(start[t + 1]) == 0) ++t;
      bend = t < T ? int(start[t + 1]) : 0;
    }
    bool done = (t >= T) || (i >= total) || !pv || __all_sync(gmask, fired == kAll);
    const uint32_t* wl = Ws + gl * FPL;
    const uint4* list4 = reinterpret_cast<const uint4*>(list);
    const uint4* gl4 = PRE ? reinterpret_cast<const uint4*>(rec + a.hdr) : nullptr;
    uint4 cur = make_uint4(0, 0, 0, 0), nxt = make_uint4(0, 0, 0, 0);
    if (PRE && !done) { cur = gl4[0]; nxt = gl4[1]; }
    while (__any_sync(0xffffffffu, !done)) {
      if (!done) {
        // one block = 4 pairs = 8 inputs: all 8 gathers are issued before the ordered
        // accumulate / threshold sequence (buckets end on pair boundaries)
        uint4 blk;
        if constexpr (PRE) { blk = cur; cur = nxt; nxt = gl4[(i >> 3) + 2]; }
        else blk = list4[i >> 3];
        const uint32_t prs[4] = {blk.x, blk.y, blk.z, blk.w};
        uint32_t wv[8][FPL];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          wgather<FPL>(wl + (prs[k] & 0xFFFFu) * FGS, wv[2 * k]);
          wgather<FPL>(wl + (prs[k] >> 16) * FGS, wv[2 * k + 1]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!done) {
#pragma unroll
            for (int j = 0; j < FPL; ++j) acc[j] += uint64_t(wv[2 * k][j]) + uint64_t(wv[2 * k + 1][j]);
            i += 2;
            if (i == bend) {  // end of the non-empty bucket t: exact threshold test
#pragma unroll
              for (int j = 0; j < FPL; ++j) {
                if (!(fired >> j & 1) && int64_t(acc[j]) > a.thr) {
                  fired |= 1u << j;
                  lo[j] = uint8_t(t);
                  vo[j] = fixed_to_float(int64_t(acc[j]));
                }
              }
              ++t;
              while (t < T && int(start[t + 1]) == i) ++t;  // skip empty buckets
              bend = t < T ? int(start[t + 1]) : 0;
              done = (t >= T) || __all_sync(gmask, fired == kAll);
            }
          }
        }
      }
    }
    if (pv) {
#pragma unroll
      for (int j = 0; j < FPL; ++j) {
        if (valid >> j & 1) {
          const int64_t o = (int64_t(b) * a.F + fbase + j) * HoWo + rem;
          a.lat_out[o] = lo[j];
          a.v_out[o] = vo[j];
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------- host
struct WalkPlan {
  int fpl, ppw, FGS, n_groups, nwarps, smem;  // walk kernel
  int sort_ppw, sort_nwarps, sort_smem;        // sort kernel (presorted mode)
  bool pre;
  int64_t chunk;                               // positions per list chunk
  WalkArgs a;                                  // walk kernel arguments / smem layout
  WalkArgs sa;                                 // sort kernel arguments / smem layout
};

static int pos_scratch_bytes(int T, int R, int lpp, int rw, WalkArgs* a) {
  int o = 0, c0, c1, c2, c3;
  c0 = o; o += al16(T * rw * 4);
  c1 = o; o += al16((T + 1) * 2);
  c2 = o; o += al16(T * 2);
  c3 = o; o += al16((R + T + 8) * 2);
  (void)lpp;
  if (a) { a->cnt_off = c0; a->start_off = c1; a->size_off = c2; a->list_off = c3; a->pos_bytes = o; }
  return o;
}

static bool walk_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, WalkPlan* pl) {
  WalkArgs& a = pl->a;
  a = WalkArgs{};
  if (int64_t(B) * (H + 2 * pad - KH + 1) * (W + 2 * pad - KW + 1) >= (int64_t(1) << 31)) return false;
  a.B = B; a.C = C; a.H = H; a.W = W; a.pad = pad; a.F = F; a.KH = KH; a.KW = KW; a.T = T;
  a.Ho = H + 2 * pad - KH + 1; a.Wo = W + 2 * pad - KW + 1; a.R = C * KH * KW;
  const int R = a.R;
  const long tables = al16(R * 4) + al16(R * 2);
  struct Cand { int ppw, fpl; };
  const Cand cands[] = {{4, 4}, {2, 4}, {1, 4}, {4, 2}, {2, 2}, {1, 2}, {1, 1}};
  // 1) fused: all features in one group with >= 8 warps of sort scratch
  int best = -1, best_warps = 0;
  for (const Cand& c : cands) {
    const int lpp = 32 / c.ppw, fgs = lpp * c.fpl;
    if (fgs < F) continue;
    if (fgs > 32 && F <= fgs / 2) continue;
    const int rw = lpp <= 16 ? 12 : 20;
    const int wb = c.ppw * pos_scratch_bytes(T, R, lpp, rw, nullptr);
    const long fixed = al16(int(long(R + 1) * fgs * 4)) + tables;
    if (fixed + 8L * wb > kWalkSmemLimit) continue;
    long warps = (kWalkSmemLimit - fixed) / wb;
    const int wcap = c.fpl == 4 ? 24 : 32;
    if (warps > wcap) warps = wcap;
    if (best < 0 || warps > best_warps + 8) { best = int(&c - cands); best_warps = int(warps); }
  }
  if (best >= 0) {
    pl->pre = false;
    pl->ppw = cands[best].ppw; pl->fpl = cands[best].fpl;
    const int lpp = 32 / pl->ppw;
    pl->FGS = lpp * pl->fpl; pl->n_groups = 1; pl->nwarps = best_warps;
    a.row_words = lpp <= 16 ? 12 : 20;
    pos_scratch_bytes(T, R, lpp, a.row_words, &a);
    a.warp_bytes = pl->ppw * a.pos_bytes;
    a.off_eoff = al16(int(long(R + 1) * pl->FGS * 4));
    a.off_ekk = a.off_eoff + al16(R * 4);
    a.off_warps = a.off_ekk + al16(R * 2);
    pl->smem = a.off_warps + pl->nwarps * a.warp_bytes;
    a.np = int64_t(B) * a.Ho * a.Wo;
    pl->chunk = a.np;
    return true;
  }
  // 2) presorted: sort once per position, walk per feature group (PPW = 1, the largest FPL that fits)
  const int fpls[3] = {4, 2, 1};
  for (int k = 0; k < 3; ++k) {
    const int fpl = fpls[k], fgs = 32 * fpl;
    if (fgs > 32 && F <= fgs / 2) continue;
    const long wsb = long(R + 1) * fgs * 4;
    const int hdr_bytes = al16((T + 1) * 2);
    if (al16(int(wsb)) + 32L * hdr_bytes > kWalkSmemLimit) continue;
    pl->pre = true;
    pl->ppw = 1; pl->fpl = fpl; pl->FGS = fgs;
    pl->n_groups = int(ceil_div(F, fgs));
    pl->nwarps = fpl == 4 ? 24 : 32;
    a.cnt_off = 0; a.start_off = 0; a.size_off = 0; a.list_off = 0;
    a.pos_bytes = hdr_bytes; a.warp_bytes = hdr_bytes;
    a.off_eoff = al16(int(wsb)); a.off_ekk = a.off_eoff; a.off_warps = a.off_eoff;
    pl->smem = a.off_warps + pl->nwarps * a.warp_bytes;
    a.hdr = int(ceil_div(T + 1, 8)) * 8;
    a.rec = a.hdr + int(ceil_div(R + T + 8, 8)) * 8;
    // sort kernel: 16 warps, 1 position per warp (PPW 1) or 4 per warp for small receptive fields
    pl->sort_ppw = R <= 256 ? 4 : 1;
    pl->sort_nwarps = 16;
    const int slpp = 32 / pl->sort_ppw;
    WalkArgs& sa = pl->sa;
    sa = a;
    sa.row_words = slpp <= 16 ? 12 : 20;
    pos_scratch_bytes(T, R, slpp, sa.row_words, &sa);
    sa.warp_bytes = pl->sort_ppw * sa.pos_bytes;
    sa.off_eoff = 0;
    sa.off_ekk = al16(R * 4);
    sa.off_warps = sa.off_ekk + al16(R * 2);
    pl->sort_smem = sa.off_warps + pl->sort_nwarps * sa.warp_bytes;
    const int64_t npos = int64_t(B) * a.Ho * a.Wo;
    int64_t ch = int64_t(kListChunkBytes / (size_t(a.rec) * 2));
    if (ch < 1024) ch = 1024;
    pl->chunk = ch < npos ? ch : npos;
    return true;
  }
  return false;
}

size_t conv_walk_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 0;
  size_t n = size_t(pl.n_groups) * (pl.a.R + 1) * pl.FGS * 4;
  n = (n + 255) & ~size_t(255);
  if (pl.pre) n += size_t(pl.chunk) * pl.a.rec * 2 + 256;  // + slack for the prefetch past the end
  return n + 256;
}

template <int FPL, int PPW, bool PRE>
static int walk_go(const WalkPlan& pl, const WalkArgs& a, cudaStream_t s) {
  auto k = conv_walk_kernel<FPL, PPW, PRE>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(walk): %s", cudaGetErrorString(e));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, pl.nwarps * 32, pl.smem);
  if (occ < 1) occ = 1;
  const int64_t per_group = ceil_div(ceil_div(a.np, PPW), pl.nwarps);
  const int64_t want = ceil_div(int64_t(num_sms()) * occ, pl.n_groups);
  int gx = int(per_group < want ? per_group : want);
  if (gx < 1) gx = 1;
  k<<<dim3(gx, pl.n_groups), pl.nwarps * 32, pl.smem, s>>>(a);
  note_launch();
  return check_launch("snn_conv_fire(walk)");
}

template <int PPW>
static int sort_go(const WalkPlan& pl, const WalkArgs& a, cudaStream_t s) {
  auto k = rf_sort_kernel<PPW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.sort_smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(sort): %s", cudaGetErrorString(e));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, pl.sort_nwarps * 32, pl.sort_smem);
  if (occ < 1) occ = 1;
  int64_t blocks = ceil_div(ceil_div(a.np, PPW), pl.sort_nwarps);
  const int64_t cap = int64_t(num_sms()) * occ;
  if (blocks > cap) blocks = cap;
  k<<<int(blocks), pl.sort_nwarps * 32, pl.sort_smem, s>>>(a);
  note_launch();
  return check_launch("snn_conv_fire(sort)");
}

// Returns 1 if this path does not apply (caller falls back), else an SNN code.
int conv_walk_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                     cudaStream_t s) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 1;
  WalkArgs a = pl.a;
  size_t wq_bytes = (size_t(pl.n_groups) * (a.R + 1) * pl.FGS * 4 + 255) & ~size_t(255);
  const size_t need = wq_bytes + (pl.pre ? size_t(pl.chunk) * a.rec * 2 + 256 : 0);
  if (ws_bytes < need) return set_error(SNN_EWORKSPACE, "snn_conv_fire: workspace %zu < %zu", ws_bytes, need);
  a.lat_in = lat_in; a.lat_out = lat_out; a.v_out = v_out;
  a.wq = reinterpret_cast<const uint32_t*>(ws);
  a.lists = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(ws) + wq_bytes);
  const double tt = floor(double(theta) * 2147483648.0);
  a.thr = tt >= 9.0e18 ? INT64_MAX : (tt < -1.0 ? -1 : int64_t(tt));
  const int64_t npos = int64_t(B) * a.Ho * a.Wo;
  int rc = weight_prep_launch(w, F, a.R, pl.FGS, pl.n_groups, reinterpret_cast<uint32_t*>(ws), s);
  if (rc) return rc;
  if (!pl.pre) {
    a.p0 = 0; a.np = npos;
    switch (pl.ppw * 10 + pl.fpl) {
      case 44: return walk_go<4, 4, false>(pl, a, s);
      case 24: return walk_go<4, 2, false>(pl, a, s);
      case 14: return walk_go<4, 1, false>(pl, a, s);
      case 42: return walk_go<2, 4, false>(pl, a, s);
      case 22: return walk_go<2, 2, false>(pl, a, s);
      case 12: return walk_go<2, 1, false>(pl, a, s);
      default: return walk_go<1, 1, false>(pl, a, s);
    }
  }
  WalkArgs sa = pl.sa;
  sa.lat_in = lat_in; sa.lists = a.lists; sa.hdr = a.hdr; sa.rec = a.rec;
  for (int64_t p0 = 0; p0 < npos; p0 += pl.chunk) {
    a.p0 = p0;
    a.np = npos - p0 < pl.chunk ? npos - p0 : pl.chunk;
    sa.p0 = a.p0; sa.np = a.np;
    rc = pl.sort_ppw == 4 ? sort_go<4>(pl, sa, s) : sort_go<1>(pl, sa, s);
    if (rc) return rc;
    switch (pl.fpl) {
      case 4: rc = walk_go<4, 1, true>(pl, a, s); break;
      case 2: rc = walk_go<2, 1, true>(pl, a, s); break;
      default: rc = walk_go<1, 1, true>(pl, a, s); break;
    }
    if (rc) return rc;
  }
  return SNN_OK;
}

}  // namespace snn
