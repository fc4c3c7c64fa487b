// conv_walk.cu -- the fast finite-threshold conv+fire kernel (a2 + a3; Eq. 2, P:122;
// DESIGN.md R3-R8, N1, K2).  Same arithmetic as conv_fire_kernel (the validation-mode kernel kept
// in conv_fire.cu for pot_out), organised for throughput:
//
//  * PPW output positions per warp, LPP = 32 / PPW lanes per position, FPL features per lane:
//    a warp-group of LPP lanes covers FGS = LPP * FPL features of one position.  Small layers
//    (F <= 32, e.g. C2 L1 F = 30) run 4 positions per warp with 4 features per lane, so the
//    per-input bookkeeping (list read, address) is shared by 4 features and the weight gather is
//    one conflict-free LDS.128 per lane.
//  * Counting sort of each receptive field by spike time into a shared-memory list: lane-private
//    u16 counters per (bucket, lane), rows scanned with vector loads (row strides chosen so 8 lanes
//    reading 8 rows hit 32 distinct banks), bucket starts by a segmented warp scan.
//  * Lockstep walk: every group consumes one pair of list entries per iteration (buckets are padded
//    to an even length with a zero-weight dummy row), accumulates exactly in int64 (units of 2^-31),
//    and at the end of a non-empty bucket tests the threshold and records (lat, v); a group stops as
//    soon as all its features fired or its list is exhausted.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace snn {

int weight_prep_launch(const float* w, int F, int R, int FGS, int n_groups, uint32_t* wq, cudaStream_t s);

constexpr int kWalkSmemLimit = 227 * 1024;

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

template <int FPL, int PPW>
__global__ void __launch_bounds__(1024, 1) conv_walk_kernel(const WalkArgs a) {
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
  uint16_t* cnt = reinterpret_cast<uint16_t*>(pb + a.cnt_off);      // [T][row_words*2] u16
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);  // [T+1]
  uint16_t* bsize = reinterpret_cast<uint16_t*>(pb + a.size_off);   // [T]
  uint16_t* list = reinterpret_cast<uint16_t*>(pb + a.list_off);    // [R+T+2]
  const int rw = a.row_words;  // u32 words per count row
  const int g = blockIdx.y;

  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wq + int64_t(g) * (R + 1) * FGS);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const int n4 = (R + 1) * FGS / 4;
    for (int i = tid; i < n4; i += blockDim.x) dst[i] = src[i];
    const int KK = a.KH * a.KW;
    for (int e = tid; e < R; e += blockDim.x) {
      const int c = e / KK, r = e - c * KK, ky = r / a.KW, kx = r - ky * a.KW;
      eoff[e] = c * a.H * a.W + ky * a.W + kx;
      ekk[e] = uint16_t((ky << 8) | kx);
    }
  }
  __syncthreads();

  const int64_t HoWo = int64_t(a.Ho) * a.Wo;
  const int64_t npos = int64_t(a.B) * HoWo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  const int fbase = g * FGS + gl * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < a.F) ? (1u << j) : 0u;
  constexpr unsigned kAll = (1u << FPL) - 1;
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1u) << (grp * LPP));
  const int64_t stride_w = int64_t(gridDim.x) * nwarps;

  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < npos; wi += stride_w) {
    const int64_t p = wi * PPW + grp;
    const bool pv = p < npos;
    const int b = pv ? int(p / HoWo) : 0;
    const int rem = pv ? int(p - int64_t(b) * HoWo) : 0;
    const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in = a.lat_in + int64_t(b) * CHW + int64_t(y0) * a.W + x0;
    const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;

    // ---------------- counting sort by spike time ----------------
    for (int t = 0; t < T; ++t) cnt[t * rw * 2 + gl] = 0;
    __syncwarp();
    if (pv) {
      for (int e = gl; e < R; e += LPP) {
        uint8_t l;
        if (interior) l = in[eoff[e]];
        else {
          const int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
          const bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
          l = ok ? in[eoff[e]] : kNoSpike;
        }
        if (l < T) cnt[l * rw * 2 + gl] += 1;
      }
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
    if (pv) {
      for (int e = gl; e < R; e += LPP) {
        uint8_t l;
        if (interior) l = in[eoff[e]];
        else {
          const int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
          const bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
          l = ok ? in[eoff[e]] : kNoSpike;
        }
        if (l < T) {
          const int c = cnt[l * rw * 2 + gl];
          cnt[l * rw * 2 + gl] = uint16_t(c + 1);
          list[c] = uint16_t(e);
        }
      }
    }
    for (int t = gl; t < T; t += LPP)
      if (bsize[t] & 1) list[start[t] + bsize[t]] = uint16_t(R);
    __syncwarp();

    // ---------------- lockstep walk ----------------
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
    const uint32_t* list32 = reinterpret_cast<const uint32_t*>(list);
    while (__any_sync(0xffffffffu, !done)) {
      if (!done) {
        const uint32_t pr = list32[i >> 1];
        uint32_t w0[FPL], w1[FPL];
        wgather<FPL>(wl + (pr & 0xFFFFu) * FGS, w0);
        wgather<FPL>(wl + (pr >> 16) * FGS, w1);
#pragma unroll
        for (int j = 0; j < FPL; ++j) acc[j] += uint64_t(w0[j]) + uint64_t(w1[j]);
        i += 2;
        if (i == bend) {  // end of the non-empty bucket t: threshold test (exact)
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
  int fpl, ppw, FGS, n_groups, nwarps, smem;
  WalkArgs a;
};

static bool walk_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, WalkPlan* pl) {
  WalkArgs& a = pl->a;
  a = WalkArgs{};
  a.B = B; a.C = C; a.H = H; a.W = W; a.pad = pad; a.F = F; a.KH = KH; a.KW = KW; a.T = T;
  a.Ho = H + 2 * pad - KH + 1; a.Wo = W + 2 * pad - KW + 1; a.R = C * KH * KW;
  const int R = a.R;
  struct Cand { int ppw, fpl; };
  // preference order: fewest feature groups first, then most features per lane
  const Cand cands[] = {{4, 4}, {2, 4}, {1, 4}, {4, 2}, {2, 2}, {1, 2}, {1, 1}};
  int best = -1, best_groups = 1 << 30, best_warps = 0;
  for (int ci = 0; ci < int(sizeof(cands) / sizeof(cands[0])); ++ci) {
    const int ppw = cands[ci].ppw, fpl = cands[ci].fpl, lpp = 32 / ppw, fgs = lpp * fpl;
    if (fgs > 32 && F <= fgs / 2) continue;  // half the lanes would idle
    const int rwords = lpp <= 16 ? 12 : 20;  // row stride (u32) of the count table
    const int pos_bytes = al16(T * rwords * 4) + al16((T + 1) * 2) + al16(T * 2) + al16((R + T + 2) * 2);
    const int warp_bytes = ppw * pos_bytes;
    const long ws_b = long(R + 1) * fgs * 4;
    const long fixed = al16(int(ws_b)) + al16(R * 4) + al16(R * 2);
    if (fixed + 8L * warp_bytes > kWalkSmemLimit) continue;
    long warps = (kWalkSmemLimit - fixed) / warp_bytes;
    if (warps > 32) warps = 32;
    const int groups = int(ceil_div(F, fgs));
    if (groups < best_groups || (groups == best_groups && warps > best_warps + 8)) {
      best = ci; best_groups = groups; best_warps = int(warps);
    }
  }
  if (best < 0) return false;
  pl->ppw = cands[best].ppw;
  pl->fpl = cands[best].fpl;
  const int lpp = 32 / pl->ppw;
  pl->FGS = lpp * pl->fpl;
  pl->n_groups = best_groups;
  pl->nwarps = best_warps;
  a.row_words = lpp <= 16 ? 12 : 20;
  int o = 0;
  a.cnt_off = o; o += al16(T * a.row_words * 4);
  a.start_off = o; o += al16((T + 1) * 2);
  a.size_off = o; o += al16(T * 2);
  a.list_off = o; o += al16((R + T + 2) * 2);
  a.pos_bytes = o;
  a.warp_bytes = pl->ppw * o;
  const long ws_b = long(R + 1) * pl->FGS * 4;
  a.off_eoff = al16(int(ws_b));
  a.off_ekk = a.off_eoff + al16(R * 4);
  a.off_warps = a.off_ekk + al16(R * 2);
  pl->smem = a.off_warps + pl->nwarps * a.warp_bytes;
  return true;
}

size_t conv_walk_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 0;
  return size_t(pl.n_groups) * (pl.a.R + 1) * pl.FGS * 4 + 256;
}

template <int FPL, int PPW>
static int walk_go(const WalkPlan& pl, int64_t npos, cudaStream_t s) {
  auto k = conv_walk_kernel<FPL, PPW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(walk): %s", cudaGetErrorString(e));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, pl.nwarps * 32, pl.smem);
  if (occ < 1) occ = 1;
  const int64_t per_group = ceil_div(ceil_div(npos, PPW), pl.nwarps);
  const int64_t want = ceil_div(int64_t(num_sms()) * occ, pl.n_groups);
  int gx = int(per_group < want ? per_group : want);
  if (gx < 1) gx = 1;
  k<<<dim3(gx, pl.n_groups), pl.nwarps * 32, pl.smem, s>>>(pl.a);
  note_launch();
  return check_launch("snn_conv_fire(walk)");
}

// Returns 1 if this path does not apply (caller falls back), else an SNN code.
int conv_walk_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                     cudaStream_t s) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 1;
  WalkArgs& a = pl.a;
  const size_t need = size_t(pl.n_groups) * (a.R + 1) * pl.FGS * 4;
  if (ws_bytes < need) return set_error(SNN_EWORKSPACE, "snn_conv_fire: workspace %zu < %zu", ws_bytes, need);
  a.lat_in = lat_in; a.lat_out = lat_out; a.v_out = v_out;
  a.wq = reinterpret_cast<const uint32_t*>(ws);
  const double tt = floor(double(theta) * 2147483648.0);
  a.thr = tt >= 9.0e18 ? INT64_MAX : (tt < -1.0 ? -1 : int64_t(tt));
  const int64_t npos = int64_t(B) * a.Ho * a.Wo;
  int rc = weight_prep_launch(w, F, a.R, pl.FGS, pl.n_groups, reinterpret_cast<uint32_t*>(ws), s);
  if (rc) return rc;
  switch (pl.ppw * 10 + pl.fpl) {
    case 44: return walk_go<4, 4>(pl, npos, s);
    case 24: return walk_go<4, 2>(pl, npos, s);
    case 14: return walk_go<4, 1>(pl, npos, s);
    case 42: return walk_go<2, 4>(pl, npos, s);
    case 22: return walk_go<2, 2>(pl, npos, s);
    case 12: return walk_go<2, 1>(pl, npos, s);
    default: return walk_go<1, 1>(pl, npos, s);
  }
}

}  // namespace snn
