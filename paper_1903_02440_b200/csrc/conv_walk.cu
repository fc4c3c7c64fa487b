// conv_walk.cu -- the throughput finite-threshold conv+fire path (a2 + a3; Eq. 2, P:122;
// DESIGN.md R3-R8, N1, K2).  Same arithmetic as conv_fire_kernel (the validation-mode kernel kept
// in conv_fire.cu for pot_out), organised for throughput:
//
//  * Receptive-field sort.  Each output position's C*KH*KW inputs are counting-sorted by spike time
//    (lane-private u16 counters per (bucket, lane), rows scanned with 16-byte loads, bucket starts by a
//    segmented warp scan).  The sorted list holds u32 BYTE OFFSETS of the inputs' weight rows in the
//    shared-memory weight slice (so the walk's gather address is one add); every bucket is padded to
//    an even length with the zero-weight row R (bucket ends fall on pair boundaries) and the tail to
//    whole 8-entry blocks.
//  * Walk.  PPW output positions per warp, LPP = 32/PPW lanes per position, FPL features per lane:
//    a group of LPP lanes covers FGS = LPP*FPL features of its position.  The list is consumed in
//    blocks of 8 inputs; each lane gathers its FPL fixed-point weights per input (one conflict-free
//    LDS.64/128) and sums the block exactly (int64, units of 2^-31, three-input adds).  Because every
//    weight is >= 0 the potential is monotone along the list, so a threshold test inside a block can
//    only fire if the potential at the block END exceeds the threshold for an unfired feature; and a
//    test is only due at a bucket end.  Blocks with no crossing, or with no bucket end strictly
//    inside, are therefore added whole (a test at most at the block end); only a block with both is
//    walked pair by pair with the exact test at each bucket end (K3).  A group stops as
//    soon as all its features fired or its list is exhausted.
//  * Two schedules.  If the layer fits one feature group (weights of all F features in shared
//    memory), sort and walk are fused in one kernel (no list traffic).  Otherwise the sort runs ONCE
//    per position in rf_sort_kernel, which writes compact bucketed lists to a workspace chunk (up to
//    512 MB: fewer, larger chunks measured faster than L2-sized ones, whose per-launch tails cost more
//    than the HBM round trip saves), and conv_walk_kernel<PRE=true> streams them through a per-warp
//    cp.async ring for every feature group -- the sort is not repeated per group.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace snn {

int weight_prep_launch(const float* w, int F, int R, int FGS, int n_groups, uint32_t* wq, cudaStream_t s);

constexpr int kWalkSmemLimit = 227 * 1024;
constexpr size_t kListChunkBytes = size_t(512) << 20;  // sorted lists per chunk (measured: fewer, larger chunks win;
                                                        // the lists stream from HBM either way)
constexpr int kBlk = 8;                               // list entries per gather block
constexpr int kIt = 16;                               // list entries per walk iteration (lists padded to this)
constexpr int kListSlack = 2048;                      // bytes read past the last record (prefetch)

struct WalkArgs {
  const uint8_t* lat_in;
  int B, C, H, W, pad;
  int F, KH, KW, T, Ho, Wo, R;
  const uint32_t* wq;  // [n_groups][R+1][FGS]
  int64_t thr;
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

__device__ __forceinline__ uint8_t rf_lat(const WalkArgs& a, const int32_t* eoff, const uint16_t* ekk,
                                          const uint8_t* in, bool interior, int y0, int x0, int e) {
  if (interior) return in[eoff[e]];
  const int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
  const bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
  return ok ? in[eoff[e]] : kNoSpike;
}

// Counting sort of one position's receptive field by a group of LPP lanes into (start, list).
// Pass 1 counts the spiking inputs of each bucket with shared-memory atomics (independent, no
// read-modify-write chains in the lane); the counts are scanned (each bucket padded to an even
// length with the zero-weight row R, so every bucket end is on a pair boundary) into the bucket
// starts; pass 2 re-reads the latencies (L1-resident) and takes each entry's slot with an atomic on
// the bucket's running position.  Entries are weight-row byte offsets e * row_bytes; the tail is
// padded to a whole walk iteration.  The order inside a bucket is whatever the atomics gave: it does
// not change any result (the sum at a bucket end is exact and order-free).
template <int LPP>
__device__ __forceinline__ void rf_sort_group(const WalkArgs& a, const int32_t* eoff, const uint16_t* ekk, bool pv,
                                              const uint8_t* in, bool interior, int y0, int x0, int gl,
                                              uint32_t* cnt, uint16_t* start, uint32_t* list) {
  const int R = a.R, T = a.T;
  const uint32_t rb = uint32_t(a.row_bytes);
  for (int t = gl; t < T; t += LPP) cnt[t] = 0;
  __syncwarp();
  if (pv) {
#pragma unroll 4
    for (int e = gl; e < R; e += LPP) {
      const int l = rf_lat(a, eoff, ekk, in, interior, y0, x0, e);
      if (l < T) atomicAdd(&cnt[l], 1u);
    }
  }
  __syncwarp();
  int carry = 0;
  for (int tb = 0; tb < T; tb += LPP) {
    const int t = tb + gl;
    const int tot = t < T ? int(cnt[t]) : 0;
    const int padded = tot + (tot & 1);  // buckets padded to even length: every bucket end is on a pair boundary
    int inc = padded;
#pragma unroll
    for (int o = 1; o < LPP; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o, LPP);
      if (gl >= o) inc += v;
    }
    const int st = carry + inc - padded;
    if (t < T) {
      start[t] = uint16_t(st);
      cnt[t] = uint32_t(st);                           // pass 2: running slot of the bucket
      if (tot & 1) list[st + tot] = uint32_t(R) * rb;  // the pad entry: zero-weight row
    }
    carry += __shfl_sync(0xffffffffu, inc, LPP - 1, LPP);
  }
  if (gl == 0) start[T] = uint16_t(carry);
  __syncwarp();
  if (pv) {
#pragma unroll 4
    for (int e = gl; e < R; e += LPP) {
      const int l = rf_lat(a, eoff, ekk, in, interior, y0, x0, e);
      if (l < T) list[atomicAdd(&cnt[l], 1u)] = uint32_t(e) * rb;
    }
  }
  {  // pad the tail to a whole walk iteration with the zero-weight row R
    const int n = carry;
    for (int k = n + gl; k < ((n + kIt - 1) & ~(kIt - 1)); k += LPP) list[k] = uint32_t(R) * rb;
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
  uint32_t* cnt = reinterpret_cast<uint32_t*>(pb + a.cnt_off);
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);
  uint32_t* list = reinterpret_cast<uint32_t*>(pb + a.list_off);
  rf_tables(a, eoff, ekk);
  __syncthreads();
  const int HoWo = a.Ho * a.Wo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < a.np; wi += int64_t(gridDim.x) * nwarps) {
    const int64_t q = wi * PPW + grp;  // chunk-relative position
    const bool pv = q < a.np;
    const int p = int(a.p0 + q);
    const int b = pv ? p / HoWo : 0;
    const int rem = pv ? p - b * HoWo : 0;
    const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in = a.lat_in + int64_t(b) * CHW + int64_t(y0) * a.W + x0;
    const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;
    rf_sort_group<LPP>(a, eoff, ekk, pv, in, interior, y0, x0, gl, cnt, start, list);
    if (pv) {  // record = [header: T+1 u16 starts, 16-aligned][entries: u32, whole blocks]
      unsigned char* rec = a.lists + q * a.rec;
      uint16_t* hdr = reinterpret_cast<uint16_t*>(rec);
      for (int t = gl; t <= a.T; t += LPP) hdr[t] = start[t];
      const int n4 = ((int(start[a.T]) + kIt - 1) / kIt) * (kIt / 4);  // uint4 per walk iteration
      const uint4* src = reinterpret_cast<const uint4*>(list);
      uint4* dst = reinterpret_cast<uint4*>(rec + a.hdr);
      for (int k = gl; k < n4; k += LPP) dst[k] = src[k];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------- walk
template <int FPL, bool PRE> struct WalkThreads { static constexpr int v = FPL == 4 ? (PRE ? 640 : 768) : 1024; };

// Fire every unfired feature whose potential at the end of bucket t exceeds the threshold.
template <int FPL>
__device__ __forceinline__ void fire_at(const uint64_t (&acc)[FPL], int64_t thr, int t, unsigned& fired,
                                        uint32_t& lo, float (&vo)[FPL]) {
#pragma unroll
  for (int j = 0; j < FPL; ++j) {
    if (!(fired >> j & 1) && int64_t(acc[j]) > thr) {
      fired |= 1u << j;
      lo = (lo & ~(0xFFu << (8 * j))) | (uint32_t(t) << (8 * j));
      vo[j] = fixed_to_float(int64_t(acc[j]));
    }
  }
}

// One 8-input block of the walk (entries e0, e1: weight-row byte offsets).  The bucket ends inside
// the block are known to the whole group beforehand (endm: bit m = a bucket ends after pair m, its
// first-spike index in byte m of tpk).  Each lane sums its features' 8 weights exactly; if no
// unfired feature of the lane then exceeds the threshold, no test inside the block could fire
// (potentials only grow along the list) and the block is taken whole; otherwise the lane re-adds it
// pair by pair from the same registers and tests at every bucket end (K3).  Lanes decide
// independently (no vote): the group's bookkeeping does not depend on the branch taken.
template <int FPL>
__device__ __forceinline__ void walk_block(const unsigned char* wl, const uint4& e0, const uint4& e1, unsigned endm,
                                           uint32_t tpk, int64_t thr, uint64_t (&acc)[FPL], unsigned& fired,
                                           uint32_t& lo, float (&vo)[FPL]) {
  const uint32_t off[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
  uint32_t wv[8][FPL];
#pragma unroll
  for (int k = 0; k < 8; ++k) wgather<FPL>(wl + off[k], wv[k]);
  uint64_t s[FPL];
  bool hit = false;
#pragma unroll
  for (int j = 0; j < FPL; ++j) {
    s[j] = acc[j] + (uint64_t(wv[0][j]) + wv[1][j]) + (uint64_t(wv[2][j]) + wv[3][j]) +
           (uint64_t(wv[4][j]) + wv[5][j]) + (uint64_t(wv[6][j]) + wv[7][j]);
    hit |= !(fired >> j & 1) && int64_t(s[j]) > thr;
  }
  if (hit && endm) {
    if (endm & 7u) {  // a bucket ends strictly inside the block: pair by pair
#pragma unroll
      for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int j = 0; j < FPL; ++j) acc[j] += uint64_t(wv[2 * m][j]) + wv[2 * m + 1][j];
        if (endm >> m & 1) fire_at<FPL>(acc, thr, int((tpk >> (8 * m)) & 0xFFu), fired, lo, vo);
      }
    } else {  // the only bucket end is the block end
      fire_at<FPL>(s, thr, int(tpk >> 24), fired, lo, vo);
    }
  }
#pragma unroll
  for (int j = 0; j < FPL; ++j) acc[j] = s[j];
}

template <int FPL, int PPW, bool PRE>
__global__ void __launch_bounds__(WalkThreads<FPL, PRE>::v, 1) conv_walk_kernel(const WalkArgs a) {
  constexpr int LPP = 32 / PPW;
  constexpr int FGS = LPP * FPL;
  constexpr unsigned kAll = (1u << FPL) - 1;
  static_assert(!PRE || PPW == 1, "presorted walk: one position per warp");
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, T = a.T;
  int32_t* eoff = reinterpret_cast<int32_t*>(smem + a.off_eoff);
  uint16_t* ekk = reinterpret_cast<uint16_t*>(smem + a.off_ekk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / LPP, gl = lane - grp * LPP;
  unsigned char* pb = smem + a.off_warps + warp * a.warp_bytes + grp * a.pos_bytes;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(pb + a.cnt_off);
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);
  uint32_t* list = reinterpret_cast<uint32_t*>(pb + a.list_off);  // fused: the sorted list; PRE: the ring
  const int g = blockIdx.y;
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wq + int64_t(g) * (R + 1) * FGS);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const int n4 = (R + 1) * FGS / 4;
    for (int i = tid; i < n4; i += blockDim.x) dst[i] = src[i];
    if (!PRE) rf_tables(a, eoff, ekk);
  }
  __syncthreads();

  const int HoWo = a.Ho * a.Wo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  const int fbase = g * FGS + gl * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < a.F) ? (1u << j) : 0u;
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1u) << (grp * LPP));
  const int64_t stride_w = int64_t(gridDim.x) * nwarps;
  const int64_t thr = a.thr;
  const unsigned char* wl = smem + gl * FPL * 4;  // this lane's features in weight row 0

  // PRE: two per-warp position buffers [header | first npre entries], each filled by one bulk copy
  // (TMA, mbarrier completion) issued one position ahead, so the list of the next position streams in
  // while this one is walked; entries past npre (rare long walks) are read from global memory
  uint64_t* pmb = reinterpret_cast<uint64_t*>(pb);
  unsigned char* pbuf = pb + 16;
  if constexpr (PRE) {
    if (lane == 0) {
      mbar_init(smem_u32(&pmb[0]), 1);
      mbar_init(smem_u32(&pmb[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const int64_t w0 = int64_t(blockIdx.x) * nwarps + warp;
      if (w0 < a.np) {
        mbar_expect_tx(smem_u32(&pmb[0]), uint32_t(a.buf_bytes));
        bulk_g2s(smem_u32(pbuf), a.lists + w0 * a.rec, uint32_t(a.buf_bytes), smem_u32(&pmb[0]));
      }
    }
    __syncwarp();
  }
  int npos_done = 0;
  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < a.np; wi += stride_w, ++npos_done) {
    const int64_t q = wi * PPW + grp;
    const bool pv = q < a.np;
    const int p = int(a.p0 + q);  // npos < 2^31 (checked by the planner)
    const int b = pv ? p / HoWo : 0;
    const int rem = pv ? p - b * HoWo : 0;
    const unsigned char* ent = nullptr;   // PRE: this position's entries in global memory
    const unsigned char* sent = nullptr;  // PRE: its first npre entries in shared memory
    if constexpr (PRE) {
      const int bi = npos_done & 1;
      if (lane == 0 && (wi + stride_w) * PPW < a.np) {  // prefetch the next position into the other buffer
        mbar_expect_tx(smem_u32(&pmb[bi ^ 1]), uint32_t(a.buf_bytes));
        bulk_g2s(smem_u32(pbuf + (bi ^ 1) * a.buf_bytes), a.lists + (wi + stride_w) * a.rec, uint32_t(a.buf_bytes),
                 smem_u32(&pmb[bi ^ 1]));
      }
      mbar_wait(smem_u32(&pmb[bi]), (npos_done >> 1) & 1);
      start = reinterpret_cast<uint16_t*>(pbuf + bi * a.buf_bytes);
      sent = pbuf + bi * a.buf_bytes + a.hdr;
      ent = a.lists + q * a.rec + a.hdr;
    } else {
      const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
      const int y0 = y - a.pad, x0 = x - a.pad;
      const uint8_t* in = a.lat_in + int64_t(b) * CHW + int64_t(y0) * a.W + x0;
      const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;
      rf_sort_group<LPP>(a, eoff, ekk, pv, in, interior, y0, x0, gl, cnt, start, list);
    }

    uint64_t acc[FPL];
    uint32_t lo = 0xFFFFFFFFu;  // byte j = lat of feature j (255 = no spike)
    float vo[FPL];
#pragma unroll
    for (int j = 0; j < FPL; ++j) { acc[j] = 0; vo[j] = 0.0f; }
    unsigned fired = ~valid & kAll;
    const int total = pv ? int(start[T]) : 0;
    if (pv && int(start[1]) == 0 && int64_t(0) > thr) {  // empty bucket 0: P[0] = 0 > a negative threshold
#pragma unroll
      for (int j = 0; j < FPL; ++j)
        if (!(fired >> j & 1)) lo &= ~(0xFFu << (8 * j));
      fired = kAll;
    }
    bool done = !pv || total == 0;  // group-uniform, like every later update of done
    {
      const unsigned nd = __ballot_sync(0xffffffffu, fired != kAll);
      if ((nd & gmask) == 0) done = true;  // all features of the group fired (or are padding)
    }
    int i = 0, t = 0, it = 0;
    while (t < T && int(start[t + 1]) == 0) ++t;  // leading empty buckets (handled above)
    int bend = t < T ? int(start[t + 1]) : 0x7FFFFFFF;  // end of the current non-empty bucket t
    int guard = (total + kIt - 1) / kIt + 2;  // iterations this group can take (a bug trap, never hit)
    // Every vote below is a full-warp ballot at a converged point; done is group-uniform.
    while (true) {
      if (__ballot_sync(0xffffffffu, !done) == 0) break;
      uint4 cur[4];  // this iteration's 16 entries: shared memory (PRE past npre: global memory)
      if (PRE && it * kIt >= a.npre) {
        const uint4* g4 = reinterpret_cast<const uint4*>(ent + it * kIt * 4);
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = __ldg(g4 + u);
      } else {
        const uint32_t sa = smem_u32(PRE ? static_cast<const void*>(sent + it * kIt * 4)
                                         : static_cast<const void*>(list + it * kIt));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(cur[u].x), "=r"(cur[u].y), "=r"(cur[u].z), "=r"(cur[u].w)
                       : "r"(sa + 16 * u));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!done) {
          // group-uniform: bucket ends inside this block (pair m ends bucket t_m)
          unsigned endm = 0;
          uint32_t tpk = 0;
          i += kBlk;
          while (bend <= i) {
            const int m = ((bend - (i - kBlk)) >> 1) - 1;
            endm |= 1u << m;
            tpk |= uint32_t(t) << (8 * m);
            ++t;
            while (t < T && int(start[t + 1]) == bend) ++t;  // empty buckets add nothing
            bend = t < T ? int(start[t + 1]) : 0x7FFFFFFF;
          }
          walk_block<FPL>(wl, cur[2 * h], cur[2 * h + 1], endm, tpk, thr, acc, fired, lo, vo);
        }
        const unsigned nf = __ballot_sync(0xffffffffu, !done && fired != kAll);
        if (!done && ((nf & gmask) == 0 || i >= total)) done = true;
      }
      ++it;
      if (!done && --guard < 0) {
        flag_error(a.err, kErrInternal);
        done = true;
      }
    }
    if (pv) {
#pragma unroll
      for (int j = 0; j < FPL; ++j) {
        if (valid >> j & 1) {
          const int64_t o = (int64_t(b) * a.F + fbase + j) * HoWo + rem;
          a.lat_out[o] = uint8_t(lo >> (8 * j));
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
  int64_t chunk;                                   // positions per list chunk
  WalkArgs a;                                      // walk kernel arguments / smem layout
  WalkArgs sa;                                     // sort kernel arguments / smem layout
};

static int pos_scratch_bytes(int T, int R, WalkArgs* a) {
  int o = 0, c0, c1, c3;
  c0 = o; o += al16(T * 4);                // bucket counters (u32, shared-memory atomics)
  c1 = o; o += al16((T + 1) * 2);          // bucket starts
  c3 = o; o += al16((R + T + kIt) * 4);    // entries + one pad per bucket + tail
  if (a) { a->cnt_off = c0; a->start_off = c1; a->list_off = c3; a->pos_bytes = o; }
  return o;
}

static bool walk_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, WalkPlan* pl) {
  WalkArgs& a = pl->a;
  a = WalkArgs{};
  if (int64_t(B) * (H + 2 * pad - KH + 1) * (W + 2 * pad - KW + 1) >= (int64_t(1) << 31)) return false;
  a.B = B; a.C = C; a.H = H; a.W = W; a.pad = pad; a.F = F; a.KH = KH; a.KW = KW; a.T = T;
  a.Ho = H + 2 * pad - KH + 1; a.Wo = W + 2 * pad - KW + 1; a.R = C * KH * KW;
  const int R = a.R;
  if (R + T + kIt >= 65536) return false;  // u16 bucket starts
  const long tables = al16(R * 4) + al16(R * 2);
  struct Cand { int ppw, fpl; };
  const Cand cands[] = {{4, 4}, {2, 4}, {1, 4}, {4, 2}, {2, 2}, {1, 2}, {1, 1}};
  // 1) fused: all features in one group with >= 8 warps of sort scratch
  int best = -1, best_warps = 0;
  for (const Cand& c : cands) {
    const int lpp = 32 / c.ppw, fgs = lpp * c.fpl;
    if (fgs < F) continue;
    if (fgs > 32 && F <= fgs / 2) continue;
    const int wb = c.ppw * pos_scratch_bytes(T, R, nullptr);
    const long fixed = al16(int(long(R + 1) * fgs * 4)) + tables;
    if (fixed + 8L * wb > kWalkSmemLimit) continue;
    long warps = (kWalkSmemLimit - fixed) / wb;
    const int wcap = c.fpl == 4 ? 24 : 32;
    if (warps > wcap) warps = wcap;
    if (best < 0) { best = int(&c - cands); best_warps = int(warps); }  // the first (widest FPL) that fits
  }
  if (const char* e = getenv("SNN_WALK_FUSED")) {  // tuning experiments: force "ppw,fpl"
    int ppw = 0, fpl = 0;
    if (sscanf(e, "%d,%d", &ppw, &fpl) == 2)
      for (const Cand& c : cands)
        if (c.ppw == ppw && c.fpl == fpl && (32 / ppw) * fpl >= F) {
          best = int(&c - cands);
          const int wb = c.ppw * pos_scratch_bytes(T, R, nullptr);
          const long fixed = al16(int(long(R + 1) * (32 / ppw) * fpl * 4)) + tables;
          long warps = (kWalkSmemLimit - fixed) / wb;
          const int wcap = c.fpl == 4 ? 24 : 32;
          best_warps = int(warps > wcap ? wcap : warps);
        }
  }
  if (best >= 0) {
    pl->pre = false;
    pl->ppw = cands[best].ppw; pl->fpl = cands[best].fpl;
    const int lpp = 32 / pl->ppw;
    pl->FGS = lpp * pl->fpl; pl->n_groups = 1; pl->nwarps = best_warps;
    a.row_bytes = pl->FGS * 4;
    pos_scratch_bytes(T, R, &a);
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
  const char* fe = getenv("SNN_WALK_PRE_FPL");  // tuning experiments: force the presorted FPL
  const int force_fpl = fe ? atoi(fe) : 0;
  for (int k = 0; k < 3; ++k) {
    const int fpl = fpls[k], fgs = 32 * fpl;
    if (force_fpl && fpl != force_fpl) continue;
    if (!force_fpl && fgs > 32 && F <= fgs / 2) continue;
    const long wsb = long(R + 1) * fgs * 4;
    const int hdr_bytes = al16((T + 1) * 2);
    if (al16(int(wsb)) + 20L * (16 + 2 * (hdr_bytes + kIt * 4)) > kWalkSmemLimit) continue;
    pl->sort_ppw = R <= 256 ? 4 : 1;  // 4 positions per warp for small receptive fields
    pl->pre = true;
    pl->ppw = 1; pl->fpl = fpl; pl->FGS = fgs;
    pl->n_groups = int(ceil_div(F, fgs));
    pl->nwarps = fpl == 4 ? 20 : 32;
    a.row_bytes = fgs * 4;
    // per warp: 2 mbarriers, then two position buffers [header | npre entries]
    const long left = (kWalkSmemLimit - al16(int(wsb))) / pl->nwarps - 16;
    int npre = int(((left / 2 - hdr_bytes) / 4) / kIt) * kIt;
    if (npre > 256) npre = 256;
    if (npre < kIt) continue;
    a.npre = npre;
    a.buf_bytes = hdr_bytes + npre * 4;
    a.cnt_off = 0; a.start_off = 0; a.list_off = 0;
    a.pos_bytes = 16 + 2 * a.buf_bytes; a.warp_bytes = a.pos_bytes;
    a.off_eoff = al16(int(wsb)); a.off_ekk = a.off_eoff; a.off_warps = a.off_eoff;
    pl->smem = a.off_warps + pl->nwarps * a.warp_bytes;
    a.hdr = hdr_bytes;
    a.rec = hdr_bytes + int(ceil_div(R + T, kIt)) * kIt * 4;
    pl->sort_nwarps = 16;
    WalkArgs& sa = pl->sa;
    sa = a;
    pos_scratch_bytes(T, R, &sa);
    sa.warp_bytes = pl->sort_ppw * sa.pos_bytes;
    sa.off_eoff = 0;
    sa.off_ekk = al16(R * 4);
    sa.off_warps = sa.off_ekk + al16(R * 2);
    pl->sort_smem = sa.off_warps + pl->sort_nwarps * sa.warp_bytes;
    const int64_t npos = int64_t(B) * a.Ho * a.Wo;
    size_t chunk_bytes = kListChunkBytes;
    if (const char* e = getenv("SNN_LIST_CHUNK_MB")) chunk_bytes = size_t(atoi(e)) << 20;  // tuning experiments
    int64_t ch = int64_t(chunk_bytes / size_t(a.rec));
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
  if (pl.pre) n += size_t(pl.chunk) * pl.a.rec + kListSlack;
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

// Plan description for snn_conv_fire_plan: 0 if the walk does not apply, else 1 (+ *pre, *chunks).
int conv_walk_describe(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, int* pre, int* chunks) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 0;
  *pre = pl.pre ? 1 : 0;
  *chunks = int(ceil_div(int64_t(B) * pl.a.Ho * pl.a.Wo, pl.chunk));
  return 1;
}

// Returns 1 if this path does not apply (caller falls back), else an SNN code.
int conv_walk_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                     cudaStream_t s) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 1;
  WalkArgs a = pl.a;
  size_t wq_bytes = (size_t(pl.n_groups) * (a.R + 1) * pl.FGS * 4 + 255) & ~size_t(255);
  const size_t need = wq_bytes + (pl.pre ? size_t(pl.chunk) * a.rec + kListSlack : 0);
  if (ws_bytes < need) return set_error(SNN_EWORKSPACE, "snn_conv_fire: workspace %zu < %zu", ws_bytes, need);
  a.lat_in = lat_in; a.lat_out = lat_out; a.v_out = v_out;
  a.err = error_word_ptr();
  a.wq = reinterpret_cast<const uint32_t*>(ws);
  a.lists = reinterpret_cast<unsigned char*>(ws) + wq_bytes;
  const double tt = floor(double(theta) * 2147483648.0);
  a.thr = tt >= 9.0e18 ? INT64_MAX : (tt < -1.0 ? -1 : int64_t(tt));
  const int64_t npos = int64_t(B) * a.Ho * a.Wo;
  if (getenv("SNN_DEBUG_PLAN"))
    fprintf(stderr, "walk plan: pre %d fpl %d ppw %d FGS %d groups %d warps %d smem %d | sort ppw %d "
            "warps %d smem %d | rec %d hdr %d chunk %lld npos %lld\n", int(pl.pre), pl.fpl, pl.ppw, pl.FGS,
            pl.n_groups, pl.nwarps, pl.smem, pl.sort_ppw, pl.sort_nwarps, pl.sort_smem, a.rec,
            a.hdr, (long long)pl.chunk, (long long)npos);
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
