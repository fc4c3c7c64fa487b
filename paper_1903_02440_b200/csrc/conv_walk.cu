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
#include "walk_dev.cuh"

namespace snn {

int weight_prep_launch(const float* w, int F, int R, int FGS, int n_groups, uint32_t* wq, cudaStream_t s,
                       int nhwc_C = 0, int KK = 1);

// ------------------------------------------------------------------------------------- K* bound (K2b)
// K* = max over features f of the smallest k such that the sum of f's k smallest weights exceeds the
// threshold: any k spiking inputs of a receptive field sum to at least that, so once a sorted list
// has passed K* entries at a bucket end every feature has fired (weights are >= 0) and the rest of the
// list can never matter.  One CTA per feature: its R fixed-point weights bitonic-sorted ascending in
// shared memory, then the first prefix above the threshold; atomicMax into *out (zeroed before).  A
// feature whose weights never exceed the threshold gives INT_MAX (no truncation).  R <= 4096.
__global__ void __launch_bounds__(256) kstar_kernel(const float* __restrict__ w, int R, int64_t thr,
                                                    int in_nhwc_C, int KK, int* out) {
  pdl_begin();
  __shared__ uint32_t v[4096];
  __shared__ int s_k;
  const int f = blockIdx.x;
  int n = 1;
  while (n < R) n <<= 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t u = 0xFFFFFFFFu;
    if (i < R) {
      const float x = __ldg(w + int64_t(f) * R + i);
      const float sx = x * 2147483648.0f;
      u = (x >= 0.0f && x <= 1.0f) ? uint32_t(sx) : 0u;  // outside the exact domain: flagged elsewhere
    }
    v[i] = u;
  }
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const uint32_t a = v[i], b = v[p];
          if (((i & k) == 0) == (a > b)) { v[i] = b; v[p] = a; }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    int k = 0x7FFFFFFF;
    if (thr < 0) k = 0;
    else
      for (int i = 0; i < R; ++i) {
        acc += v[i];
        if (acc > thr) { k = i + 1; break; }
      }
    s_k = k;
  }
  // kmin (K2e) = min over features of the smallest k such that the sum of f's k LARGEST weights exceeds
  // the threshold: fewer than kmin spiking inputs cannot fire any feature, so the buckets of a sorted
  // list that end below kmin entries need no threshold test.  out[1] = max over f of INT_MAX - k_f
  // (zeroed before; a feature that can never fire contributes 0).
  if (threadIdx.x == 32) {
    int64_t acc = 0;
    int k = 0x7FFFFFFF;
    if (thr < 0) k = 0;
    else
      for (int i = R - 1; i >= 0; --i) {
        acc += v[i];
        if (acc > thr) { k = R - i; break; }
      }
    atomicMax(out + 1, 0x7FFFFFFF - k);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(out, s_k);
  (void)in_nhwc_C; (void)KK;
}

int kstar_launch(const float* w, int F, int R, int64_t thr, int* out, cudaStream_t s) {
  if (cudaMemsetAsync(out, 0, 2 * sizeof(int), s) != cudaSuccess) return check_launch("snn_conv_fire(K* memset)");
  launch_k(kstar_kernel, dim3(F), dim3(256), 0, s, w, R, thr, 0, 1, out);
  note_launch();
  return check_launch("snn_conv_fire(K*)");
}

// ------------------------------------------------------------------------------------- sort only
template <int PPW>
__global__ void __launch_bounds__(512) rf_sort_kernel(const WalkArgs a) {
  pdl_wait();
  constexpr int LPP = 32 / PPW;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / LPP, gl = lane - grp * LPP;
  unsigned char* wbase = smem + a.off_warps + warp * a.warp_bytes;
  unsigned char* pb = wbase + grp * a.pos_bytes;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(pb + a.cnt_off);
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);
  uint32_t* list = reinterpret_cast<uint32_t*>(pb + a.list_off);
  rf_tables(a, smem);
  __syncthreads();
  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < a.np; wi += int64_t(gridDim.x) * nwarps) {
    const int64_t q = wi * PPW + grp;  // chunk-relative position
    const bool pv = q < a.np;
    rf_sort_warp<PPW, true>(a, smem, wbase, wi * PPW, lane, grp, gl, pv, cnt, start, list);
    if (pv) {  // record = [header: T+1 u16 starts, 16-aligned][entries: u32, whole blocks]
      unsigned char* rec = a.lists + q * a.rec;
      uint16_t* hdr = reinterpret_cast<uint16_t*>(rec);
      for (int t = gl; t <= a.T; t += LPP) hdr[t] = start[t];
      const int n4 = (((int(start[a.T]) & -a.pad_unit) + kIt - 1) / kIt) * (kIt / 4);  // uint4 per walk iteration
      SNN_DCHECK(a.hdr + n4 * 16 <= a.rec && q < a.np);
      const uint4* src = reinterpret_cast<const uint4*>(list);
      uint4* dst = reinterpret_cast<uint4*>(rec + a.hdr);
      for (int k = gl; k < n4; k += LPP) dst[k] = src[k];
    }
    __syncwarp();
  }
}

// The per-position loop of conv_walk_kernel once the CTA's weight slice is staged (S28: the slice is
// in units of 2^-28, see walk_block).
template <int FPL, int PPW, bool PRE, bool S28, bool BW, bool GW = false, bool LS = false>
__device__ __forceinline__ void walk_positions(const WalkArgs& a, unsigned char* smem) {
  constexpr int LPP = 32 / PPW;
  constexpr int FGS = LPP * FPL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / LPP, gl = lane - grp * LPP;
  unsigned char* wbase = smem + a.off_warps + warp * a.warp_bytes;
  unsigned char* pb = wbase + grp * a.pos_bytes;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(pb + a.cnt_off);
  uint16_t* start = reinterpret_cast<uint16_t*>(pb + a.start_off);
  uint32_t* list = reinterpret_cast<uint32_t*>(pb + a.list_off);  // fused: the sorted list; PRE: the ring
  const int g = blockIdx.y;
  const int HoWo = a.Ho * a.Wo;
  const int fbase = g * FGS + gl * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < a.F) ? (1u << j) : 0u;
  const unsigned gmask = (LPP == 32) ? 0xffffffffu : (((1u << LPP) - 1u) << (grp * LPP));
  const int64_t stride_w = int64_t(gridDim.x) * nwarps;
  // this lane's features in weight row 0: the shared-memory slice, or (GW) the group's prepared slice
  const unsigned char* wl = GW ? reinterpret_cast<const unsigned char*>(a.wq + int64_t(g) * (a.R + 1) * FGS) + gl * FPL * 4
                               : smem + gl * FPL * 4;

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
  // channels-last outputs with F % FPL == 0 and aligned pointers: a lane's FPL outputs are contiguous
  const bool vec_out = a.nhwc && (a.F % FPL) == 0 && (reinterpret_cast<uintptr_t>(a.lat_out) % FPL) == 0 &&
                       (reinterpret_cast<uintptr_t>(a.v_out) % (4 * FPL)) == 0;
  int need = 1;  // K2e (presorted lists): max(kmin, 1), the entries a list needs before any feature can fire
  if constexpr (PRE) {
    if (a.kmin) { const int km = 0x7FFFFFFF - __ldg(a.kmin); need = km > 1 ? km : 1; }
  }
  int npos_done = 0;
  for (int64_t wi = int64_t(blockIdx.x) * nwarps + warp; wi * PPW < a.np; wi += stride_w, ++npos_done) {
    const int64_t q = wi * PPW + grp;
    const bool pv = q < a.np;
    const int p = int(a.p0 + q);  // npos < 2^31 (checked by the planner)
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
      rf_sort_warp<PPW>(a, smem, wbase, wi * PPW, lane, grp, gl, pv, cnt, start, list);
    }

    uint32_t lo;
    float vo[FPL];
    if constexpr (LS) walk_list_lockstep<FPL, PPW, S28>(a, wl, start, list, pv, valid, lo, vo);
    else walk_list<FPL, PPW, PRE, S28, BW, GW>(a, wl, start, sent, ent, list, pv, valid, gmask, lo, vo, need);
    if (pv) {
      // NHWC: the warp's features of one position are contiguous (one or two lines per store);
      // NCHW: every feature is a separate plane (a line per lane per store)
      int64_t o0 = int64_t(p) * a.F + fbase;
      if (!a.nhwc) {  // planar: (image, position in the image) -- a division only for this layout
        const int b = p / HoWo, rem = p - b * HoWo;
        o0 = (int64_t(b) * a.F + fbase) * HoWo + rem;
      }
      if (FPL > 1 && vec_out) {  // the lane's FPL outputs as one vector store each (a lane past F: none)
        if (valid == 0) {
        } else if constexpr (FPL == 2) {
          *reinterpret_cast<uint16_t*>(a.lat_out + o0) = uint16_t(lo);
          if (a.v_out) __stcs(reinterpret_cast<float2*>(a.v_out + o0), make_float2(vo[0], vo[1]));
        } else if constexpr (FPL == 4) {
          *reinterpret_cast<uint32_t*>(a.lat_out + o0) = lo;
          if (a.v_out) __stcs(reinterpret_cast<float4*>(a.v_out + o0), make_float4(vo[0], vo[1], vo[2], vo[3]));
        }
      } else {
        const int64_t fs = a.nhwc ? 1 : HoWo;
#pragma unroll
        for (int j = 0; j < FPL; ++j) {
          if (valid >> j & 1) {
            a.lat_out[o0 + j * fs] = uint8_t(lo >> (8 * j));
            if (a.v_out) a.v_out[o0 + j * fs] = vo[j];
          }
        }
      }
    }
    __syncwarp();
  }
}

// K7: the fused schedule by row tiles (channels-last input).  A warp takes one tile -- output row y of
// image b, output columns [x0, x0 + nxs) -- sorts its input halo once (rows_sort), then walks the tile's
// positions PPW at a time in lockstep (walk_rows_lockstep) and stores their outputs as walk_positions
// does.
template <int FPL, int PPW, bool S28>
__device__ __forceinline__ void walk_rows(const WalkArgs& a, unsigned char* smem) {
  constexpr int LPP = 32 / PPW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int grp = lane / LPP, gl = lane - grp * LPP;
  unsigned char* wbase = smem + a.off_warps + warp * a.warp_bytes;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(wbase + a.cnt_off);
  uint16_t* base = reinterpret_cast<uint16_t*>(wbase + a.start_off);
  uint16_t* list = reinterpret_cast<uint16_t*>(wbase + a.list_off);
  const uint8_t* colof = smem + a.off_eoff;
  const int fbase = gl * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < a.F) ? (1u << j) : 0u;
  const bool vec_out = a.nhwc && (a.F % FPL) == 0 && (reinterpret_cast<uintptr_t>(a.lat_out) % FPL) == 0 &&
                       (reinterpret_cast<uintptr_t>(a.v_out) % (4 * FPL)) == 0;
  const uint32_t wl = smem_u32(smem + gl * FPL * 4), lb = smem_u32(list);
  const uint32_t rb = uint32_t(a.row_bytes), cstep = uint32_t(a.C) * rb;
  // pool2 (SNN_CONV_POOL2): a unit is the output row PAIR (2 py, 2 py + 1) of one tile; the pair's
  // latencies stay in the warp's shared-memory row buffer and only the 2 x 2 / stride 2 minimum is stored
  const int rpu = a.pool2 ? 2 : 1, ny = a.Ho / rpu;
  uint32_t* rowbuf = reinterpret_cast<uint32_t*>(wbase + a.pool_off);  // [2][nx][LPP] latency words
  const int HoWo = a.Ho * a.Wo, per_img = ny * a.nseg;
  const int64_t units = int64_t(a.B) * per_img;
  for (int64_t u = int64_t(blockIdx.x) * nwarps + warp; u < units; u += int64_t(gridDim.x) * nwarps) {
    const int b = int(u / per_img), rem = int(u - int64_t(b) * per_img);
    const int yu = rem / a.nseg, x0 = (rem - yu * a.nseg) * a.nx;
    const int nxs = min(a.nx, a.Wo - x0), ncol = nxs + a.KW - 1;
    for (int h = 0; h < rpu; ++h) {
    const int y = yu * rpu + h;
    rows_sort(a, b, y, x0, ncol, colof, cnt, base, list, lane);
    for (int q0 = 0; q0 < nxs; q0 += PPW) {
      const int xr = q0 + grp;
      const bool pv = xr < nxs;
      uint32_t lo;
      float vo[FPL];
      if (a.rows_g == 2)
        walk_rows_lockstep<FPL, PPW, S28, 2>(a, wl - uint32_t(xr) * cstep, uint32_t(a.R) * rb + uint32_t(xr) * cstep,
                                             base + xr, ncol, lb, pv, valid, lo, vo);
      else
        walk_rows_lockstep<FPL, PPW, S28, 1>(a, wl - uint32_t(xr) * cstep, uint32_t(a.R) * rb + uint32_t(xr) * cstep,
                                             base + xr, ncol, lb, pv, valid, lo, vo);
      if (a.pool2) {
        if (pv) rowbuf[(h * a.nx + xr) * LPP + gl] = lo;
      } else if (pv) {
        const int p = b * HoWo + y * a.Wo + x0 + xr;
        int64_t o0 = int64_t(p) * a.F + fbase;
        if (!a.nhwc) o0 = (int64_t(b) * a.F + fbase) * HoWo + (p - b * HoWo);
        if (FPL > 1 && vec_out) {
          if (valid == 0) {
          } else if constexpr (FPL == 2) {
            *reinterpret_cast<uint16_t*>(a.lat_out + o0) = uint16_t(lo);
            if (a.v_out) __stcs(reinterpret_cast<float2*>(a.v_out + o0), make_float2(vo[0], vo[1]));
          } else if constexpr (FPL == 4) {
            *reinterpret_cast<uint32_t*>(a.lat_out + o0) = lo;
            if (a.v_out) __stcs(reinterpret_cast<float4*>(a.v_out + o0), make_float4(vo[0], vo[1], vo[2], vo[3]));
          }
        } else {
          const int64_t fs = a.nhwc ? 1 : HoWo;
#pragma unroll
          for (int j = 0; j < FPL; ++j) {
            if (valid >> j & 1) {
              a.lat_out[o0 + j * fs] = uint8_t(lo >> (8 * j));
              if (a.v_out) a.v_out[o0 + j * fs] = vo[j];
            }
          }
        }
      }
    }
    __syncwarp();
    }
    if (a.pool2) {  // lat_o = min over the 2 x 2 window (R: pool, latency-only), channels-last [B, Ho/2, Wo/2, F]
      const int nx2 = nxs >> 1, PWo = a.Wo >> 1;
      for (int i = lane; i < nx2 * LPP; i += 32) {
        const int px = i / LPP, qd = i - px * LPP, f0 = qd * FPL;
        if (f0 >= a.F) continue;
        const uint32_t* r0 = rowbuf + (2 * px) * LPP + qd;
        const uint32_t* r1 = r0 + a.nx * LPP;
        const uint32_t m = __vminu4(__vminu4(r0[0], r0[LPP]), __vminu4(r1[0], r1[LPP]));
        uint8_t* o = a.lat_out + ((int64_t(b) * ny + yu) * PWo + (x0 >> 1) + px) * a.F + f0;
        const int nf = min(FPL, a.F - f0);
        if (nf == 4 && (reinterpret_cast<uintptr_t>(o) & 3) == 0) {
          *reinterpret_cast<uint32_t*>(o) = m;
        } else if ((reinterpret_cast<uintptr_t>(o) & 1) == 0) {
          if (nf >= 2) *reinterpret_cast<uint16_t*>(o) = uint16_t(m);
          if (nf == 4) *reinterpret_cast<uint16_t*>(o + 2) = uint16_t(m >> 16);
          else if (nf == 3) o[2] = uint8_t(m >> 16);
          else if (nf == 1) o[0] = uint8_t(m);
        } else {
          for (int j = 0; j < nf; ++j) o[j] = uint8_t(m >> (8 * j));
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void rows_tables(const WalkArgs& a, unsigned char* tabs) {
  uint8_t* colof = tabs + a.off_eoff;
  for (int j = threadIdx.x; j < (a.nx + a.KW - 1) * a.C; j += blockDim.x) colof[j] = uint8_t(j / a.C);
}

template <int FPL, int PPW, bool PRE, bool WCONV = false, bool BW = true, bool GW = false, bool LS = false,
          bool RW = false>
__global__ void __launch_bounds__(WalkThreads<FPL, PRE>::v, 1) conv_walk_kernel(const WalkArgs a) {
  pdl_wait();
  constexpr int LPP = 32 / PPW;
  constexpr int FGS = LPP * FPL;
  static_assert(!PRE || PPW == 1, "presorted walk: one position per warp");
  static_assert(!GW || PRE, "global-weight walk: presorted lists");
  extern __shared__ __align__(16) unsigned char smem[];
  if constexpr (GW) {  // the slice stays in global memory (units of 2^-31, from weight_prep)
    walk_positions<FPL, PPW, PRE, false, BW, true>(a, smem);
    return;
  }
  const int R = a.R;
  const int tid = threadIdx.x;
  const int g = blockIdx.y;
  // Stage the group's weight slice as fixed point (units of 2^-31) and test whether every weight is
  // also a multiple of 2^-28 (bits 0-2 clear): then the whole slice is rescaled to 2^-28 and the
  // walk sums blocks in 32 bits (S28).  Each CTA decides for its own slice (its features only).
  bool ok28 = true;
  if constexpr (WCONV) {  // fixed point straight from the fp32 weights (exact domain checked, N1)
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
    for (int i = tid; i < (R + 1) * FGS; i += blockDim.x) {
      const int e = i / FGS, f = g * FGS + (i - (i / FGS) * FGS);
      uint32_t u = 0;
      if (f < a.F && e < R) {
        int se = e;  // the row's source element in w[f] = [C][KH][KW]
        if (a.in_nhwc) { const int kk = e / a.C; se = (e - kk * a.C) * (a.KH * a.KW) + kk; }
        const float x = __ldg(a.wf32 + int64_t(f) * R + se);
        const float sx = x * 2147483648.0f;  // exact power-of-two scaling
        if (!(x >= 0.0f && x <= 1.0f) || sx != truncf(sx)) flag_error(a.err, kErrInexact);
        else u = uint32_t(sx);
      }
      ok28 &= (u & 7u) == 0;
      dst[i] = u;
    }
    rf_tables(a, smem);
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(a.wq + int64_t(g) * (R + 1) * FGS);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const int n4 = (R + 1) * FGS / 4;
    for (int i = tid; i < n4; i += blockDim.x) {
      const uint4 v = src[i];
      ok28 &= ((v.x | v.y | v.z | v.w) & 7u) == 0;
      dst[i] = v;
    }
    if (RW) rows_tables(a, smem);
    else if (!PRE) rf_tables(a, smem);
  }
  const bool s28 = __syncthreads_and(ok28) != 0;
  if (s28) {
    uint4* w4 = reinterpret_cast<uint4*>(smem);
    for (int i = tid; i < (R + 1) * FGS / 4; i += blockDim.x) {
      uint4 v = w4[i];
      v.x >>= 3; v.y >>= 3; v.z >>= 3; v.w >>= 3;
      w4[i] = v;
    }
    __syncthreads();
    if constexpr (RW) walk_rows<FPL, PPW, true>(a, smem);
    else walk_positions<FPL, PPW, PRE, true, BW, false, LS>(a, smem);
  } else {
    if constexpr (RW) walk_rows<FPL, PPW, false>(a, smem);
    else walk_positions<FPL, PPW, PRE, false, BW, false, LS>(a, smem);
  }
}

// ------------------------------------------------------------------------------------- host
struct WalkPlan {
  int fpl, ppw, FGS, n_groups, nwarps, smem;  // walk kernel
  bool gw;                                     // presorted walk gathering from global memory (large R)
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
  c3 = o; o += al16(list_cap(R, T) * 4);  // entries + up to 3 pads per bucket + tail + over-read
  if (a) { a->cnt_off = c0; a->start_off = c1; a->list_off = c3; a->pos_bytes = o; }
  return o;
}

// Layout of the sort's tables (from byte `base`) and per-warp scratch (PPW position scratches + the
// input patch, rf_sort_warp); a.pos_bytes must be set.  Returns the offset of the warps' regions.
static int sort_layout(WalkArgs& a, int ppw, int base) {
  a.patch_w = a.KW + ppw - 1;
  const long pn = long(a.C) * a.KH * a.patch_w;
  // the patch pays when several positions share it; one position per warp (or a large receptive
  // field) reads its latencies from global memory (measured C5: 47.6 ms without, 50.4 ms with)
  a.patch_n = (ppw > 1 && pn <= 4096) ? int(pn) : 0;
  a.off_eoff = base;
  a.off_ekk = a.off_eoff + al16(a.R * 4);
  a.off_eoffp = a.off_ekk + al16(a.R * 2);
  a.off_ptab = a.off_eoffp + al16(a.R * 2);
  a.off_pkk = a.off_ptab + al16(a.patch_n * 4);
  a.off_warps = a.off_pkk + al16(a.patch_n * 2);
  a.patch_off = ppw * a.pos_bytes;
  a.warp_bytes = a.patch_off + al16(a.patch_n);
  return a.off_warps;
}

// positions per warp of the sort kernel (more independent positions per warp hide the gather latency;
// measured C2 conv2 (R 270): 1.20 ms at 1, 1.14 ms at 4; C5 (R 800): 50 ms at 1, 64 ms at 4);
// SNN_SORT_PPW overrides: 1, 2, 4
static int sort_ppw_for(int R) {
  if (const char* e = getenv("SNN_SORT_PPW")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4) return v;
  }
  return R <= 512 ? 4 : 1;
}

// Bucket-by-bucket walk (pad unit 4) when the buckets hold enough entries to amortise a test and a
// vote per bucket (R >= 8 T: C2's second layer, C3, C5), else K3 blocks across buckets (pad unit 2:
// C1, C2's first layer, C4's first layer).  SNN_WALK_BW=0/1 forces one (experiments).
static bool walk_bucketwise(int R, int T) {
  if (const char* e = getenv("SNN_WALK_BW")) return e[0] == '1';
  return R >= 8 * T;
}

static bool walk_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, WalkPlan* pl) {
  WalkArgs& a = pl->a;
  a = WalkArgs{};
  pl->gw = false;
  if (int64_t(B) * (H + 2 * pad - KH + 1) * (W + 2 * pad - KW + 1) >= (int64_t(1) << 31)) return false;
  a.B = B; a.C = C; a.H = H; a.W = W; a.pad = pad; a.F = F; a.KH = KH; a.KW = KW; a.T = T;
  a.Ho = H + 2 * pad - KH + 1; a.Wo = W + 2 * pad - KW + 1; a.R = C * KH * KW;
  const int R = a.R;
  if (list_cap(R, T) >= 65536) return false;  // u16 bucket starts
  a.pad_unit = walk_bucketwise(R, T) ? 4 : 2;
  struct Cand { int ppw, fpl; };
  auto sort_cost = [&](int ppw, long* tables) {  // (tables bytes, per-warp bytes) of a fused candidate
    WalkArgs t = a;
    pos_scratch_bytes(T, R, &t);
    *tables = sort_layout(t, ppw, 0);
    return long(t.warp_bytes);
  };
  const Cand cands[] = {{4, 4}, {2, 4}, {1, 4}, {4, 2}, {2, 2}, {1, 2}, {1, 1}};
  // 1) fused: all features in one group with >= 8 warps of sort scratch
  int best = -1, best_warps = 0;
  for (const Cand& c : cands) {
    const int lpp = 32 / c.ppw, fgs = lpp * c.fpl;
    if (fgs < F) continue;
    if (fgs > 32 && F <= fgs / 2) continue;
    long tables;
    const long wb = sort_cost(c.ppw, &tables);
    const long fixed = al16(int(long(R + 1) * fgs * 4)) + tables;
    if (fixed + 8L * wb > kWalkSmemLimit) continue;
    long warps = (kWalkSmemLimit - fixed) / wb;
    const int wcap = c.fpl == 4 ? 24 : 32;
    if (warps > wcap) warps = wcap;
    // the first (widest FPL) that fits; a map of few positions (one image: latency, not throughput)
    // takes the first one-position-per-warp candidate instead -- all lanes sort its receptive field
    // (measured C1: PPW 4 / FPL 4 53.1 us per step, PPW 1 / FPL 1 50.9 us)
    const bool latency = int64_t(B) * a.Ho * a.Wo <= int64_t(num_sms()) * 16;
    if (best < 0 || (latency && c.ppw == 1 && cands[best].ppw != 1)) { best = int(&c - cands); best_warps = int(warps); }
  }
  if (const char* e = getenv("SNN_WALK_FUSED")) {  // tuning experiments: force "ppw,fpl"
    int ppw = 0, fpl = 0;
    if (sscanf(e, "%d,%d", &ppw, &fpl) == 2)
      for (const Cand& c : cands)
        if (c.ppw == ppw && c.fpl == fpl && (32 / ppw) * fpl >= F) {
          best = int(&c - cands);
          long tables;
          const long wb = sort_cost(c.ppw, &tables);
          const long fixed = al16(int(long(R + 1) * (32 / ppw) * fpl * 4)) + tables;
          long warps = (kWalkSmemLimit - fixed) / wb;
          const int wcap = c.fpl == 4 ? 24 : 32;
          best_warps = int(warps > wcap ? wcap : warps);
        }
  }
  if (getenv("SNN_WALK_NOFUSE")) best = -1;  // tuning experiments: force the presorted schedule
  if (best >= 0) {
    pl->pre = false;
    pl->ppw = cands[best].ppw; pl->fpl = cands[best].fpl;
    // several positions per warp: their lists are walked in lockstep (K3c, no pads); SNN_WALK_LOCKSTEP=0
    // keeps the per-group walks (experiments)
    if (pl->ppw > 1 && !(getenv("SNN_WALK_LOCKSTEP") && getenv("SNN_WALK_LOCKSTEP")[0] == '0')) a.pad_unit = 1;
    const int lpp = 32 / pl->ppw;
    pl->FGS = lpp * pl->fpl; pl->n_groups = 1; pl->nwarps = best_warps;
    a.row_bytes = pl->FGS * 4;
    pos_scratch_bytes(T, R, &a);
    sort_layout(a, pl->ppw, al16(int(long(R + 1) * pl->FGS * 4)));
    pl->smem = a.off_warps + pl->nwarps * a.warp_bytes;
    a.np = int64_t(B) * a.Ho * a.Wo;
    pl->chunk = a.np;
    return true;
  }
  // 2) presorted: sort once per position, walk per feature group (PPW = 1, the largest FPL that fits)
  const int fpls[3] = {4, 2, 1};
  const char* fe = getenv("SNN_WALK_PRE_FPL");  // tuning experiments: force the presorted FPL
  const int force_fpl = fe ? atoi(fe) : 0;
  // 3) receptive fields too large for any shared-memory slice (e.g. C2's layer 3 at a finite
  //    threshold, R = 6,250): the same presorted walk gathering from the prepared slice in global
  //    memory (L2-resident, (R + 1) x FGS x 4 bytes per group) -- Eq. 2 holds for any kernel size
  for (int k = 0; k < 6; ++k) {
    const bool gw = k >= 3;
    const int fpl = fpls[k % 3], fgs = 32 * fpl;
    if (force_fpl && fpl != force_fpl) continue;
    if (!force_fpl && fgs > 32 && F <= fgs / 2) continue;
    if (gw && getenv("SNN_WALK_NOGW")) continue;
    const long wsb = gw ? 0 : long(R + 1) * fgs * 4;
    const int hdr_bytes = al16((T + 1) * 2);
    if (al16(int(wsb)) + 20L * (16 + 2 * (hdr_bytes + kIt * 4)) > kWalkSmemLimit) continue;
    pl->gw = gw;
    pl->sort_ppw = sort_ppw_for(R);
    pl->pre = true;
    pl->ppw = 1; pl->fpl = fpl; pl->FGS = fgs;
    pl->n_groups = int(ceil_div(F, fgs));
    pl->nwarps = fpl == 4 ? 24 : 32;  // measured C2 conv2: 20 warps 1.155 ms, 24 warps 1.121 ms
    if (const char* e = getenv("SNN_WALK_PRE_WARPS")) {  // tuning experiments
      const int v = atoi(e);
      if (v >= 1 && v <= (fpl == 4 ? 24 : 32)) pl->nwarps = v;
    }
    a.row_bytes = fgs * 4;
    // per warp: 2 mbarriers, then two position buffers [header | npre entries]
    const long left = (kWalkSmemLimit - al16(int(wsb))) / pl->nwarps - 16;
    int npre = int(((left / 2 - hdr_bytes) / 4) / kIt) * kIt;
    int npre_cap = 256;
    if (const char* e = getenv("SNN_WALK_NPRE")) npre_cap = atoi(e) / kIt * kIt;  // tuning experiments
    if (npre > npre_cap) npre = npre_cap;
    if (npre < kIt) continue;
    a.npre = npre;
    a.buf_bytes = hdr_bytes + npre * 4;
    a.cnt_off = 0; a.start_off = 0; a.list_off = 0;
    a.pos_bytes = 16 + 2 * a.buf_bytes; a.warp_bytes = a.pos_bytes;
    a.off_eoff = al16(int(wsb)); a.off_ekk = a.off_eoff; a.off_warps = a.off_eoff;
    pl->smem = a.off_warps + pl->nwarps * a.warp_bytes;
    a.hdr = hdr_bytes;
    a.rec = hdr_bytes + int(ceil_div(list_cap(R, T), kIt)) * kIt * 4;
    pl->sort_nwarps = 16;
    WalkArgs& sa = pl->sa;
    sa = a;
    pos_scratch_bytes(T, R, &sa);
    sort_layout(sa, pl->sort_ppw, 0);
    while (pl->sort_nwarps > 1 && sa.off_warps + pl->sort_nwarps * sa.warp_bytes > kWalkSmemLimit) pl->sort_nwarps /= 2;
    pl->sort_smem = sa.off_warps + pl->sort_nwarps * sa.warp_bytes;
    if (pl->sort_smem > kWalkSmemLimit) return false;  // not even one warp's sort scratch fits
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
  n += 256;  // the K* word
  if (pl.pre) n += size_t(pl.chunk) * pl.a.rec + kListSlack;
  return n + 256;
}

template <int FPL, int PPW, bool PRE, bool WCONV = false, bool GW = false>
static int walk_go(const WalkPlan& pl, const WalkArgs& a, cudaStream_t s) {
  auto k = a.pad_unit == 4 ? conv_walk_kernel<FPL, PPW, PRE, WCONV, true, GW>
           : (PPW > 1 && !PRE && a.pad_unit == 1) ? conv_walk_kernel<FPL, PPW, PRE, WCONV, false, GW, PPW != 1>
                                                  : conv_walk_kernel<FPL, PPW, PRE, WCONV, false, GW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(walk): %s", cudaGetErrorString(e));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, pl.nwarps * 32, pl.smem);
  if (occ < 1) occ = 1;
  const int64_t per_group = ceil_div(ceil_div(a.np, PPW), pl.nwarps);
  const int64_t want = ceil_div(int64_t(num_sms()) * occ, pl.n_groups);
  int gx = int(per_group < want ? per_group : want);
  if (gx < 1) gx = 1;
  launch_k(k, dim3(dim3(gx, pl.n_groups)), dim3(pl.nwarps * 32), pl.smem, s, a);
  note_launch();
  return check_launch("snn_conv_fire(walk)");
}

// K7 row-tile layout of a fused PPW = 4 / FPL = 4 plan (channels-last input): tiles of nx positions
// (a multiple of 4, <= 32; nseg tiles per output row), per warp the (t, column) counters, the u16 bucket
// bases and the u16 list; the CTA table colof (halo byte -> column).  False if the u16 weight-row byte
// offsets or shared memory do not fit (the per-position fused walk runs instead).  SNN_WALK_ROWS=0 off.
static bool rows_plan(WalkPlan& pl) {
  if (const char* e = getenv("SNN_WALK_ROWS")) if (e[0] == '0') return false;
  WalkArgs& a = pl.a;
  if (pl.pre || pl.ppw != 4 || pl.fpl != 4 || !a.in_nhwc) return false;
  if (a.pool2 && (a.Ho < 2 || a.Wo < 2 || !a.nhwc || a.v_out)) return false;
  a.nseg = int(ceil_div(a.Wo, 32));
  a.nx = int(ceil_div(ceil_div(a.Wo, a.nseg), 4)) * 4;
  const int ncolmax = a.nx + a.KW - 1;
  if (ncolmax * a.C > 65535 || ncolmax > 255) return false;
  if ((long((a.KH - 1) * a.KW * a.C + ncolmax * a.C) + a.R) * a.row_bytes >= 65536) return false;
  if (long(a.T) * ncolmax >= 65535 || long(a.KH) * ncolmax * a.C >= 65535) return false;
  a.cnt_off = 0;
  a.start_off = al16(a.T * ncolmax * 4);
  a.list_off = a.start_off + al16((a.T * ncolmax + 1) * 2);
  a.pool_off = a.list_off + al16(a.KH * ncolmax * a.C * 2);
  a.warp_bytes = a.pool_off + (a.pool2 ? al16(2 * a.nx * 8 * 4) : 0);
  a.off_eoff = al16(int(long(a.R + 1) * pl.FGS * 4));
  a.off_warps = a.off_eoff + al16(ncolmax * a.C);
  int nw = int((kWalkSmemLimit - a.off_warps) / a.warp_bytes);
  if (nw > 24) nw = 24;
  if (const char* e = getenv("SNN_WALK_ROWS_WARPS")) { const int v = atoi(e); if (v >= 1 && v < nw) nw = v; }
  if (nw < 8) return false;
  // K7c: two buckets per threshold test where buckets are small (R < 6 T, a few spiking inputs each;
  // measured C4 L1 22.2 -> 19.9 ms, C2 L1 unchanged at 1, 4 buckets slower on both: register spills)
  a.rows_g = a.R < 6 * a.T ? 2 : 1;
  if (const char* e = getenv("SNN_WALK_ROWS_G")) { const int v = atoi(e); if (v == 1 || v == 2) a.rows_g = v; }
  pl.nwarps = nw;
  pl.smem = a.off_warps + nw * a.warp_bytes;
  return true;
}

static int rows_go(const WalkPlan& pl, const WalkArgs& a, cudaStream_t s) {
  auto k = conv_walk_kernel<4, 4, false, false, false, false, false, true>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(rows): %s", cudaGetErrorString(e));
  const int64_t units = int64_t(a.B) * (a.pool2 ? a.Ho / 2 : a.Ho) * a.nseg;
  const int64_t per = ceil_div(units, pl.nwarps);
  const int64_t want = num_sms();
  launch_k(k, dim3(int(per < want ? per : want)), dim3(pl.nwarps * 32), pl.smem, s, a);
  note_launch();
  return check_launch("snn_conv_fire(rows)");
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
  launch_k(k, dim3(int(blocks)), dim3(pl.sort_nwarps * 32), pl.sort_smem, s, a);
  note_launch();
  return check_launch("snn_conv_fire(sort)");
}

// Sorted receptive-field lists of every output position of B images, in the presorted record format
// (header + u32 weight-row byte offsets for weight rows of row_bytes), one record of rec bytes per
// position, no chunking: the input of the persistent plasticity chain (seq_train.cu).
int rf_sort_lists_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int KH, int KW, int T,
                         int row_bytes, unsigned char* lists, int rec, int hdr, cudaStream_t s) {
  WalkPlan pl;
  WalkArgs& sa = pl.sa;
  sa = WalkArgs{};
  sa.B = B; sa.C = C; sa.H = H; sa.W = W; sa.pad = pad; sa.KH = KH; sa.KW = KW; sa.T = T;
  sa.Ho = H + 2 * pad - KH + 1; sa.Wo = W + 2 * pad - KW + 1; sa.R = C * KH * KW;
  sa.row_bytes = row_bytes; sa.lists = lists; sa.rec = rec; sa.hdr = hdr;
  sa.pad_unit = 4;  // seq_train walks bucket by bucket
  sa.lat_in = lat_in; sa.p0 = 0; sa.np = int64_t(B) * sa.Ho * sa.Wo;
  const int R = sa.R;
  pl.sort_ppw = sort_ppw_for(R);
  pl.sort_nwarps = 16;
  pos_scratch_bytes(T, R, &sa);
  sort_layout(sa, pl.sort_ppw, 0);
  pl.sort_smem = sa.off_warps + pl.sort_nwarps * sa.warp_bytes;
  if (pl.sort_smem > kWalkSmemLimit) return set_error(SNN_ESHAPE, "rf_sort_lists: receptive field too large");
  return pl.sort_ppw == 4 ? sort_go<4>(pl, sa, s) : pl.sort_ppw == 2 ? sort_go<2>(pl, sa, s) : sort_go<1>(pl, sa, s);
}

// Plan description for snn_conv_fire_plan: 0 if the walk does not apply, else 1 (+ *pre, *chunks).
int conv_walk_describe(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, int* pre, int* chunks,
                       int* launches) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 0;
  *pre = pl.pre ? (pl.gw ? 2 : 1) : 0;
  *launches = pl.pre ? 1 + 2 * int(ceil_div(int64_t(B) * pl.a.Ho * pl.a.Wo, pl.chunk)) : (pl.ppw == 1 ? 1 : 2);
  *chunks = int(ceil_div(int64_t(B) * pl.a.Ho * pl.a.Wo, pl.chunk));
  return 1;
}

// Returns 1 if this path does not apply (caller falls back), else an SNN code.
int conv_walk_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                     cudaStream_t s, int nhwc, int in_nhwc, int pool2) {
  WalkPlan pl;
  if (!walk_plan(B, C, H, W, pad, F, KH, KW, T, &pl)) return 1;
  WalkArgs a = pl.a;
  size_t wq_bytes = (size_t(pl.n_groups) * (a.R + 1) * pl.FGS * 4 + 255) & ~size_t(255);
  const size_t need = wq_bytes + 256 + (pl.pre ? size_t(pl.chunk) * a.rec + kListSlack : 0);
  if (ws_bytes < need) return set_error(SNN_EWORKSPACE, "snn_conv_fire: workspace %zu < %zu", ws_bytes, need);
  a.lat_in = lat_in; a.lat_out = lat_out; a.v_out = v_out; a.nhwc = nhwc; a.in_nhwc = in_nhwc;
  a.err = error_word_ptr(s);
  a.wq = reinterpret_cast<const uint32_t*>(ws);
  int* kstar = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(ws) + wq_bytes);
  a.lists = reinterpret_cast<unsigned char*>(ws) + wq_bytes + 256;
  const double tt = floor(double(theta) * 2147483648.0);
  a.thr = tt >= 9.0e18 ? INT64_MAX : (tt < -1.0 ? -1 : int64_t(tt));
  const double t28 = floor(double(theta) * 268435456.0);
  a.thr28 = t28 >= 9.0e18 ? INT64_MAX : (t28 < -1.0 ? -1 : int64_t(t28));
  const int64_t npos = int64_t(B) * a.Ho * a.Wo;
  if (getenv("SNN_DEBUG_PLAN"))
    fprintf(stderr, "walk plan: pre %d fpl %d ppw %d FGS %d groups %d warps %d smem %d | sort ppw %d "
            "warps %d smem %d | rec %d hdr %d chunk %lld npos %lld gw %d\n", int(pl.pre), pl.fpl, pl.ppw, pl.FGS,
            pl.n_groups, pl.nwarps, pl.smem, pl.sort_ppw, pl.sort_nwarps, pl.sort_smem, a.rec,
            a.hdr, (long long)pl.chunk, (long long)npos, int(pl.gw));
  // K7 row tiles (decided before any launch: SNN_CONV_POOL2 needs them)
  WalkPlan rp = pl;
  rp.a = a;
  rp.a.pool2 = pool2;
  const bool rows = !pl.pre && rows_plan(rp);
  if (pool2 && !rows) return 1;
  if (!pl.pre && pl.ppw == 1) {  // latency mode (few positions): the walk converts the weights itself
    a.wf32 = w;
    a.p0 = 0; a.np = npos;
    switch (pl.fpl) {
      case 4: return walk_go<4, 1, false, true>(pl, a, s);
      case 2: return walk_go<2, 1, false, true>(pl, a, s);
      default: return walk_go<1, 1, false, true>(pl, a, s);
    }
  }
  int rc = weight_prep_launch(w, F, a.R, pl.FGS, pl.n_groups, reinterpret_cast<uint32_t*>(ws), s, in_nhwc ? C : 0,
                              KH * KW);
  if (rc) return rc;
  // K* bound for the list truncation (K2b; on its own measured no faster -- C2 1.06 -> 1.18 ms for conv1 +
  // conv2 -- the sort's first pass, not its placements, sets its time -- so it only rides along with kmin)
  // kmin bound for the test-free list prefix (K2e): on for the bucket walk where the threshold needs several
  // average buckets of inputs (theta >= R / T: C5 conv 27.8 -> 26.1 ms; C2's second layer, whose kmin is about
  // one bucket, measured 0.676 -> 0.691 ms with it); SNN_KMIN=0 / 1 overrides
  {
    const char* ek = getenv("SNN_KMIN");
    const char* es = getenv("SNN_KSTAR");
    bool want_kmin = pl.pre && a.pad_unit == 4 && double(theta) * a.T >= double(a.R);
    // K2b list truncation at K*: free where the bound is computed anyway (presorted lists; C5 conv 24.83 ->
    // 24.68 ms: fewer placements and shorter records to copy); SNN_KSTAR=0 / 1 overrides
    bool want_kstar = want_kmin;
    if (es) want_kstar = atoi(es) != 0;
    if (ek) want_kmin = pl.pre && a.pad_unit == 4 && atoi(ek) != 0;
    if (a.R <= 4096 && a.thr != INT64_MAX && (want_kstar || want_kmin)) {
      rc = kstar_launch(w, F, a.R, a.thr, kstar, s);
      if (want_kstar) a.kstar = kstar;
      if (want_kmin) a.kmin = kstar + 1;
    }
  }
  if (rc) return rc;
  if (!pl.pre) {
    a.p0 = 0; a.np = npos;
    if (rows) {
      rp.a.wq = a.wq; rp.a.kstar = a.kstar;
      if (getenv("SNN_DEBUG_PLAN"))
        fprintf(stderr, "walk rows: nx %d nseg %d warps %d smem %d g %d pool2 %d\n", rp.a.nx, rp.a.nseg, rp.nwarps,
                rp.smem, rp.a.rows_g, rp.a.pool2);
      return rows_go(rp, rp.a, s);
    }
    switch (pl.ppw * 10 + pl.fpl) {
      case 44: return walk_go<4, 4, false>(pl, a, s);
      case 24: return walk_go<4, 2, false>(pl, a, s);
      case 42: return walk_go<2, 4, false>(pl, a, s);
      case 22: return walk_go<2, 2, false>(pl, a, s);
      case 14: return walk_go<4, 1, false>(pl, a, s);
      case 12: return walk_go<2, 1, false>(pl, a, s);
      default: return walk_go<1, 1, false>(pl, a, s);
    }
  }
  WalkArgs sa = pl.sa;
  sa.in_nhwc = in_nhwc;
  sa.kstar = a.kstar;
  sa.kmin = a.kmin;  // K2e: the sort leaves the test-free prefix unpadded for the same bound
  sa.lat_in = lat_in; sa.lists = a.lists; sa.hdr = a.hdr; sa.rec = a.rec;
  for (int64_t p0 = 0; p0 < npos; p0 += pl.chunk) {
    a.p0 = p0;
    a.np = npos - p0 < pl.chunk ? npos - p0 : pl.chunk;
    sa.p0 = a.p0; sa.np = a.np;
    rc = pl.sort_ppw == 4 ? sort_go<4>(pl, sa, s) : pl.sort_ppw == 2 ? sort_go<2>(pl, sa, s) : sort_go<1>(pl, sa, s);
    if (rc) return rc;
    if (pl.gw) {
      switch (pl.fpl) {
        case 4: rc = walk_go<4, 1, true, false, true>(pl, a, s); break;
        case 2: rc = walk_go<2, 1, true, false, true>(pl, a, s); break;
        default: rc = walk_go<1, 1, true, false, true>(pl, a, s); break;
      }
    } else {
      switch (pl.fpl) {
        case 4: rc = walk_go<4, 1, true>(pl, a, s); break;
        case 2: rc = walk_go<2, 1, true>(pl, a, s); break;
        default: rc = walk_go<1, 1, true>(pl, a, s); break;
      }
    }
    if (rc) return rc;
  }
  return SNN_OK;
}

}  // namespace snn
