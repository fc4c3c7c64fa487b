// conv_tct.cu -- a2 + a3 for a finite threshold on the tensor cores, time step by time step
// ("process all of the time-steps simultaneously"; K3).
//
// For every time step t the paper convolves the cumulative spike-wave S[t] (Eq. 1) with the weights,
// P[t] = W (*) S[t].  With the one-spike property S[t] = [lat <= t] is a binary im2col matrix,
// so P[t] is a dense int8 contraction on tcgen05: the 32-bit fixed-point weights (N1) are
// split into four u8 limbs (n = 4 f + limb), accumulated exactly in s32 TMEM columns and recombined in
// int64 by the epilogue, which applies the threshold (spike iff P[t] > theta) and records the first
// crossing (lat = t, v = fp32(P[t])).
//
// One CTA = 128 output positions x one chunk of Fc features (N = 4 Fc <= 256 columns):
//   prologue  : the chunk's weight limbs (N x Kp bytes) arrive by one bulk copy; producer warps gather
//               the tile's receptive-field latencies L[128][Kp] into shared memory (core-matrix layout)
//               and the set of time steps that carry new spikes;
//   per step  : producers turn L into S[t] = [L <= t] bytewise (SIMD byte compares) into one of two
//               A buffers; one thread issues Kp/32 tcgen05.mma (kind::i8) into one of two TMEM
//               accumulators; four epilogue warps read the other accumulator (the previous step)
//               -- so building A, the MMAs and the threshold epilogue of consecutive steps overlap.
//   Steps with no new input spike are skipped: P[t] = P[t-1] there and no neuron can newly cross.
// Shared-memory operands use the canonical K-major no-swizzle layout over the whole K:
//   byte(row, k) = (row/8) * (Kp*8) + (k/16) * 128 + (row%8) * 16 + k%16,  LBO = 128, SBO = Kp*8.
// Warp roles (9 warps): 0-3 producers, 4 TMEM allocator + MMA issuer + weight copy, 5-8 epilogue
// (TMEM lane quadrant = warp % 4).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace snn {

constexpr int kTtM = 128;
constexpr int kTtThreads = 288;
constexpr int kTtSmemLimit = 227 * 1024;

struct TtPlan {
  int M, R, Kp, nch, Fc, N, Ho, Wo;
  int slab, smem, ctas_per_sm;
  size_t b_bytes;  // nch * N * Kp
};

static bool tt_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, TtPlan* p) {
  p->Ho = H + 2 * pad - KH + 1;
  p->Wo = W + 2 * pad - KW + 1;
  p->M = B * p->Ho * p->Wo;
  p->R = C * KH * KW;
  p->Kp = int(ceil_div(p->R, 32)) * 32;
  p->nch = int(ceil_div(F, 64));
  p->Fc = int(ceil_div(ceil_div(F, p->nch), 4)) * 4;
  p->N = 4 * p->Fc;
  const int l_bytes = kTtM * p->Kp;
  // input slab staged per tile: the input rows of every image the tile's 128 positions touch
  const int HoWo = p->Ho * p->Wo;
  long slab;
  if (HoWo >= kTtM) {
    const int orows = int(ceil_div(kTtM, p->Wo)) + 1;
    const int irows = orows + KH - 1 < H ? orows + KH - 1 : H;
    slab = 2L * C * irows * W;
  } else {
    if (ceil_div(kTtM, HoWo) + 1 > 8) return false;  // at most 8 image segments per tile
    slab = long(ceil_div(kTtM, HoWo) + 1) * C * H * W;
  }
  p->slab = int((slab + 15) & ~15L);
  p->smem = p->N * p->Kp + 3 * l_bytes + p->slab + 1024;
  if (p->smem > kTtSmemLimit) return false;
  if (p->Kp * 8 / 16 >= (1 << 14)) return false;  // SBO field
  p->ctas_per_sm = kTtSmemLimit / p->smem;
  p->b_bytes = size_t(p->nch) * p->N * p->Kp;
  return true;
}

size_t conv_tct_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW) {
  TtPlan p;
  if (!tt_plan(B, C, H, W, pad, F, KH, KW, &p)) return 0;
  return p.b_bytes + 256;
}

__device__ __forceinline__ uint32_t tt_off(int row, int k, int Kp) {
  return uint32_t((row >> 3) * (Kp * 8) + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

// B operand: u8 limbs of the fixed-point weights in the full-K core-matrix layout, one block per chunk.
__global__ void tt_prep_b_kernel(const float* __restrict__ w, int F, int R, int Kp, int N, int Fc, int nch,
                                 uint8_t* __restrict__ bq, int* err) {
  const int64_t total = int64_t(nch) * N * Kp;
  int bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int k = int(i % Kp);
    const int64_t rest = i / Kp;
    const int n = int(rest % N), ch = int(rest / N);
    const int f = ch * Fc + (n >> 2), limb = n & 3;
    uint8_t val = 0;
    if (f < F && k < R) {
      const float x = w[int64_t(f) * R + k];
      const float s = x * 2147483648.0f;
      if (!(x >= 0.0f && x <= 1.0f) || s != truncf(s)) bad = 1;
      else val = uint8_t(uint32_t(s) >> (8 * limb));
    }
    bq[size_t(ch) * N * Kp + tt_off(n, k, Kp)] = val;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_error(err, kErrInexact);
}

struct TtArgs {
  const uint8_t* lat_in;
  const uint8_t* bq;
  int C, H, W, pad, KH, KW, T, F;
  int64_t thr;
  uint8_t* lat_out;
  float* v_out;
  TtPlan p;
  uint32_t tmem_cols;
};

__global__ void __launch_bounds__(kTtThreads, 1) conv_tct_kernel(const TtArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TtPlan& p = a.p;
  const int Kp = p.Kp, N = p.N, T = a.T;
  const uint32_t l_bytes = uint32_t(kTtM) * Kp, b_bytes = uint32_t(N) * Kp;
  uint8_t* sB = smem;
  uint8_t* sL = smem + b_bytes;
  uint8_t* sA0 = sL + l_bytes;  // two A buffers follow
  uint8_t* sS = sA0 + 2 * size_t(l_bytes);  // input slab
  __shared__ __align__(8) uint64_t b_full, a_full[2], a_empty[2], d_full[2], d_empty[2], mma_done;
  __shared__ uint32_t tmem_base_sh, present[8];
  __shared__ uint8_t steps[256];
  __shared__ int nsteps;
  __shared__ int seg_b[8], seg_r0[8], seg_nr[8], seg_off[8], nseg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int ch = int(blockIdx.x % unsigned(p.nch)), mt = int(blockIdx.x / unsigned(p.nch));
  const int HoWo = p.Ho * p.Wo;

  if (tid == 0) {
    mbar_init(smem_u32(&b_full), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&a_full[i]), 128);
      mbar_init(smem_u32(&a_empty[i]), 1);
      mbar_init(smem_u32(&d_full[i]), 1);
      mbar_init(smem_u32(&d_empty[i]), 128);
    }
    mbar_init(smem_u32(&mma_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 8) present[tid] = 0;
  if (warp == 4) tmem_alloc(smem_u32(&tmem_base_sh), a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 4 && lane == 0) {  // weight limbs of this chunk: one bulk copy
    mbar_expect_tx(smem_u32(&b_full), b_bytes);
    const uint8_t* src = a.bq + size_t(ch) * b_bytes;
    uint32_t off = 0;
    while (off < b_bytes) {  // bulk copies of <= 64 KB each
      const uint32_t nb = b_bytes - off < 65536u ? b_bytes - off : 65536u;
      bulk_g2s(smem_u32(sB + off), src + off, nb, smem_u32(&b_full));
      off += nb;
    }
  }
  if (warp < 4) {
    // ---- producers: stage the input rows the tile touches (coalesced), then gather the tile's
    //      receptive-field latencies L (255 = no spike / padding) from shared memory ----
    const int m0 = mt * kTtM, m1 = (m0 + kTtM < p.M ? m0 + kTtM : p.M) - 1;
    if (tid == 0) {
      int n = 0, off = 0;
      for (int b = m0 / HoWo; b <= m1 / HoWo; ++b) {
        const int ya = (b == m0 / HoWo) ? (m0 - b * HoWo) / p.Wo : 0;
        const int yb = (b == m1 / HoWo) ? (m1 - b * HoWo) / p.Wo : p.Ho - 1;
        int r0 = ya - a.pad, r1 = yb - a.pad + a.KH;  // input rows [r0, r1)
        r0 = r0 < 0 ? 0 : r0;
        r1 = r1 > a.H ? a.H : r1;
        seg_b[n] = b; seg_r0[n] = r0; seg_nr[n] = r1 > r0 ? r1 - r0 : 0; seg_off[n] = off;
        off += a.C * seg_nr[n] * a.W;
        ++n;
      }
      nseg = n;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int sg = 0; sg < nseg; ++sg) {
      const int nr = seg_nr[sg], rowlen = a.W;
      const int64_t cstride = int64_t(a.H) * a.W;
      const uint8_t* src = a.lat_in + int64_t(seg_b[sg]) * a.C * cstride + int64_t(seg_r0[sg]) * a.W;
      uint8_t* dst = sS + seg_off[sg];
      const int total = a.C * nr * rowlen;
      for (int i = tid; i < total; i += 128) {
        const int c = i / (nr * rowlen), rest = i - c * nr * rowlen;
        dst[i] = src[int64_t(c) * cstride + rest];
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int KK = a.KH * a.KW;
    uint32_t pres[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int nchunk = kTtM * (Kp / 16);
    for (int c = tid; c < nchunk; c += 128) {
      const int row = c & (kTtM - 1), k0 = (c >> 7) * 16;  // consecutive threads: consecutive rows
      const int m = m0 + row;
      uint32_t wv[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
      if (m < p.M) {
        const int b = m / HoWo, rem = m - b * HoWo, y = rem / p.Wo, x = rem - (rem / p.Wo) * p.Wo;
        int sg = 0;
        while (seg_b[sg] != b) ++sg;
        const uint8_t* base = sS + seg_off[sg];
        const int r0 = seg_r0[sg], nr = seg_nr[sg];
        int cc = k0 / KK, r = k0 - cc * KK, ky = r / a.KW, kx = r - ky * a.KW;
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
          if (k0 + j < p.R) {
            const int yy = y + ky - a.pad, xx = x + kx - a.pad;
            uint32_t l = 255;
            if (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W) l = base[(cc * nr + (yy - r0)) * a.W + xx];
            if (l < uint32_t(T)) {
              pres[l >> 5] |= 1u << (l & 31);
              wv[j >> 2] = (wv[j >> 2] & ~(0xFFu << (8 * (j & 3)))) | (l << (8 * (j & 3)));
            }
          }
          if (++kx == a.KW) { kx = 0; if (++ky == a.KH) { ky = 0; ++cc; } }
        }
      }
      *reinterpret_cast<uint4*>(sL + tt_off(row, k0, Kp)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t v = pres[i];
      for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicOr(&present[i], v);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int n = 0;
    for (int t = 0; t < T; ++t)
      if (present[t >> 5] >> (t & 31) & 1) steps[n++] = uint8_t(t);
    nsteps = n;
  }
  __syncthreads();
  const int ns = nsteps;

  if (warp < 4) {
    // ---- producers: S[t] = [L <= t] into A buffer (k & 1) ----
    const int nwords = int(l_bytes / 16);
    for (int k = 0; k < ns; ++k) {
      const int buf = k & 1, use = k >> 1;
      if (k >= 2) mbar_wait(smem_u32(&a_empty[buf]), (use - 1) & 1);
      const uint32_t t4 = uint32_t(steps[k]) * 0x01010101u;
      const uint4* src = reinterpret_cast<const uint4*>(sL);
      uint4* dst = reinterpret_cast<uint4*>(sA0 + size_t(buf) * l_bytes);
      for (int i = tid; i < nwords; i += 128) {
        const uint4 l = src[i];
        dst[i] = make_uint4(__vcmpleu4(l.x, t4) & 0x01010101u, __vcmpleu4(l.y, t4) & 0x01010101u,
                            __vcmpleu4(l.z, t4) & 0x01010101u, __vcmpleu4(l.w, t4) & 0x01010101u);
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
      mbar_arrive(smem_u32(&a_full[buf]));
    }
  } else if (warp == 4) {
    if (lane == 0) {
      // ---- MMA issuer: D[buf] = S[t] x B (fresh accumulation per step) ----
      const uint32_t idesc = (2u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(kTtM >> 4) << 24);
      const uint32_t sbo = uint32_t(Kp) * 8;
      mbar_wait(smem_u32(&b_full), 0);
      for (int k = 0; k < ns; ++k) {
        const int buf = k & 1, use = k >> 1;
        mbar_wait(smem_u32(&a_full[buf]), use & 1);
        if (k >= 2) mbar_wait(smem_u32(&d_empty[buf]), (use - 1) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA0 + size_t(buf) * l_bytes), b_base = smem_u32(sB);
        const uint32_t d = tmem_base + uint32_t(buf * N);
        for (int ks = 0; ks < Kp / 32; ++ks)
          umma_i8(d, umma_desc(a_base + ks * 256, 128, sbo), umma_desc(b_base + ks * 256, 128, sbo), idesc, ks > 0);
        umma_commit(smem_u32(&a_empty[buf]));
        umma_commit(smem_u32(&d_full[buf]));
      }
      umma_commit(smem_u32(&mma_done));
      mbar_wait(smem_u32(&mma_done), 0);
    }
    __syncwarp();
  } else {
    // ---- epilogue: threshold test on P[t], first crossings ----
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int m = mt * kTtM + row;
    const bool mv = m < p.M;
    const int b = mv ? m / HoWo : 0, rem = mv ? m - b * HoWo : 0;
    const int fbase = ch * p.Fc;
    uint32_t fired[2] = {0u, 0u};
    for (int k = 0; k < ns; ++k) {
      const int buf = k & 1, use = k >> 1;
      const int t = steps[k];
      mbar_wait(smem_u32(&d_full[buf]), use & 1);
      tc_fence_after();
      const uint32_t trow = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(buf * N);
      for (int g = 0; g < p.Fc / 4; ++g) {
        uint32_t v[16];
        tmem_ld16(trow + uint32_t(g * 16), v);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int fl = g * 4 + j;
          const int64_t acc = int64_t(v[4 * j]) + (int64_t(v[4 * j + 1]) << 8) + (int64_t(v[4 * j + 2]) << 16) +
                              (int64_t(v[4 * j + 3]) << 24);
          if (mv && !(fired[fl >> 5] >> (fl & 31) & 1) && acc > a.thr && fbase + fl < a.F) {
            fired[fl >> 5] |= 1u << (fl & 31);
            const int64_t o = (int64_t(b) * a.F + fbase + fl) * HoWo + rem;
            a.lat_out[o] = uint8_t(t);
            a.v_out[o] = fixed_to_float(acc);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&d_empty[buf]));
    }
    if (mv)
      for (int fl = 0; fl < p.Fc; ++fl)
        if (!(fired[fl >> 5] >> (fl & 31) & 1) && fbase + fl < a.F) {
          const int64_t o = (int64_t(b) * a.F + fbase + fl) * HoWo + rem;
          a.lat_out[o] = kNoSpike;
          a.v_out[o] = 0.0f;
        }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// Returns 1 if this path does not apply (caller falls back), else an SNN code.
int conv_tct_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                    int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                    cudaStream_t s) {
  TtPlan p;
  if (!(theta >= 0.0f) || !tt_plan(B, C, H, W, pad, F, KH, KW, &p)) return 1;
  if (ws_bytes < p.b_bytes) return 1;
  TtArgs a;
  a.lat_in = lat_in; a.bq = reinterpret_cast<const uint8_t*>(ws);
  a.C = C; a.H = H; a.W = W; a.pad = pad; a.KH = KH; a.KW = KW; a.T = T; a.F = F;
  const double tt = floor(double(theta) * 2147483648.0);
  a.thr = tt >= 9.0e18 ? INT64_MAX : int64_t(tt);
  a.lat_out = lat_out; a.v_out = v_out; a.p = p;
  uint32_t cols = 32;
  while (cols < uint32_t(2 * p.N)) cols <<= 1;
  if (cols > 512) return 1;
  // TMEM has 512 columns per SM: cap the CTAs per SM through the shared-memory request
  int smem = p.smem;
  const int max_ctas = int(512 / cols);
  if (p.ctas_per_sm > max_ctas) smem = kTtSmemLimit / max_ctas - 1024;
  a.tmem_cols = cols;
  a.p = p;
  {
    const int64_t total = int64_t(p.nch) * p.N * p.Kp;
    int64_t blocks = ceil_div(total, 256);
    if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
    tt_prep_b_kernel<<<int(blocks), 256, 0, s>>>(w, F, p.R, p.Kp, p.N, p.Fc, p.nch, const_cast<uint8_t*>(a.bq),
                                                 error_word_ptr());
    note_launch();
  }
  cudaError_t e = cudaFuncSetAttribute(conv_tct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(tct): %s", cudaGetErrorString(e));
  const int mtiles = int(ceil_div(p.M, kTtM));
  conv_tct_kernel<<<unsigned(int64_t(mtiles) * p.nch), kTtThreads, smem, s>>>(a);  // 1-D: chunks fastest
  note_launch();
  return check_launch("snn_conv_fire(tct)");
}

}  // namespace snn
