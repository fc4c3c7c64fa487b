// conv_tct.cu -- a2 + a3 for a finite threshold on the tensor cores, time step by time step
// ("process all of the time-steps simultaneously"; K4).
//
// For every time step t the paper convolves the cumulative spike-wave S[t] (Eq. 1) with the weights,
// P[t] = W (*) S[t].  With the one-spike property S[t] = [lat <= t] is a binary im2col matrix,
// so P[t] is a dense int8 contraction on tcgen05: the 32-bit fixed-point weights (N1) are
// split into four u8 limbs (column n = 4 f + limb), accumulated exactly in s32 TMEM columns and
// recombined in int64 by the epilogue, which applies the threshold (spike iff P[t] > theta) and
// records the first crossing (lat = t, v = fp32(P[t])).
//
// Persistent CTAs, each bound to one chunk of Fc features (N = 4 Fc TMEM columns, weight limbs
// resident in shared memory for the whole launch), loop over tiles of 128 output positions:
//   tile prologue (all warps): gather the tile's receptive-field latencies L[128][Kp] into shared
//     memory (canonical K-major core-matrix layout) and the set of time steps that carry spikes;
//   per time step t (steps without a new spike are skipped: P[t] = P[t-1] there):
//     producer warps 4-5 write S[t] = [L <= t] (SIMD byte compares) into A buffer (step & 1),
//     warp 6 (one thread) issues Kp/32 tcgen05.mma kind::i8 into TMEM accumulator (step % nbuf),
//     epilogue warps 0-3 (TMEM lane quadrant = warp) read an earlier accumulator, test the
//     threshold and record first crossings in shared memory,
//   so building S, the MMAs and the threshold epilogue of consecutive steps overlap; one mbarrier
//   hand-off per step and role.  The tile ends as soon as every neuron of it has fired (early exit:
//   the remaining steps still pass through the pipeline but do no work); the recorded (lat, v) are
//   then written out coalesced (unfired: 255, 0).
// Shared-memory operands use the canonical K-major no-swizzle layout:
//   byte(row, k) = (row/8) * (Kp*8) + (k/16) * 128 + (row%8) * 16 + k%16, LBO = 128, SBO = Kp*8.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace snn {

constexpr int kT2M = 128;              // positions per tile (UMMA M)
constexpr int kT2Epi = 8;              // epilogue warps 0-7: TMEM lane quadrant w % 4, feature groups of parity w / 4
constexpr int kT2ProdW = 4;            // producer warps 8-11
constexpr int kT2Mma = kT2Epi + kT2ProdW;  // warp 12: TMEM allocation + MMA issue
constexpr int kT2Threads = 32 * (kT2Mma + 1);
constexpr int kT2Prod = 32 * kT2ProdW;  // producer threads
constexpr int kT2EpiT = 32 * kT2Epi;   // epilogue threads
constexpr int kT2SmemLimit = 225 * 1024;  // dynamic shared memory (227 KB per CTA minus the static part)

struct T2Plan {
  int M, R, Kp, nks, nch, Fc, N, Ho, Wo, nbuf;
  int smem, ctas_per_sm;
  uint32_t tmem_cols;
  size_t b_bytes;  // nch * N * Kp
};

static long t2_smem(int n, int fc, int Kp) {  // B + L + 2 A buffers + (lat, v) staging + alignment
  return long(n) * Kp + 3L * kT2M * Kp + 5L * kT2M * fc + 1024;
}

static bool t2_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, T2Plan* p) {
  p->Ho = H + 2 * pad - KH + 1;
  p->Wo = W + 2 * pad - KW + 1;
  if (int64_t(B) * p->Ho * p->Wo >= (int64_t(1) << 31)) return false;
  p->M = B * p->Ho * p->Wo;
  p->R = C * KH * KW;
  p->Kp = int(ceil_div(p->R, 32)) * 32;
  p->nks = p->Kp / 32;
  if (p->Kp * 8 / 16 >= (1 << 14)) return false;  // SBO field of the descriptor
  if (T > 255) return false;
  // feature chunk: the largest that runs 2 CTAs per SM, else the largest that runs 1
  const int fall = int(ceil_div(F, 4)) * 4;
  const int fcs[4] = {64, 32, 16, 8};
  int best = -1, best_ctas = 0;
  for (int i = 0; i < 4; ++i) {
    int fc = fcs[i] < fall ? fcs[i] : fall;
    if (fc < 4) fc = 4;
    const int n = 4 * fc;
    if (n % 16) continue;
    const long smem = t2_smem(n, fc, p->Kp);
    if (smem > kT2SmemLimit) continue;
    uint32_t cols = 32;
    while (cols < uint32_t(2 * n)) cols <<= 1;
    int ctas = int(kT2SmemLimit / smem);
    if (ctas > int(512 / cols)) ctas = int(512 / cols);
    if (ctas > 1) ctas = 1;  // 13 warps x ~120 registers: one CTA per SM
    if (best < 0 || ctas > best_ctas) { best = fc; best_ctas = ctas; }
    break;  // the largest chunk that fits
  }
  if (best < 0) return false;
  p->Fc = best;
  p->N = 4 * best;
  p->nch = int(ceil_div(F, best));
  p->smem = int(t2_smem(p->N, p->Fc, p->Kp));
  p->ctas_per_sm = best_ctas;
  // accumulators: as many as the CTA's share of the 512 TMEM columns holds (2 or 4)
  const int share = 512 / best_ctas;
  p->nbuf = (4 * p->N <= share) ? 4 : 2;
  uint32_t cols = 32;
  while (cols < uint32_t(p->nbuf * p->N)) cols <<= 1;
  p->tmem_cols = cols;
  p->b_bytes = size_t(p->nch) * p->N * p->Kp;
  return true;
}

bool conv_tct_applies(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta) {
  T2Plan p;
  return theta >= 0.0f && t2_plan(B, C, H, W, pad, F, KH, KW, T, &p);
}

size_t conv_tct_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T) {
  T2Plan p;
  if (!t2_plan(B, C, H, W, pad, F, KH, KW, T, &p)) return 0;
  return p.b_bytes + 256;
}

__device__ __forceinline__ uint32_t t2_off(int row, int k, int Kp) {
  return uint32_t((row >> 3) * (Kp * 8) + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

// B operand: u8 limbs of the fixed-point weights (n = 4 f_local + limb) in the full-K core-matrix
// layout, one block of N x Kp bytes per feature chunk.
__global__ void t2_prep_b_kernel(const float* __restrict__ w, int F, int R, int Kp, int N, int Fc, int nch,
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
    bq[size_t(ch) * N * Kp + t2_off(n, k, Kp)] = val;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_error(err, kErrInexact);
}

struct T2Args {
  const uint8_t* lat_in;
  const uint8_t* bq;
  int C, H, W, pad, KH, KW, T, F;
  int64_t thr;
  uint8_t* lat_out;
  float* v_out;
  T2Plan p;
  int units;  // tiles * chunks
  int dbg;    // timing experiments only (SNN_TCT_DBG): 1 = no epilogue work, 2 = no MMAs, 4 = no S writes
  int nhwc;   // output layout [B, Ho, Wo, F] (else [B, F, Ho, Wo])
};

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Threshold test of NF features (4 TMEM columns each: the limbs) at step t: exact int64
// recombination, branch-free test; first crossings are recorded in the shared staging arrays.
template <int NF>
__device__ __forceinline__ void t2_fire(const uint32_t* v, int f0, int t, uint64_t thr, uint64_t& fired,
                                        uint8_t* sLat, float* sV, int row) {
  uint64_t acc[NF];
  uint32_t hit = 0;
#pragma unroll
  for (int j = 0; j < NF; ++j) {
    acc[j] = uint64_t(v[4 * j]) + (uint64_t(v[4 * j + 1]) << 8) + (uint64_t(v[4 * j + 2]) << 16) +
             (uint64_t(v[4 * j + 3]) << 24);
    hit |= uint32_t(acc[j] > thr) << j;
  }
  hit &= ~uint32_t(fired >> f0) & ((1u << NF) - 1u);
  if (hit) {
#pragma unroll
    for (int j = 0; j < NF; ++j)
      if (hit >> j & 1) {
        sLat[(f0 + j) * kT2M + row] = uint8_t(t);
        sV[(f0 + j) * kT2M + row] = fixed_to_float(int64_t(acc[j]));
      }
    fired |= uint64_t(hit) << f0;
  }
}

// Barrier phases run continuously across the tiles of a CTA (running step counter ks): every role
// walks every step of every tile; after the tile's early exit (all neurons fired) the steps still
// pass through the pipeline, only their work (S writes, MMAs, TMEM reads) is skipped.
__global__ void __launch_bounds__(kT2Threads, 1) conv_tct_kernel(const T2Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const T2Plan& p = a.p;
  const int Kp = p.Kp, N = p.N, T = a.T, nks = p.nks, NB = p.nbuf;
  const uint32_t ab = uint32_t(kT2M) * Kp;   // bytes of L and of one A buffer
  uint8_t* sB = smem;                        // [N x Kp] weight limbs of this CTA's chunk
  uint8_t* sL = sB + size_t(N) * Kp;         // [128 x Kp] receptive-field latencies of the tile
  uint8_t* sA = sL + ab;                     // [2][128 x Kp] S[t] buffers
  float* sV = reinterpret_cast<float*>(sA + 2 * size_t(ab));  // [Fc][128] potentials at the crossing
  uint8_t* sLat = reinterpret_cast<uint8_t*>(sV + p.Fc * kT2M);  // [Fc][128] first-spike times
  __shared__ __align__(8) uint64_t a_full[2], a_empty[2], d_full[4], d_empty[4], b_full;
  __shared__ uint32_t tmem_base_sh, present[8];
  __shared__ int64_t rowout[kT2M];           // output offset (b * F) * HoWo + rem of each row, -1 = none
  __shared__ uint8_t steps[256];
  __shared__ int nsteps, rows_done;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int HoWo = p.Ho * p.Wo;
  const int KK = a.KH * a.KW;
  const int ch = int(blockIdx.x % unsigned(p.nch));  // grid is a multiple of nch: fixed chunk per CTA
  const int fbase = ch * p.Fc;

  if (warp == kT2Mma) tmem_alloc(smem_u32(&tmem_base_sh), p.tmem_cols);
  if (tid == 0) {
    mbar_init(smem_u32(&b_full), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&a_full[s]), kT2Prod);
      mbar_init(smem_u32(&a_empty[s]), 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(smem_u32(&d_full[s]), 1);
      mbar_init(smem_u32(&d_empty[s]), kT2EpiT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  if (tid == 0) {  // this chunk's weight limbs, once per launch
    const uint32_t b_bytes = uint32_t(N) * Kp;
    mbar_expect_tx(smem_u32(&b_full), b_bytes);
    const uint8_t* src = a.bq + size_t(ch) * b_bytes;
    for (uint32_t off = 0; off < b_bytes;) {
      const uint32_t nb = b_bytes - off < 65536u ? b_bytes - off : 65536u;
      bulk_g2s(smem_u32(sB + off), src + off, nb, smem_u32(&b_full));
      off += nb;
    }
  }
  if (warp == kT2Mma && lane == 0) mbar_wait(smem_u32(&b_full), 0);
  int ks = 0;  // running step counter (barrier phases)

  for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
    const int m0 = (u / p.nch) * kT2M;
    // ---------------- tile prologue ----------------
    if (tid == 0) { stop = 0; rows_done = 0; }
    if (tid < 8) present[tid] = 0;
    if (tid < kT2M) {
      const int m = m0 + tid;
      if (m < p.M) {
        const int b = m / HoWo;
        rowout[tid] = a.nhwc ? int64_t(m) * a.F + fbase : (int64_t(b) * a.F + fbase) * HoWo + (m - b * HoWo);
      } else {
        rowout[tid] = -1;
      }
    }
    for (int i = tid; i < p.Fc * kT2M; i += kT2Threads) { sLat[i] = kNoSpike; sV[i] = 0.0f; }
    __syncthreads();
    {  // gather L: item = (row, 16-byte k chunk); consecutive threads take consecutive rows
      uint32_t pres[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // time steps present (registers: static indices only)
      const int nitems = kT2M * (Kp / 16);
      for (int it = tid; it < nitems; it += kT2Threads) {
        const int row = it & (kT2M - 1), k0 = (it >> 7) * 16;
        const int m = m0 + row;
        uint32_t wv[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
        if (m < p.M) {
          const int b = m / HoWo, rem = m - b * HoWo, y = rem / p.Wo, x = rem - (rem / p.Wo) * p.Wo;
          const uint8_t* base = a.lat_in + int64_t(b) * a.C * a.H * a.W;
          int c = k0 / KK, r = k0 - c * KK, ky = r / a.KW, kx = r - ky * a.KW;
          uint32_t lv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {  // all 16 loads in flight
            const int yy = y + ky - a.pad, xx = x + kx - a.pad;
            lv[j] = (k0 + j < p.R && yy >= 0 && yy < a.H && xx >= 0 && xx < a.W)
                        ? uint32_t(__ldg(base + (int64_t(c) * a.H + yy) * a.W + xx)) : 255u;
            if (++kx == a.KW) { kx = 0; if (++ky == a.KH) { ky = 0; ++c; } }
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t l = lv[j] < uint32_t(T) ? lv[j] : 255u;
            wv[j >> 2] = (wv[j >> 2] & ~(0xFFu << (8 * (j & 3)))) | (l << (8 * (j & 3)));
            if (T <= 32) {
              pres[0] |= l < 32u ? (1u << l) : 0u;
            } else {
#pragma unroll
              for (int w = 0; w < 8; ++w) pres[w] |= (l >> 5) == uint32_t(w) && l != 255u ? (1u << (l & 31)) : 0u;
            }
          }
        }
        *reinterpret_cast<uint4*>(sL + t2_off(row, k0, Kp)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t v = pres[i];
#pragma unroll
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

    if (warp >= kT2Epi && warp < kT2Mma) {
      // ---------------- producers: S[t] = [L <= t] into A buffer (ks & 1) ----------------
      const int pt = tid - kT2EpiT;
      const uint4* src = reinterpret_cast<const uint4*>(sL);
      const int nw = int(ab / 16);
      for (int k = 0; k < ns; ++k) {
        const int s = (ks + k) & 1, use = (ks + k) >> 1;
        if (use > 0) mbar_wait(smem_u32(&a_empty[s]), (use - 1) & 1);
        if (!stop && !(a.dbg & 4)) {
          const uint32_t t4 = uint32_t(steps[k]) * 0x01010101u;
          uint4* dst = reinterpret_cast<uint4*>(sA + size_t(s) * ab);
#pragma unroll 4
          for (int i = pt; i < nw; i += kT2Prod) {
            const uint4 l = src[i];
            dst[i] = make_uint4(__vcmpleu4(l.x, t4) & 0x01010101u, __vcmpleu4(l.y, t4) & 0x01010101u,
                                __vcmpleu4(l.z, t4) & 0x01010101u, __vcmpleu4(l.w, t4) & 0x01010101u);
          }
          fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        }
        mbar_arrive(smem_u32(&a_full[s]));
      }
    } else if (warp == kT2Mma) {
      // ---------------- MMA issuer: D[ks % nbuf] = S[t_k] x B ----------------
      if (lane == 0) {
        const uint32_t idesc = (2u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(kT2M >> 4) << 24);
        const uint32_t sbo = uint32_t(Kp) * 8;
        const uint32_t b_base = smem_u32(sB), a_base0 = smem_u32(sA);
        for (int k = 0; k < ns; ++k) {
          const int kg = ks + k;
          const int s = kg & 1, d = kg % NB;
          mbar_wait(smem_u32(&a_full[s]), (kg >> 1) & 1);
          if (kg >= NB) mbar_wait(smem_u32(&d_empty[d]), ((kg / NB) - 1) & 1);
          tc_fence_after();
          if (!stop && !(a.dbg & 2)) {
            const uint32_t a_base = a_base0 + uint32_t(s) * ab, dt = tmem_base + uint32_t(d * N);
            for (int j = 0; j < nks; ++j)
              umma_i8(dt, umma_desc(a_base + j * 256, 128, sbo), umma_desc(b_base + j * 256, 128, sbo), idesc, j > 0);
          }
          umma_commit(smem_u32(&a_empty[s]));  // A buffer free once these MMAs have read it
          umma_commit(smem_u32(&d_full[d]));
        }
      }
      __syncwarp();
    } else {
      // ---------------- epilogue: threshold test on P[t], first crossings ----------------
      const int q = warp & 3, half = warp >> 2;  // TMEM lane quadrant, feature-group parity
      const int row = q * 32 + lane;
      const bool mv = rowout[row] >= 0;
      // this warp's features: groups g (8 features) with g % 2 == half, plus the tail group of 4
      uint64_t mine = 0;
      for (int f = 0; f < p.Fc; ++f)
        if (((f >> 3) & 1) == half) mine |= 1ull << f;
      uint64_t fired = ~mine;
      for (int f = 0; f < p.Fc; ++f)
        if (!mv || fbase + f >= a.F) fired |= 1ull << f;
      bool wdone = __all_sync(0xffffffffu, fired == ~0ull);
      if (wdone && lane == 0 && atomicAdd(&rows_done, 1) + 1 == kT2Epi) stop = 1;
      const uint32_t trow = tmem_base + (uint32_t(q * 32) << 16);
      for (int k = 0; k < ns; ++k) {
        const int kg = ks + k;
        const int d = kg % NB;
        mbar_wait(smem_u32(&d_full[d]), (kg / NB) & 1);
        tc_fence_after();
        if (!wdone && !(a.dbg & 1)) {  // warp-uniform
          const int t = steps[k];
          const uint32_t tcol = trow + uint32_t(d * N);
          for (int g = half; g < p.Fc / 8; g += 2) {
            // skip groups whose 8 x 32 neurons all fired (TMEM reads are 64 B/clk/SM)
            if (__all_sync(0xffffffffu, ((fired >> (g * 8)) & 0xFFull) == 0xFFull)) continue;
            uint32_t v[32];
            tmem_ld32(tcol + uint32_t(g * 32), v);
            t2_fire<8>(v, g * 8, t, uint64_t(a.thr), fired, sLat, sV, row);
          }
          if ((p.Fc & 7) && ((p.Fc >> 3) & 1) == half &&
              !__all_sync(0xffffffffu, ((fired >> (p.Fc & ~7)) & 0xFull) == 0xFull)) {  // tail of 4
            uint32_t v[16];
            tmem_ld16(tcol + uint32_t((p.Fc & ~7) * 4), v);
            t2_fire<4>(v, p.Fc & ~7, t, uint64_t(a.thr), fired, sLat, sV, row);
          }
          wdone = __all_sync(0xffffffffu, fired == ~0ull);
          if (wdone && lane == 0 && atomicAdd(&rows_done, 1) + 1 == kT2Epi) stop = 1;
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&d_empty[d]));
      }
      // coalesced write-out of the tile: consecutive threads take consecutive rows of one feature
      asm volatile("bar.sync 1, %0;" ::"n"(kT2EpiT) : "memory");
      const int nf = (a.F - fbase) < p.Fc ? (a.F - fbase) : p.Fc;
      for (int i = tid; i < nf * kT2M; i += kT2EpiT) {
        const int f = i >> 7, r = i & (kT2M - 1);
        const int64_t o = rowout[r];
        if (o >= 0) {
          const int64_t fo = a.nhwc ? int64_t(f) : int64_t(f) * HoWo;
          a.lat_out[o + fo] = sLat[i];
          if (a.v_out) a.v_out[o + fo] = sV[i];
        }
      }
    }
    ks += ns;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (warp == kT2Mma) tmem_dealloc(tmem_base, p.tmem_cols);
}

// Returns 1 if this path does not apply (caller falls back), else an SNN code.
int conv_tct_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                    int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                    cudaStream_t s, int nhwc) {
  T2Plan p;
  if (!(theta >= 0.0f) || !t2_plan(B, C, H, W, pad, F, KH, KW, T, &p)) return 1;
  if (ws_bytes < p.b_bytes) return 1;
  T2Args a;
  a.lat_in = lat_in; a.bq = reinterpret_cast<const uint8_t*>(ws);
  a.C = C; a.H = H; a.W = W; a.pad = pad; a.KH = KH; a.KW = KW; a.T = T; a.F = F;
  const double tt = floor(double(theta) * 2147483648.0);
  a.thr = tt >= 9.0e18 ? INT64_MAX : int64_t(tt);
  a.lat_out = lat_out; a.v_out = v_out; a.p = p; a.nhwc = nhwc;
  a.dbg = getenv("SNN_TCT_DBG") ? atoi(getenv("SNN_TCT_DBG")) : 0;
  const int mtiles = int(ceil_div(p.M, kT2M));
  a.units = mtiles * p.nch;
  {
    const int64_t total = int64_t(p.nch) * p.N * p.Kp;
    int64_t blocks = ceil_div(total, 256);
    if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
    t2_prep_b_kernel<<<int(blocks), 256, 0, s>>>(w, F, p.R, p.Kp, p.N, p.Fc, p.nch, const_cast<uint8_t*>(a.bq),
                                                 error_word_ptr(s));
    note_launch();
  }
  // TMEM (512 columns per SM) and shared memory both cap the resident CTAs: request enough shared
  // memory that no more than ctas_per_sm land on one SM
  int smem = p.smem;
  const int min_smem = kT2SmemLimit / (p.ctas_per_sm + 1) + 1024;  // (ctas_per_sm + 1) CTAs do not fit
  if (smem < min_smem) smem = min_smem;
  if (smem > kT2SmemLimit) smem = kT2SmemLimit;
  cudaError_t e = cudaFuncSetAttribute(conv_tct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(tct): %s", cudaGetErrorString(e));
  int grid = num_sms() * p.ctas_per_sm;
  grid = (grid / p.nch) * p.nch;
  if (grid < p.nch) grid = p.nch;
  if (grid > a.units) grid = int(ceil_div(a.units, p.nch)) * p.nch;
  conv_tct_kernel<<<grid, kT2Threads, smem, s>>>(a);
  note_launch();
  return check_launch("snn_conv_fire(tct)");
}

}  // namespace snn
