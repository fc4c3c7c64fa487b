// conv_tc.cu -- a2 + a3 for an infinite threshold (Eq. 5) on the 5th-generation tensor
// cores (tcgen05, sm_100a).  With theta = +inf only P[T-1] matters, and P[T-1] is a dense contraction
// of the binary spike-wave at the last step, S[T-1] (every spiking input counts), with the weights:
//     P[pos, f] = sum_k A[pos, k] * Wq[f, k],   A = im2col(S[T-1]) in {0, 1},  Wq = w * 2^31 (uint32)
// Exactness (N1): Wq is split into four u8 limbs, Wq = sum_l L_l * 2^(8 l); each limb GEMM
// runs as tcgen05.mma kind::i8 (u8 x u8 -> s32; max column sum 255 * 6250 < 2^31, exact) and the
// epilogue recombines the four int32 accumulators in int64.  The limbs are interleaved feature-major
// in the N dimension (n = 4 f + l), so one 16-column TMEM load yields 4 features x 4 limbs.
//
// Operands are staged by tiny prep kernels in the canonical K-major, no-swizzle UMMA layout: per
// (row tile, 128-byte K tile) a block of 8x16-byte core matrices [row/8][k/16][row%8][16 B]
// (LBO = 128 B between K-adjacent core matrices, SBO = 1024 B between 8-row groups), so the GEMM's
// producer moves each stage with two contiguous cp.async.bulk copies completing on an mbarrier.
// Warp roles: warp 0 = bulk-copy producer, warp 1 = MMA issuer (one elected thread), warp 2 = TMEM
// allocator, warps 4..7 = epilogue (TMEM lane quadrant = warp % 4).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace snn {

constexpr int kTcM = 128;          // UMMA M (one CTA)
constexpr int kTcKT = 128;         // bytes (= int8 elements) of K per pipeline stage
#ifndef SNN_TC_STAGES
#define SNN_TC_STAGES 4
#endif
constexpr int kTcStages = SNN_TC_STAGES;
constexpr int kTcThreads = 256;

struct TcPlan {
  int M, K, Kp, Mt, Kt, nch, Fc, N;  // N = 4 * Fc (multiple of 16, <= 256)
  size_t a_bytes, b_bytes;
  // A from a shared-memory band of RB output rows (nbands per image) when band = 1; with hwc = 1 the
  // K order is (ky, kx, c) with channels padded to Cp (a multiple of 16), so every 16-byte core-matrix
  // row of A is 16 channels of one input pixel: one 16-byte shared-memory load per row.  Otherwise K
  // is the receptive-field order (c, ky, kx).
  int band, hwc, Cp, RB, nbands, band_smem;
  // split-K for grids too small to fill the GPU (C4's one-image layer: 2 x 2 tiles): KS CTAs share an
  // output tile, each adds its exact integer partial sums into part[M][F] (int64, atomics; integer
  // addition is order-free, so the result stays exact) and a finalize kernel writes (lat, v)
  int KS;
  size_t part_bytes;
  // K9 (fcP > 0): the layer rewritten as a fully connected one -- a kernel larger than its input (H W < KH KW,
  // C2's third layer: 5 x 5 on a 4 x 4 map) makes most of the im2col padding, so every output position p
  // becomes fcF features of a "KH = H, KW = W, pad 0" layer with fcP fcF features, whose weights are the real
  // kernel shifted by p (zero where the shifted tap leaves the kernel).  fcF = the real F, fcP = the real
  // Ho Wo; fcW / fcWo / fcPad / fcKH / fcKW = the real geometry (B operand gather, output index).
  int fcF, fcP, fcW, fcWo, fcPad, fcKH, fcKW;
  size_t fc_l_bytes;  // K9: the real weights' limb rows L[F][4][KH KW][Cp]
};

static TcPlan tc_plan(int B, int C, int H, int W, int pad, int KH, int KW, int F, int sms) {
  TcPlan p;
  const int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1, Wp = W + 2 * pad;
  const int R = C * KH * KW;
  p.M = B * Ho * Wo;
  // bands: the largest band of output rows whose padded input rows fit 48 KB of shared memory; a batch
  // too small to give every SM two bands keeps the per-row gather kernel (and the (c, ky, kx) order)
  const int Cp16 = int(ceil_div(C, 16)) * 16;
  p.RB = Ho;
  while (p.RB > 1 && int64_t(Cp16) * (p.RB + KH - 1) * Wp > 48 * 1024) p.RB = (p.RB + 1) / 2;
  p.nbands = int(ceil_div(Ho, p.RB));
  p.band = int64_t(Cp16) * (p.RB + KH - 1) * Wp <= 48 * 1024 && int64_t(B) * p.nbands >= 2 * sms;
  p.hwc = p.band && (C % 16 == 0 || (C >= 64 && int64_t(Cp16) * 100 <= int64_t(C) * 104));
  p.Cp = p.hwc ? Cp16 : C;
  p.band_smem = int((int64_t(p.Cp) * (p.RB + KH - 1) * Wp + 15) & ~int64_t(15));
  p.K = p.hwc ? KH * KW * p.Cp : R;
  p.Kp = int(ceil_div(p.K, kTcKT)) * kTcKT;
  p.Mt = int(ceil_div(p.M, kTcM));
  p.Kt = p.Kp / kTcKT;
  p.nch = int(ceil_div(F, 64));
  if (const char* e = getenv("SNN_TC_NCH")) {  // tuning experiments: feature chunks (N = 4 * ceil(F / nch) <= 256)
    const int v = atoi(e);
    if (v >= p.nch && v <= F) p.nch = v;
  }
  p.Fc = int(ceil_div(ceil_div(F, p.nch), 4)) * 4;
  p.N = 4 * p.Fc;
  p.a_bytes = size_t(p.Mt) * p.Kt * kTcM * kTcKT;
  p.b_bytes = size_t(p.nch) * p.Kt * p.N * kTcKT;
  const int tiles = p.Mt * p.nch;
  p.KS = 1;
  if (tiles * 2 < sms) {  // at least 4 K tiles per slice (pipeline depth, atomic traffic)
    p.KS = sms / tiles < p.Kt / 4 ? sms / tiles : p.Kt / 4;
    if (p.KS < 1) p.KS = 1;
  }
  p.part_bytes = p.KS > 1 ? size_t(p.M) * F * sizeof(int64_t) : 0;
  p.fcF = p.fcP = p.fcW = p.fcWo = p.fcPad = p.fcKH = p.fcKW = 0;
  p.fc_l_bytes = 0;
  return p;
}

// K9: the fully connected rewrite of a theta = inf layer whose kernel is larger than its input.  Returns
// true and the rewritten plan (virtual layer: pad 0, KH = H, KW = W, Ho Wo F features, one position per
// image) when it applies: fewer K columns than the im2col (H W < KH KW), the (ky, kx, c) K order (the B
// gather below assumes it), and a feature count the chunking handles.  SNN_TC_FC=0 turns it off.
static bool tc_fc_plan(int B, int C, int H, int W, int pad, int KH, int KW, int F, int sms, TcPlan* out) {
  const int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
  if (const char* e = getenv("SNN_TC_FC")) if (e[0] == '0') return false;
  if (Ho < 1 || Wo < 1 || H * W >= KH * KW || int64_t(Ho) * Wo * F > 32768) return false;
  TcPlan p = tc_plan(B, C, H, W, 0, H, W, Ho * Wo * F, sms);
  if (!p.hwc) return false;
  p.fcF = F; p.fcP = Ho * Wo; p.fcW = W; p.fcWo = Wo; p.fcPad = pad; p.fcKH = KH; p.fcKW = KW;
  p.fc_l_bytes = (size_t(F) * 4 * KH * KW * p.Cp + 1023) & ~size_t(1023);
  *out = p;
  return true;
}

int conv_tc_launches(int B, int C, int H, int W, int pad, int KH, int KW, int F) {
  TcPlan p = tc_plan(B, C, H, W, pad, KH, KW, F, num_sms()), q;
  if (tc_fc_plan(B, C, H, W, pad, KH, KW, F, num_sms(), &q)) p = q;  // K9
  return (p.KS > 1 ? 4 : 3) + (p.fcP ? 1 : 0);  // prep B (K9: two kernels), prep A, GEMM (+ finalize)
}

size_t conv_tc_workspace(int B, int C, int H, int W, int pad, int KH, int KW, int F) {
  TcPlan p = tc_plan(B, C, H, W, pad, KH, KW, F, num_sms());
  size_t n = ((p.a_bytes + 1023) & ~size_t(1023)) + ((p.b_bytes + 1023) & ~size_t(1023)) + p.part_bytes + 1024;
  TcPlan q;
  if (tc_fc_plan(B, C, H, W, pad, KH, KW, F, num_sms(), &q)) {  // K9: either plan may run (prepared A: the first)
    const size_t m = ((q.a_bytes + 1023) & ~size_t(1023)) + ((q.b_bytes + 1023) & ~size_t(1023)) + q.part_bytes +
                     q.fc_l_bytes + 2048;
    if (m > n) n = m;
  }
  return n;
}

// byte offset of element (row, k) inside a [row tiles][K tiles] blocked core-matrix array
__device__ __forceinline__ size_t tc_off(int row, int k, int rows_per_tile, int Kt) {
  const int rt = row / rows_per_tile, r = row - rt * rows_per_tile;
  const int kt = k / kTcKT, kk = k - kt * kTcKT;
  return (size_t(rt) * Kt + kt) * size_t(rows_per_tile) * kTcKT + size_t(r >> 3) * 1024 + (kk >> 4) * 128 +
         (r & 7) * 16 + (kk & 15);
}

// A operand: binary im2col of the spike-wave at T-1 (any spike, since every spike time is <= T-1).
// One thread per 16-byte core-matrix row = 16 consecutive receptive-field entries of one position.
// grid.y > 1: blockIdx.y is an image of a batch prepared image by image (snn_conv_inf_prepare), each
// with its own one-image plan p and an A block of img_bytes.
__global__ void tc_prep_a_kernel(const uint8_t* __restrict__ lat_in, int C, int H, int W, int pad, int KH, int KW,
                                 int Ho, int Wo, int T, TcPlan p, uint8_t* __restrict__ aq, size_t img_bytes,
                                 int in_nhwc) {
  pdl_begin();
  lat_in += int64_t(blockIdx.y) * C * H * W;
  aq += size_t(blockIdx.y) * img_bytes;
  const int KK = KH * KW;
  const int64_t rows16 = int64_t(p.Mt) * kTcM * (p.Kp / 16);
  const int nk16 = p.Kp / 16;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows16; i += int64_t(gridDim.x) * blockDim.x) {
    // 8 consecutive threads fill the 8 rows of one 128-byte core matrix (coalesced 16-byte stores)
    const int r8 = int(i & 7);
    const int64_t rest = i >> 3;
    const int k0 = int(rest % nk16) * 16;
    const int m = int(rest / nk16) * 8 + r8;
    uint32_t wv[4] = {0, 0, 0, 0};
    if (m < p.M) {
      const int HoWo = Ho * Wo;
      const int b = m / HoWo, rem = m - b * HoWo, y = rem / Wo, x = rem - (rem / Wo) * Wo;
      int c = k0 / KK, r = k0 - c * KK, ky = r / KW, kx = r - ky * KW;
      const uint8_t* base = lat_in + int64_t(b) * C * H * W;
      uint32_t lv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // addresses and predicates first, then all loads in flight
        const int yy = y + ky - pad, xx = x + kx - pad;
        const bool in = k0 + j < p.K && yy >= 0 && yy < H && xx >= 0 && xx < W;
        lv[j] = in ? base[in_nhwc ? (int64_t(yy) * W + xx) * C + c : (int64_t(c) * H + yy) * W + xx] : 0xFFu;
        if (++kx == KW) { kx = 0; if (++ky == KH) { ky = 0; ++c; } }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (lv[j] < uint32_t(T)) wv[j >> 2] |= 1u << (8 * (j & 3));
    }
    *reinterpret_cast<uint4*>(aq + tc_off(m, k0, kTcM, p.Kt)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

// B operand, vectorised: one thread per (chunk, feature, 16 consecutive k): 16 weights -> the four
// 16-byte limb rows n = 4 f_local + limb of one core-matrix column.
__global__ void tc_prep_b16_kernel(const float* __restrict__ w, int F, int R, int KK, TcPlan p,
                                   uint8_t* __restrict__ bq, int* err) {
  pdl_begin();
  const int nk16 = p.Kp / 16;
  const int64_t total = int64_t(p.nch) * p.Fc * nk16;
  int bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int k16 = int(i % nk16);
    const int64_t rest = i / nk16;
    const int fl = int(rest % p.Fc), ch = int(rest / p.Fc);
    const int f = ch * p.Fc + fl, k0 = k16 * 16;
    uint32_t limb[4][4] = {};
    if (f < F && k0 < p.K) {
      // weight index of GEMM column k: (c, ky, kx) order = k itself; (ky, kx, c) order = c * KK + kyx
      const int kyx = p.hwc ? k0 / p.Cp : 0, c0 = p.hwc ? k0 - kyx * p.Cp : 0;
      const int C = R / KK;
      float xs[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // all 16 loads issued before any use
        const bool in = p.hwc ? (c0 + j < C) : (k0 + j < R);
        const int widx = p.hwc ? (c0 + j) * KK + kyx : k0 + j;
        xs[j] = in ? __ldg(w + int64_t(f) * R + widx) : 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float x = xs[j];
        const float s = x * 2147483648.0f;
        if (!(x >= 0.0f && x <= 1.0f) || s != truncf(s)) { bad = 1; continue; }
        const uint32_t q = uint32_t(s);
#pragma unroll
        for (int l = 0; l < 4; ++l) limb[l][j >> 2] |= ((q >> (8 * l)) & 0xFFu) << (8 * (j & 3));
      }
    }
    uint8_t* base = bq + size_t(ch) * p.Kt * p.N * kTcKT;
#pragma unroll
    for (int l = 0; l < 4; ++l)
      *reinterpret_cast<uint4*>(base + tc_off(4 * fl + l, k0, p.N, p.Kt)) =
          make_uint4(limb[l][0], limb[l][1], limb[l][2], limb[l][3]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_error(err, kErrInexact);
}

// K9 B operand, stage 1: the real weights as limb rows L[f][limb][tap][Cp] (bytes; tap = ky KW + kx, channels
// padded to Cp with zeros): one thread per (feature, tap, 16 channels), the arithmetic of tc_prep_b16_kernel.
__global__ void tc_prep_limbs_kernel(const float* __restrict__ w, int F, int C, int KK, int Cp,
                                     uint8_t* __restrict__ L, int* err) {
  pdl_begin();
  const int nc16 = Cp / 16;
  const int64_t total = int64_t(F) * KK * nc16;
  int bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int c16 = int(i % nc16);
    const int64_t rest = i / nc16;
    const int tap = int(rest % KK), f = int(rest / KK), c0 = c16 * 16;
    float xs[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) xs[j] = c0 + j < C ? __ldg(w + (int64_t(f) * C + c0 + j) * KK + tap) : 0.0f;
    uint32_t limb[4][4] = {};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = xs[j];
      const float sx = x * 2147483648.0f;
      if (!(x >= 0.0f && x <= 1.0f) || sx != truncf(sx)) { bad = 1; continue; }
      const uint32_t q = uint32_t(sx);
#pragma unroll
      for (int l = 0; l < 4; ++l) limb[l][j >> 2] |= ((q >> (8 * l)) & 0xFFu) << (8 * (j & 3));
    }
#pragma unroll
    for (int l = 0; l < 4; ++l)
      *reinterpret_cast<uint4*>(L + ((int64_t(f) * 4 + l) * KK + tap) * Cp + c0) =
          make_uint4(limb[l][0], limb[l][1], limb[l][2], limb[l][3]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_error(err, kErrInexact);
}

// K9 B operand, stage 2: the virtual layer's limb rows are 16-byte pieces of L -- virtual feature
// (position pp = (y, x), real feature fr), virtual tap = input pixel (iy, ix): the real tap
// (iy - y + pad, ix - x + pad), or zeros where it leaves the kernel.  One thread per (chunk, virtual
// feature, 16 consecutive k) as in tc_prep_b16_kernel; consecutive threads read consecutive 16-byte pieces.
__global__ void tc_prep_b_fc_kernel(const uint8_t* __restrict__ L, int Fv, TcPlan p, uint8_t* __restrict__ bq) {
  pdl_begin();
  const int nk16 = p.Kp / 16, KK = p.fcKH * p.fcKW;
  const int64_t total = int64_t(p.nch) * p.Fc * nk16;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int k16 = int(i % nk16);
    const int64_t rest = i / nk16;
    const int fl = int(rest % p.Fc), ch = int(rest / p.Fc);
    const int f = ch * p.Fc + fl, k0 = k16 * 16;
    const uint8_t* src = nullptr;
    if (f < Fv && k0 < p.K) {
      const int pix = k0 / p.Cp, c0 = k0 - pix * p.Cp;
      const int pp = f / p.fcF, fr = f - pp * p.fcF, y = pp / p.fcWo, x = pp - y * p.fcWo;
      const int iy = pix / p.fcW, ix = pix - iy * p.fcW;
      const int ky = iy - y + p.fcPad, kx = ix - x + p.fcPad;
      if (ky >= 0 && ky < p.fcKH && kx >= 0 && kx < p.fcKW)
        src = L + (int64_t(fr) * 4 * KK + ky * p.fcKW + kx) * p.Cp + c0;
    }
    uint8_t* base = bq + size_t(ch) * p.Kt * p.N * kTcKT;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const uint4 v = src ? __ldg(reinterpret_cast<const uint4*>(src + int64_t(l) * KK * p.Cp)) : make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(base + tc_off(4 * fl + l, k0, p.N, p.Kt)) = v;
    }
  }
}

// K9 A operand: row m = image m, K order (input pixel, channel padded to Cp) -- the binary S[T-1] of the
// whole (small) input map, no im2col.  One thread per 16-byte core-matrix row (image, pixel, 16 channels);
// a warp takes 8 consecutive images x 4 consecutive 16-channel pieces, i.e. four whole 128-byte core
// matrices per store and 64 contiguous input bytes per image per load step (channels-last input); rows
// M .. Mt * 128 and the K padding are zero-filled.  (Kp is a multiple of 128, so nk16 is a multiple of 4.)
__global__ void tc_prep_a_fc_kernel(const uint8_t* __restrict__ lat_in, int C, int HW, int T, TcPlan p,
                                    uint8_t* __restrict__ aq, int in_nhwc) {
  pdl_begin();
  const int nk16 = p.Kp / 16, rows = p.Mt * kTcM, mblocks = rows / 8;
  const int64_t total = int64_t(rows) * nk16;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int lane = int(i & 31);
    const int64_t wg = i >> 5;  // (8-image block, quad of 16-channel pieces); total is a multiple of 32
    const int m = int(wg % mblocks) * 8 + (lane & 7), k0 = (int(wg / mblocks) * 4 + (lane >> 3)) * 16;
    uint32_t wv[4] = {0u, 0u, 0u, 0u};
    if (m < p.M && k0 < p.K) {
      const int pix = k0 / p.Cp, c0 = k0 - pix * p.Cp;
      const uint8_t* lb = lat_in + int64_t(m) * C * HW;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = c0 + j;
        if (c < C) {
          const uint8_t l = __ldg(lb + (in_nhwc ? int64_t(pix) * C + c : int64_t(c) * HW + pix));
          wv[j >> 2] |= (l < T ? 1u : 0u) << (8 * (j & 3));
        }
      }
    }
    *reinterpret_cast<uint4*>(aq + tc_off(m, k0, kTcM, p.Kt)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

// A operand from a shared-memory band: one CTA per (image, band of RB output rows) stages the binary
// spike-wave S[T-1] of the band's input rows (zero padded, [C][RB + KH - 1][W + 2 pad]) once, then
// writes the band's core-matrix rows (16 receptive-field entries of one position per thread,
// consecutive threads = consecutive positions, so 8 threads fill one 128-byte core matrix).  KS CTAs
// share a band (each stages it and writes every KS-th 16-byte K column), so small batches still fill
// the GPU.  The last CTA zero-fills the padding rows M .. Mt * 128.
__global__ void __launch_bounds__(256) tc_prep_a_band_kernel(const uint8_t* __restrict__ lat_in, int C, int H, int W,
                                                             int pad, int KH, int KW, int Ho, int Wo, int T,
                                                             TcPlan p, int RB, int nbands, int B, int KS,
                                                             uint8_t* __restrict__ aq, int in_nhwc) {
  pdl_begin();
  extern __shared__ uint8_t band[];
  const int Wp = W + 2 * pad, TR = RB + KH - 1, KK = KH * KW, nk16 = p.Kp / 16;
  if (int(blockIdx.x) == B * nbands * KS) {  // padding rows
    const int64_t rows = (int64_t(p.Mt) * kTcM - p.M) * nk16;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      const int m = p.M + int(i % (p.Mt * kTcM - p.M)), k16 = int(i / (p.Mt * kTcM - p.M));
      *reinterpret_cast<uint4*>(aq + tc_off(m, k16 * 16, kTcM, p.Kt)) = make_uint4(0, 0, 0, 0);
    }
    return;
  }
  const int ks = blockIdx.x % KS, bb = blockIdx.x / KS;
  const int b = bb / nbands, ya = (bb % nbands) * RB;
  const int yb = ya + RB < Ho ? ya + RB : Ho;
  const uint8_t* lb = lat_in + int64_t(b) * C * H * W;
  {  // zero the band (padding never spikes), then scatter the band's input rows (coalesced per channel)
    uint4* b16 = reinterpret_cast<uint4*>(band);
    for (int i = threadIdx.x; i < (C * TR * Wp + 15) / 16; i += blockDim.x) b16[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int top = ya - pad;  // input row of band row 0
    const int iy0 = top > 0 ? top : 0, iy1 = (top + TR - 1 < H - 1 ? top + TR - 1 : H - 1);
    const int nr = iy1 - iy0 + 1, per_c = nr * W;
    for (int i = threadIdx.x; i < C * per_c; i += blockDim.x) {
      const int c = i / per_c, r = i - c * per_c, ry = r / W, ix = r - ry * W;
      const int64_t li = in_nhwc ? (int64_t(iy0 + ry) * W + ix) * C + c : (int64_t(c) * H + iy0 + ry) * W + ix;
      band[(c * TR + iy0 + ry - top) * Wp + ix + pad] = __ldg(lb + li) < T ? 1 : 0;
    }
  }
  const int mcount = (yb - ya) * Wo, m0 = b * Ho * Wo + ya * Wo;
  const int nks = (nk16 - ks + KS - 1) / KS;  // this CTA's K columns: ks, ks + KS, ...
  for (int i = threadIdx.x; i < mcount * nks; i += blockDim.x) {
    const int k16 = ks + (i / mcount) * KS, mi = i - (i / mcount) * mcount;
    const int yl = mi / Wo, x = mi - yl * Wo, k0 = k16 * 16;
    int c = k0 / KK, r = k0 - c * KK, ky = r / KW, kx = r - ky * KW;
    uint32_t wv[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (k0 + j < p.K) wv[j >> 2] |= uint32_t(band[(c * TR + yl + ky) * Wp + x + kx]) << (8 * (j & 3));
      if (++kx == KW) { kx = 0; if (++ky == KH) { ky = 0; ++c; } }
    }
    *reinterpret_cast<uint4*>(aq + tc_off(m0 + mi, k0, kTcM, p.Kt)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

// A operand, (ky, kx, c) order: the band is staged channel-innermost ([RB + KH - 1][W + 2 pad][Cp],
// binary S[T-1], zero padded), so each core-matrix row (16 channels of one input pixel) is one 16-byte
// shared-memory load and one 16-byte global store.
__global__ void __launch_bounds__(256) tc_prep_a_hwc_kernel(const uint8_t* __restrict__ lat_in, int C, int H, int W,
                                                            int pad, int KH, int KW, int Ho, int Wo, int T, TcPlan p,
                                                            int B, uint8_t* __restrict__ aq, int in_nhwc) {
  pdl_begin();
  extern __shared__ __align__(16) uint8_t hband[];
  const int Wp = W + 2 * pad, TR = p.RB + KH - 1, Cp = p.Cp, nk16 = p.Kp / 16;
  if (int(blockIdx.x) == B * p.nbands) {  // padding rows
    const int pr = p.Mt * kTcM - p.M;
    for (int64_t i = threadIdx.x; i < int64_t(pr) * nk16; i += blockDim.x) {
      const int m = p.M + int(i % pr), k16 = int(i / pr);
      *reinterpret_cast<uint4*>(aq + tc_off(m, k16 * 16, kTcM, p.Kt)) = make_uint4(0, 0, 0, 0);
    }
    return;
  }
  const int b = blockIdx.x / p.nbands, ya = (blockIdx.x % p.nbands) * p.RB;
  const int yb = ya + p.RB < Ho ? ya + p.RB : Ho;
  const uint8_t* lb = lat_in + int64_t(b) * C * H * W;
  {
    uint4* b16 = reinterpret_cast<uint4*>(hband);
    for (int i = threadIdx.x; i < p.band_smem / 16; i += blockDim.x) b16[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int top = ya - pad;
    const int iy0 = top > 0 ? top : 0, iy1 = (top + TR - 1 < H - 1 ? top + TR - 1 : H - 1);
    const int npx = (iy1 - iy0 + 1) * W;
    for (int i = threadIdx.x; i < C * npx; i += blockDim.x) {  // channel fastest: conflict-free byte stores
      const int px = i / C, c = i - px * C, ry = px / W, ix = px - ry * W;
      // channels-last input: i runs along memory (coalesced); planar input: a byte gather per channel
      const int64_t li = in_nhwc ? int64_t(iy0) * W * C + i : (int64_t(c) * H + iy0 + ry) * W + ix;
      hband[((iy0 + ry - top) * Wp + ix + pad) * Cp + c] = __ldg(lb + li) < T ? 1 : 0;
    }
  }
  __syncthreads();
  const int mcount = (yb - ya) * Wo, m0 = b * Ho * Wo + ya * Wo;
  const int kcols = p.K / 16;  // columns >= K / 16 are zero (K = KH KW Cp is a multiple of 16)
  for (int i = threadIdx.x; i < mcount * nk16; i += blockDim.x) {
    const int k16 = i / mcount, mi = i - k16 * mcount;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (k16 < kcols) {
      const int k0 = k16 * 16, kyx = k0 / Cp, c0 = k0 - kyx * Cp, ky = kyx / KW, kx = kyx - ky * KW;
      const int yl = mi / Wo, x = mi - yl * Wo;
      v = *reinterpret_cast<const uint4*>(hband + ((yl + ky) * Wp + x + kx) * Cp + c0);
    }
    *reinterpret_cast<uint4*>(aq + tc_off(m0 + mi, k16 * 16, kTcM, p.Kt)) = v;
  }
}

// ------------------------------------------------------------------------------- the GEMM
// Implicit im2col (K8): with lat != nullptr the A operand is not read from aq but built in the CTA.  The
// binary spike-wave S[T-1] of the input pixels the M tile's receptive fields touch -- per image of the
// tile, the input rows its output rows need, full width, channels padded to Cp -- is staged once into
// shared memory (the "band", foot bytes); then per pipeline stage the four epilogue warps (idle until the
// accumulator is done) write the stage's A tile -- row r = position mt * 128 + r, 16-byte core-matrix rows
// of 16 channels of one input pixel, (ky, kx, c) K order, zero outside the input -- in the canonical
// K-major layout, fence the generic-proxy stores for the tensor core and arrive on the stage's full
// barrier next to the producer's B bulk copy.  No A operand in HBM (tc_prep_a_hwc's write + the GEMM's
// read of Mt x Kp x 128 bytes).
struct TcImpl {
  const uint8_t* lat;  // channels-last [B, H, W, C] latencies; nullptr = A prepared in aq
  int C, H, W, pad, KH, KW, Wo, HoWo, T;
  int foot;            // band bytes (the largest tile footprint, host-computed)
};
constexpr int kTcMaxImg = 128;  // images one M tile can touch (HoWo >= 1)

__global__ void __launch_bounds__(kTcThreads + 128, 1) conv_tc_kernel(const uint8_t* __restrict__ aq,
                                                                 const uint8_t* __restrict__ bq, TcPlan p, int F,
                                                                 int HoWo, int T, uint32_t tmem_cols,
                                                                 uint8_t* __restrict__ lat_out,
                                                                 float* __restrict__ v_out,
                                                                 unsigned long long* __restrict__ part, int nhwc,
                                                                 const TcImpl im) {
  pdl_begin();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = kTcM * kTcKT, b_bytes = uint32_t(p.N) * kTcKT, stage_bytes = a_bytes + b_bytes;
  __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages], done_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int img_off[kTcMaxImg + 1], img_r0[kTcMaxImg];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ksi = int(blockIdx.x % unsigned(p.KS)), tile = int(blockIdx.x / unsigned(p.KS));  // K slices fastest
  const int ch = tile % p.nch, mt = tile / p.nch;  // then feature chunks
  const int kt0 = int(int64_t(ksi) * p.Kt / p.KS), kt1 = int(int64_t(ksi + 1) * p.Kt / p.KS);
  const bool impl = im.lat != nullptr;
  uint8_t* band = smem + size_t(kTcStages) * stage_bytes;
  const int m_first = mt * kTcM, m_last = min(p.M, m_first + kTcM) - 1;
  const int b_first = impl ? m_first / im.HoWo : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), impl ? 9 : 1);  // impl: + one arrival per A-writing warp
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&done_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0 && lane == 0) {
    // ---------------- producer: two bulk copies per stage (impl: B only) ----------------
    const uint8_t* a_src = aq + size_t(mt) * p.Kt * a_bytes;
    const uint8_t* b_src = bq + size_t(ch) * p.Kt * b_bytes;
    for (int kt = kt0; kt < kt1; ++kt) {
      const int s = (kt - kt0) % kTcStages, u = (kt - kt0) / kTcStages;
      if (kt - kt0 >= kTcStages) mbar_wait(smem_u32(&empty_bar[s]), (u - 1) & 1);
      const uint32_t fb = smem_u32(&full_bar[s]);
      mbar_expect_tx(fb, impl ? b_bytes : stage_bytes);
      const uint32_t dst = smem_u32(smem + size_t(s) * stage_bytes);
      if (!impl) bulk_g2s(dst, a_src + size_t(kt) * a_bytes, a_bytes, fb);
      bulk_g2s(dst + a_bytes, b_src + size_t(kt) * b_bytes, b_bytes, fb);
    }
  } else if (impl && warp >= 4) {
    // ---------------- A writers (K8) ----------------
    // stage the tile's binary S[T-1] footprint: per image, its input rows (full width), pixel stride
    // PS = Cp + 16 bytes (16-byte loads of consecutive pixels fall in distinct bank groups); the B bulk
    // copies of the first stages are already in flight
    const int PS = p.Cp + 16, Ho = im.HoWo / im.Wo;
    const int b_last = m_last / im.HoWo, nimg = b_last - b_first + 1;
    const int wt = threadIdx.x - 128;  // 0..255: the 8 writer warps (4..11)
    if (wt == 0) {
      int off = 0;
      for (int b = b_first, i = 0; b <= b_last; ++b, ++i) {
        const int y0 = b == b_first ? (m_first - b * im.HoWo) / im.Wo : 0;
        const int y1 = b == b_last ? (m_last - b * im.HoWo) / im.Wo : Ho - 1;
        const int r0 = max(0, y0 - im.pad), r1 = min(im.H - 1, y1 - im.pad + im.KH - 1);
        img_off[i] = off;
        img_r0[i] = r0;
        off += max(0, r1 - r0 + 1) * im.W * PS;
      }
      img_off[nimg] = off;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    {
      uint4* z = reinterpret_cast<uint4*>(band);
      for (int i = wt; i < img_off[nimg] / 16; i += 256) z[i] = make_uint4(0, 0, 0, 0);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    for (int i = 0; i < nimg; ++i) {  // one warp per input pixel, lanes along its C contiguous channels
      const int npx = (img_off[i + 1] - img_off[i]) / PS;
      const uint8_t* src = im.lat + ((int64_t(b_first + i) * im.H + img_r0[i]) * im.W) * im.C;
      uint8_t* dst = band + img_off[i];
      for (int px = warp - 4; px < npx; px += 8)
        for (int c = lane; c < im.C; c += 32) dst[px * PS + c] = __ldg(src + int64_t(px) * im.C + c) < im.T ? 1 : 0;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    // then row r of every stage's A tile from the band: warps 4-7 the K bytes 0-63, warps 8-11 64-127
    const int r = wt & 127, kh = wt >> 7, m = m_first + r;
    const bool mv = m <= m_last;
    const int b = mv ? m / im.HoWo : b_first, rem = m - b * im.HoWo;
    const int y = mv ? rem / im.Wo : 0, x = mv ? rem - y * im.Wo : 0;
    const uint8_t* bb = band + img_off[b - b_first];
    const int r0 = img_r0[b - b_first], Cp = p.Cp, KK = im.KH * im.KW;
    const uint32_t rofs = uint32_t(r >> 3) * 1024u + uint32_t(r & 7) * 16u;
    // (ky, kx, c0) of the row's first 16-byte column of stage kt0, advanced incrementally
    int k = kt0 * kTcKT + kh * (kTcKT / 2), kyx = k / Cp, c0 = k - kyx * Cp, ky = kyx / im.KW, kx = kyx - ky * im.KW;
    for (int kt = kt0; kt < kt1; ++kt) {
      const int s = (kt - kt0) % kTcStages, u = (kt - kt0) / kTcStages;
      if (kt - kt0 >= kTcStages) mbar_wait(smem_u32(&empty_bar[s]), (u - 1) & 1);
      uint8_t* at = smem + size_t(s) * stage_bytes;
      if (Cp % kTcKT == 0) {  // the stage's 128 K bytes are 128 channels of ONE input pixel
        const int kq = kt * kTcKT + kh * (kTcKT / 2), kq_yx = kq / Cp, cq = kq - kq_yx * Cp, kqy = kq_yx / im.KW, kqx = kq_yx - kqy * im.KW;
        const int iy = y + kqy - im.pad, ix = x + kqx - im.pad;
        const bool ok = mv && kq_yx < KK && iy >= 0 && iy < im.H && ix >= 0 && ix < im.W;
        const uint4* src = reinterpret_cast<const uint4*>(bb + ((iy - r0) * im.W + ix) * (Cp + 16) + cq);
        uint4 v[kTcKT / 32];
#pragma unroll
        for (int k16 = 0; k16 < kTcKT / 32; ++k16) v[k16] = ok ? src[k16] : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k16 = 0; k16 < kTcKT / 32; ++k16) *reinterpret_cast<uint4*>(at + rofs + (kh * 4 + k16) * 128) = v[k16];
      } else {
#pragma unroll
      for (int k16 = kh * 4; k16 < kh * 4 + kTcKT / 32; ++k16) {
        uint4 v = make_uint4(0, 0, 0, 0);
        const int iy = y + ky - im.pad, ix = x + kx - im.pad;
        if (mv && kyx < KK && iy >= 0 && iy < im.H && ix >= 0 && ix < im.W)
          v = *reinterpret_cast<const uint4*>(bb + ((iy - r0) * im.W + ix) * (Cp + 16) + c0);
        *reinterpret_cast<uint4*>(at + rofs + k16 * 128) = v;
        c0 += 16;
        if (c0 == Cp) { c0 = 0; ++kyx; if (++kx == im.KW) { kx = 0; ++ky; } }
      }
#pragma unroll
      for (int k16 = 0; k16 < kTcKT / 32; ++k16) {  // skip the other writer half's 64 K bytes
        c0 += 16;
        if (c0 == Cp) { c0 = 0; ++kyx; if (++kx == im.KW) { kx = 0; ++ky; } }
      }
      }
      fence_proxy_async_smem();  // the generic-proxy stores, visible to the tensor core's async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full_bar[s]));
    }
  }
  if (warp == 0 || (impl && warp >= 4)) {
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (2u << 4)                       // D format: s32
                           | (0u << 7) | (0u << 10)        // A, B: unsigned 8-bit
                           | (uint32_t(p.N >> 3) << 17)    // N
                           | (uint32_t(kTcM >> 4) << 24);  // M = 128
    for (int kt = kt0; kt < kt1; ++kt) {
      const int s = (kt - kt0) % kTcStages, u = (kt - kt0) / kTcStages;
      mbar_wait(smem_u32(&full_bar[s]), u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_base = smem_u32(smem + size_t(s) * stage_bytes);
      const uint32_t b_base = a_base + a_bytes;
#pragma unroll
      for (int ks = 0; ks < kTcKT / 32; ++ks) {  // K = 32 bytes per tcgen05.mma (kind::i8)
        const uint64_t da = umma_desc(a_base + ks * 256, 128, 1024);
        const uint64_t db = umma_desc(b_base + ks * 256, 128, 1024);
        umma_i8(tmem_base, da, db, idesc, ((kt - kt0) | ks) != 0);
      }
      umma_commit(smem_u32(&empty_bar[s]));  // frees the stage once these MMAs have read it
    }
    umma_commit(smem_u32(&done_bar));
  }
  if (warp >= 4 && warp < 8) {
    // ---------------- epilogue: TMEM -> registers -> exact recombination -> (lat, v) ----------------
    mbar_wait(smem_u32(&done_bar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int m = mt * kTcM + row;
    const uint32_t trow = tmem_base + (uint32_t(q * 32) << 16);
    const int b = m / HoWo, rem = m - (m / HoWo) * HoWo;
    for (int g = 0; g < p.Fc / 4; ++g) {
      uint32_t v[16];
      tmem_ld16(trow + uint32_t(g * 16), v);  // warp-collective: every lane participates
      if (m < p.M) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int f = ch * p.Fc + g * 4 + j;
          if (f < F) {
            const int64_t acc = int64_t(v[4 * j]) + (int64_t(v[4 * j + 1]) << 8) + (int64_t(v[4 * j + 2]) << 16) +
                                (int64_t(v[4 * j + 3]) << 24);
            if (part) {  // split-K: exact partial sum of this K slice
              SNN_DCHECK(m < p.M && f < F);
              atomicAdd(part + int64_t(m) * F + f, (unsigned long long)acc);
              continue;
            }
            int64_t o = nhwc ? int64_t(m) * F + f : (int64_t(b) * F + f) * HoWo + rem;
            if (p.fcP) {  // K9: virtual feature f = (position pp, real feature fr) of image m
              const int pp = f / p.fcF, fr = f - pp * p.fcF;
              o = nhwc ? (int64_t(m) * p.fcP + pp) * p.fcF + fr : (int64_t(m) * p.fcF + fr) * p.fcP + pp;
            }
            lat_out[o] = acc > 0 ? uint8_t(T - 1) : kNoSpike;
            if (v_out) v_out[o] = fixed_to_float(acc);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols) : "memory");
  }
}

// split-K finalize: the summed fixed-point potentials -> (lat, v) (Eq. 5).
__global__ void conv_tc_finalize_kernel(const unsigned long long* __restrict__ part, int M, int F, int HoWo, int T,
                                        uint8_t* __restrict__ lat_out, float* __restrict__ v_out, int nhwc,
                                        int fcF, int fcP) {
  pdl_begin();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < int64_t(M) * F;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int m = int(i / F), f = int(i - int64_t(m) * F);
    const int b = m / HoWo, rem = m - b * HoWo;
    const int64_t acc = int64_t(part[i]);
    int64_t o = nhwc ? i : (int64_t(b) * F + f) * HoWo + rem;
    if (fcP) {  // K9 (conv_tc_kernel's epilogue)
      const int pp = f / fcF, fr = f - pp * fcF;
      o = nhwc ? (int64_t(m) * fcP + pp) * fcF + fr : (int64_t(m) * fcF + fr) * fcP + pp;
    }
    lat_out[o] = acc > 0 ? uint8_t(T - 1) : kNoSpike;
    if (v_out) v_out[o] = fixed_to_float(acc);
  }
}

int conv_tc_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH, int KW,
                   int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes, cudaStream_t s,
                   const uint8_t* aq_pre = nullptr, int nhwc = 0, int in_nhwc = 0);

// A operands of B images, one one-image block each (tc_plan(1, ...)), for later snn_conv_fire_prepared.
size_t conv_inf_prepare_bytes(int B, int C, int H, int W, int pad, int F, int KH, int KW) {
  return size_t(B) * tc_plan(1, C, H, W, pad, KH, KW, F, num_sms()).a_bytes;
}

int conv_inf_prepare_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                            void* prep, size_t prep_bytes, cudaStream_t s) {
  const TcPlan p = tc_plan(1, C, H, W, pad, KH, KW, F, num_sms());
  if (prep_bytes < size_t(B) * p.a_bytes)
    return set_error(SNN_EWORKSPACE, "snn_conv_inf_prepare: %zu < %zu bytes", prep_bytes, size_t(B) * p.a_bytes);
  const int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
  const int64_t rows16 = int64_t(p.Mt) * kTcM * (p.Kp / 16);
  const int blocks = int(ceil_div(rows16, 256));
  if (B > 65535) return set_error(SNN_ESHAPE, "snn_conv_inf_prepare: B > 65535");
  launch_k(tc_prep_a_kernel, dim3(blocks, B), dim3(256), 0, s, lat_in, C, H, W, pad, KH, KW, Ho, Wo, T, p,
           static_cast<uint8_t*>(prep), p.a_bytes, 0);
  note_launch();
  return check_launch("snn_conv_inf_prepare");
}

int conv_fire_prepared_launch(const void* prep, int b, int C, int H, int W, int pad, const float* w, int F, int KH,
                              int KW, int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                              cudaStream_t s) {
  const TcPlan p = tc_plan(1, C, H, W, pad, KH, KW, F, num_sms());
  const uint8_t* aq = static_cast<const uint8_t*>(prep) + size_t(b) * p.a_bytes;
  return conv_tc_launch(nullptr, 1, C, H, W, pad, w, F, KH, KW, T, lat_out, v_out, ws, ws_bytes, s, aq);
}

int conv_tc_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH, int KW,
                   int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes, cudaStream_t s,
                   const uint8_t* aq_pre, int nhwc, int in_nhwc) {
  const int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1, R = C * KH * KW;
  TcPlan p = tc_plan(B, C, H, W, pad, KH, KW, F, num_sms());
  // K9: the geometry the A prep and the GEMM see (the fully connected rewrite: one position per image,
  // Ho Wo F features); the B prep and the output index use the real geometry through p.fc*
  int pad_v = pad, KH_v = KH, KW_v = KW, Ho_v = Ho, Wo_v = Wo, F_v = F;
  {
    TcPlan q;
    if (!aq_pre && tc_fc_plan(B, C, H, W, pad, KH, KW, F, num_sms(), &q)) {
      p = q; pad_v = 0; KH_v = H; KW_v = W; Ho_v = Wo_v = 1; F_v = Ho * Wo * F;
    }
  }
  const size_t a_off = 0, b_off = (p.a_bytes + 1023) & ~size_t(1023);
  const size_t part_off = b_off + ((p.b_bytes + 1023) & ~size_t(1023));
  const size_t l_off = (part_off + p.part_bytes + 1023) & ~size_t(1023);
  if (ws_bytes < (p.fcP ? l_off + p.fc_l_bytes : part_off + p.part_bytes))
    return set_error(SNN_EWORKSPACE, "snn_conv_fire(tc): workspace too small");
  unsigned long long* part =
      p.KS > 1 ? reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + part_off) : nullptr;
  if (part && cudaMemsetAsync(part, 0, p.part_bytes, s) != cudaSuccess) return check_launch("snn_conv_fire(tc) memset");
  uint8_t* aq = reinterpret_cast<uint8_t*>(ws) + a_off;
  uint8_t* bq = reinterpret_cast<uint8_t*>(ws) + b_off;
  if (p.fcP) {  // K9: the real limb rows once, then the virtual layer's B as 16-byte pieces of them
    uint8_t* L = reinterpret_cast<uint8_t*>(ws) + l_off;
    int64_t blocks = ceil_div(int64_t(F) * KH * KW * (p.Cp / 16), 256);
    if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
    launch_k(tc_prep_limbs_kernel, dim3(int(blocks)), dim3(256), 0, s, w, F, C, KH * KW, p.Cp, L, error_word_ptr(s));
    note_launch();
    blocks = ceil_div(int64_t(p.nch) * p.Fc * (p.Kp / 16), 256);
    if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
    launch_k(tc_prep_b_fc_kernel, dim3(int(blocks)), dim3(256), 0, s, static_cast<const uint8_t*>(L), F_v, p, bq);
    note_launch();
  } else {
    const int64_t total = int64_t(p.nch) * p.Fc * (p.Kp / 16);
    int64_t blocks = ceil_div(total, 256);
    if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
    launch_k(tc_prep_b16_kernel, dim3(int(blocks)), dim3(256), 0, s, w, F, R, KH * KW, p, bq, error_word_ptr(s));
    note_launch();
  }
  // K8 implicit im2col: channels-last input on the (ky, kx, c) path, every tile's footprint (the input rows
  // of its images' output rows, full width, Cp channels) fits next to the pipeline stages
  TcImpl im{};
  const int smem_stages = kTcStages * (kTcM * kTcKT + p.N * kTcKT) + 1024;
  // Opt-in (SNN_TC_IMPLICIT=1): measured on C2's third layer 0.180 ms against 0.153 ms for the explicit
  // prep + bulk-copy GEMM (8 A-writer warps; 4 warps: 0.216 ms) -- per stage the writers' 16-byte loads
  // and stores add ~19 % shared-memory traffic to the MMA's reads and the bulk copies, and every feature
  // chunk's CTA rebuilds the same A tile, which costs more than the prep kernel's HBM round trip saves.
  if (!aq_pre && !p.fcP && p.hwc && in_nhwc && p.Mt <= 65536 && getenv("SNN_TC_IMPLICIT") && getenv("SNN_TC_IMPLICIT")[0] == '1') {
    const int HoWo = Ho * Wo;
    long foot = 0;
    for (int mt = 0; mt < p.Mt && foot >= 0; ++mt) {
      const int m0 = mt * kTcM, m1 = (m0 + kTcM < p.M ? m0 + kTcM : p.M) - 1;
      if (m1 / HoWo - m0 / HoWo + 1 > kTcMaxImg) { foot = -1; break; }
      long f = 0;
      for (int b = m0 / HoWo; b <= m1 / HoWo; ++b) {
        const int y0 = b == m0 / HoWo ? (m0 - b * HoWo) / Wo : 0, y1 = b == m1 / HoWo ? (m1 - b * HoWo) / Wo : Ho - 1;
        const int r0 = y0 - pad > 0 ? y0 - pad : 0, r1 = y1 - pad + KH - 1 < H - 1 ? y1 - pad + KH - 1 : H - 1;
        f += long(r1 >= r0 ? r1 - r0 + 1 : 0) * W * (p.Cp + 16);
      }
      if (f > foot) foot = f;
    }
    foot = (foot + 15) & ~15L;
    if (foot >= 0 && smem_stages + foot <= 227 * 1024) {
      im.lat = lat_in; im.C = C; im.H = H; im.W = W; im.pad = pad; im.KH = KH; im.KW = KW; im.Wo = Wo;
      im.HoWo = HoWo; im.T = T; im.foot = int(foot);
    }
  }
  if (im.lat) {
  } else if (aq_pre) {  // prepared by snn_conv_inf_prepare
    aq = const_cast<uint8_t*>(aq_pre);
  } else if (p.fcP) {  // K9: the input map itself (binary, channels padded), one row per image
    int64_t blocks = ceil_div(int64_t(p.Mt) * kTcM * (p.Kp / 16), 256);
    if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
    launch_k(tc_prep_a_fc_kernel, dim3(int(blocks)), dim3(256), 0, s, lat_in, C, H * W, T, p, aq, in_nhwc);
    note_launch();
  } else {
    if (p.hwc) {
      launch_k(tc_prep_a_hwc_kernel, dim3(unsigned(int64_t(B) * p.nbands + 1)), dim3(256), p.band_smem, s, lat_in, C, H, W,
               pad_v, KH_v, KW_v, Ho_v, Wo_v, T, p, B, aq, in_nhwc);
    } else if (p.band) {
      launch_k(tc_prep_a_band_kernel, dim3(unsigned(int64_t(B) * p.nbands + 1)), dim3(256), p.band_smem, s, 
          lat_in, C, H, W, pad_v, KH_v, KW_v, Ho_v, Wo_v, T, p, p.RB, p.nbands, B, 1, aq, in_nhwc);
    } else {
      const int64_t rows16 = int64_t(p.Mt) * kTcM * (p.Kp / 16);
      int64_t blocks = ceil_div(rows16, 256);
      if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
      launch_k(tc_prep_a_kernel, dim3(int(blocks)), dim3(256), 0, s, lat_in, C, H, W, pad_v, KH_v, KW_v, Ho_v, Wo_v, T, p,
               aq, size_t(0), in_nhwc);
    }
    note_launch();
  }
  uint32_t cols = 32;
  while (cols < uint32_t(p.N)) cols <<= 1;
  const int smem = smem_stages + im.foot;
  cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_conv_fire(tc): %s", cudaGetErrorString(e));
  if (getenv("SNN_DEBUG_PLAN"))
    fprintf(stderr, "tc plan: Mt %d nch %d KS %d N %d Kt %d hwc %d implicit %d foot %d smem %d fc %d\n", p.Mt, p.nch, p.KS,
            p.N, p.Kt, p.hwc, im.lat != nullptr, im.foot, smem, p.fcP);
  launch_k(conv_tc_kernel, dim3(unsigned(int64_t(p.Mt) * p.nch * p.KS)), dim3(im.lat ? kTcThreads + 128 : kTcThreads), smem,
           s, aq, bq, p, F_v, Ho_v * Wo_v, T, cols, lat_out, v_out, part, nhwc, im);
  note_launch();
  if (part) {
    const int64_t n = int64_t(p.M) * F_v;
    int blocks = int(ceil_div(n, 256));
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    launch_k(conv_tc_finalize_kernel, dim3(blocks), dim3(256), 0, s, part, p.M, F_v, Ho_v * Wo_v, T, lat_out, v_out, nhwc,
             p.fcF, p.fcP);
    note_launch();
  }
  return check_launch("snn_conv_fire(tc)");
}

}  // namespace snn

namespace snn {

__device__ unsigned long long g_rstdp_stamps[4 * 4096];  // timing experiments (SNN_RSTDP_DBG & 8)
extern "C" __attribute__((visibility("default"))) int snn_debug_rstdp_stamps(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_rstdp_stamps, sizeof(unsigned long long) * 4 * (n < 4096 ? n : 4096)) ==
                 cudaSuccess ? 0 : -3;
}

// ------------------------------------------------------------------ f1: theta = +inf R-STDP chain
// The per-image chain of a theta = +inf plastic layer (C4's second layer, Eq. 5, P:191,
// P:258, Eq. 4 / P:161): conv (Eq. 5) -> one winner (k-WTA, k = 1) -> decision vs label -> reward ->
// R-STDP of the winner's feature.  Per image two kernels: the split-K tcgen05 GEMM of the image's
// prepared A operand (snn_conv_inf_prepare) with the resident B limbs, whose epilogue adds exact
// int64 partial sums into part[M][F]; and one tail CTA that reads and clears part, takes the minimum
// key (lat = T - 1 iff P > 0, v = fp32(P), flat index f H W + y W + x: the snn_k_winners order, R13/
// R14), decides (the block decision_map of snn_decide, R24/R25), applies Eq. 4 to the winner's
// weights (the snn_stdp_update arithmetic, R17-R22) and re-quantises only that feature's B limbs.
// No host round trip and no full re-quantisation of the weights per image.
// State shared by the two tail kernels of one image (zeroed by the launcher once; each image leaves it
// clean for the next): the running minimum key, the CTA ticket, and the decided winner and reward.
struct RstdpState {
  unsigned long long best;  // minimum key over the CTAs (~0 = none)
  unsigned int ticket;      // CTAs done with their slice
  int f, y, x;              // winner of the image (f = -1: silent)
  float rw;                 // its reward (+1, -1, 0 = no plasticity)
};

// Eq. 4 on one 16-column group k0 = 16 g16 of the winner f's GEMM columns (post = T - 1, Eq. 5; the
// snn_stdp_update arithmetic, R17-R22): the 16 weights' updates, then the four 16-byte limb rows of that
// core-matrix column (the tc_prep_b16 layout) -- every load issued before any use.  Returns true if a
// new weight left the exact domain.
__device__ __forceinline__ bool rstdp_eq4_group(int g16, int f, int y, int x, float ap, float am, int post,
                                                const uint8_t* __restrict__ lat_img, int C, int H, int W, int KH,
                                                int KW, int pad, float* __restrict__ w, uint8_t* __restrict__ bq,
                                                const TcPlan& p, float lb, float ub, int stabilizer) {
  const int KK = KH * KW, R = C * KK;
  float* wf = w + int64_t(f) * R;
  const int ch = f / p.Fc, fl = f - ch * p.Fc;
  uint8_t* base = bq + size_t(ch) * p.Kt * p.N * kTcKT;
  bool bad = false;
  const int k0 = g16 * 16;
  uint32_t limb[4][4] = {};
  const int kyx = p.hwc ? k0 / p.Cp : 0, c0 = p.hwc ? k0 - kyx * p.Cp : 0;
  int ev[16], pre[16];
  float w0v[16];
  // (c, ky, kx) of column k0 by divisions once, then stepped column by column
  int cc, kyy, kxx;
  if (p.hwc) { cc = c0; kyy = kyx / KW; kxx = kyx - kyy * KW; }
  else { cc = k0 / KK; const int rr = k0 - cc * KK; kyy = rr / KW; kxx = rr - kyy * KW; }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    int e = -1;
    const int c = cc, ky = kyy, kx = kxx;
    if (p.hwc) {  // column k = kyx Cp + c (channels padded to Cp)
      if (c < C) e = c * KK + kyx;
      ++cc;
    } else {      // column k = e = (c KH + ky) KW + kx
      if (k0 + j < R) e = k0 + j;
      if (++kxx == KW) { kxx = 0; if (++kyy == KH) { kyy = 0; ++cc; } }
    }
    ev[j] = e;
    const int yy = y + ky - pad, xx = x + kx - pad;
    const bool inb = e >= 0 && yy >= 0 && yy < H && xx >= 0 && xx < W;
    pre[j] = inb ? int(__ldg(lat_img + (int64_t(c) * H + yy) * W + xx)) : int(kNoSpike);
    w0v[j] = e >= 0 ? wf[e] : 0.0f;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int e = ev[j];
    if (e < 0) continue;
    const float a = (pre[j] != kNoSpike && pre[j] <= post) ? ap : am;
    const float w0 = w0v[j];
    const float dw = stabilizer ? __fmul_rn(__fmul_rn(a, __fsub_rn(w0, lb)), __fsub_rn(ub, w0)) : a;
    float w1 = __fadd_rn(w0, dw);
    if (stabilizer != 2) {
      w1 = w1 < lb ? lb : w1;
      w1 = w1 > ub ? ub : w1;
    }
    wf[e] = w1;
    const float sx = w1 * 2147483648.0f;
    uint32_t q = 0;
    if (!(w1 >= 0.0f && w1 <= 1.0f) || sx != truncf(sx)) bad = true;
    else q = uint32_t(sx);
#pragma unroll
    for (int l = 0; l < 4; ++l) limb[l][j >> 2] |= ((q >> (8 * l)) & 0xFFu) << (8 * (j & 3));
  }
#pragma unroll
  for (int l = 0; l < 4; ++l)
    *reinterpret_cast<uint4*>(base + tc_off(4 * fl + l, k0, p.N, p.Kt)) =
        make_uint4(limb[l][0], limb[l][1], limb[l][2], limb[l][3]);
  return bad;
}

// Tail 1: CTAs share the M x F partial sums (each reads and clears its slice and offers its minimum key,
// lat = T - 1 and v = fp32(P) descending, then flat index f H W + y W + x ascending: the snn_k_winners
// order, R13/R14); the last CTA to finish decides (snn_decide's block decision_map, R24/R25) and
// writes the image's outputs and the winner for tail 2.
__global__ void __launch_bounds__(256) rstdp_inf_tail1_kernel(
    unsigned long long* __restrict__ part, int M, int Wo, int F, int T, const int32_t* __restrict__ labels, int b,
    int n_classes, RstdpState* st, int32_t* __restrict__ winners, int32_t* __restrict__ count,
    int32_t* __restrict__ decision, float* __restrict__ reward, int dbg) {
  pdl_begin();
  if ((dbg & 8) && blockIdx.x == 0 && threadIdx.x == 0 && b < 4096) g_rstdp_stamps[4 * b + 0] = globaltimer_ns();
  __shared__ uint64_t wmin[8];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int MF = M * F;
  const int per = int(ceil_div(MF, gridDim.x));
  const int i0 = blockIdx.x * per, i1 = min(MF, i0 + per);
  uint64_t best = ~uint64_t(0);
  for (int i = i0 + tid; i < i1; i += blockDim.x) {
    const int64_t acc = int64_t(part[i]);
    part[i] = 0ull;
    if (acc > 0) {
      const int m = i / F, f = i - m * F;
      const uint64_t key = wta_key(uint8_t(T - 1), fixed_to_float(acc), uint32_t(f * M + m));
      best = key < best ? key : best;
    }
  }
  best = warp_min_u64(best);
  if (lane == 0) wmin[warp] = best;
  __syncthreads();
  if (tid == 0) {
    uint64_t x = ~uint64_t(0);
    for (int w = 0; w < int(blockDim.x >> 5); ++w) x = wmin[w] < x ? wmin[w] : x;
    if (x != ~uint64_t(0)) atomicMin(&st->best, (unsigned long long)x);
    __threadfence();
    s_last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  {
    __threadfence();
    const uint64_t k = atomicExch(&st->best, ~0ull);  // read and reset for the next image
    st->ticket = 0;
    int f = -1, y = -1, x = -1, d = -1;
    float rw = 0.0f;
    if (k != ~0ull) {
      const int idx = int(k & 0xFFFFFFu);
      f = idx / M;
      const int pos = idx - f * M;
      y = pos / Wo;
      x = pos - y * Wo;
      d = f / (F / n_classes);
      if (labels) rw = (d == labels[b]) ? 1.0f : -1.0f;
    }
    winners[0] = f; winners[1] = y; winners[2] = x;
    count[0] = f >= 0 ? 1 : 0;
    if (decision) decision[0] = d;
    if (reward) reward[0] = rw;
    st->f = f; st->y = y; st->x = x; st->rw = rw;
    if ((dbg & 8) && b < 4096) g_rstdp_stamps[4 * b + 1] = globaltimer_ns();
  }
}

// Tail 2: Eq. 4 on the winner's weights and the re-quantisation of only that feature's B limbs, one
// thread per 16 consecutive GEMM columns (rstdp_eq4_group).  Spread over several CTAs: measured on C4,
// 8.5 us as its own kernel against 11.8 us inside tail 1's last CTA.
__global__ void __launch_bounds__(128) rstdp_inf_tail2_kernel(
    const RstdpState* __restrict__ st, int T, const uint8_t* __restrict__ lat_img, int C, int H, int W, int KH,
    int KW, int pad, float* __restrict__ w, uint8_t* __restrict__ bq, TcPlan p, float a_plus, float a_minus,
    float lb, float ub, int stabilizer, int* err, int b, int dbg) {
  pdl_begin();
  const int f = st->f;
  const float rw = st->rw;
  if (f < 0 || rw == 0.0f) return;
  const float ap = rw > 0.0f ? a_plus : -a_plus, am = rw > 0.0f ? a_minus : -a_minus;
  const int nk16 = p.K / 16 + (p.K % 16 ? 1 : 0);
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (g < nk16) bad = rstdp_eq4_group(g, f, st->y, st->x, ap, am, T - 1, lat_img, C, H, W, KH, KW, pad, w, bq, p, lb,
                                      ub, stabilizer);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_error(err, kErrInexact);
  if ((dbg & 8) && blockIdx.x == 0 && threadIdx.x == 0 && b < 4096) g_rstdp_stamps[4 * b + 2] = globaltimer_ns();
}

// ------------------------------------------------------------- f1, one launch: the persistent chain
// The whole N-image chain as ONE cooperative kernel (one CTA per (M tile, feature chunk, K slice) of the
// split-K GEMM, all co-resident; TMEM allocated once).  Per image three phases separated by grid
// barriers: A) the CTA's K slice of the image's GEMM (bulk-copy + mbarrier pipeline whose stage/phase
// counters run on across images), exact int64 partial sums added into part[M][F]; B) every CTA reads and
// clears a slice of part, takes its minimum key (the snn_k_winners order) and folds it into the image's
// best key (double-buffered: best[i & 1]); C) every CTA decodes the winner and decision, and applies
// Eq. 4 to its share of the winner's 16-column groups (w and the B limbs, rstdp_eq4_group).
// Bit-identical to the per-image kernels; no launch or host round trip per image.
struct PersistArgs {
  const uint8_t* prep;            // snn_conv_inf_prepare A blocks
  int b0, N;
  const uint8_t* lat_in;          // [N][C][H][W]
  int C, H, W, pad, KH, KW, F, T, Ho, Wo;
  float* w;
  uint8_t* bq;
  unsigned long long* part;       // [M][F] (zero on entry, left zero)
  unsigned long long* best;       // [2] (~0 on entry)
  unsigned* bar;                  // [2] grid barrier (zero on entry)
  const int32_t* labels;
  int n_classes;
  float a_plus, a_minus, lb, ub;
  int stabilizer;
  int32_t *winners, *count, *decision;
  float* reward;
  int* err;
  TcPlan p;
  uint32_t tmem_cols;
};

__device__ __forceinline__ void tc_grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = gen;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(&bar[1], g + 1);
    } else {
      const uint64_t t0 = globaltimer_ns();
      for (;;) {
        unsigned cur;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
        if (cur != g) break;
        watchdog(t0);
      }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

__global__ void __launch_bounds__(kTcThreads, 1) rstdp_inf_persist_kernel(const PersistArgs q) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TcPlan& p = q.p;
  const uint32_t a_bytes = kTcM * kTcKT, b_bytes = uint32_t(p.N) * kTcKT, stage_bytes = a_bytes + b_bytes;
  __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages], done_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint64_t wmin[kTcThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ksi = int(blockIdx.x % unsigned(p.KS)), tile = int(blockIdx.x / unsigned(p.KS));
  const int ch = tile % p.nch, mt = tile / p.nch;
  const int kt0 = int(int64_t(ksi) * p.Kt / p.KS), kt1 = int(int64_t(ksi + 1) * p.Kt / p.KS);
  const int F = q.F, M = p.M, MF = M * F;
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&done_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(q.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  unsigned gen = 0;
  int it0 = 0;  // pipeline stages consumed before this image (counters run on across images)
  const int nk = kt1 - kt0;
  const int post = q.T - 1;
  const int nk16 = p.K / 16 + (p.K % 16 ? 1 : 0);
  const int64_t CHW = int64_t(q.C) * q.H * q.W;
  for (int i = 0; i < q.N; ++i) {
    // ---------------- A: this CTA's K slice of image i's GEMM ----------------
    const uint8_t* aq = q.prep + size_t(q.b0 + i) * p.a_bytes;
    if (warp == 0 && lane == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");  // B limbs written by phase C (generic proxy)
      const uint8_t* a_src = aq + size_t(mt) * p.Kt * a_bytes;
      const uint8_t* b_src = q.bq + size_t(ch) * p.Kt * b_bytes;
      for (int kt = kt0; kt < kt1; ++kt) {
        const int c = it0 + (kt - kt0), s = c % kTcStages, u = c / kTcStages;
        if (c >= kTcStages) mbar_wait(smem_u32(&empty_bar[s]), (u - 1) & 1);
        const uint32_t fb = smem_u32(&full_bar[s]);
        mbar_expect_tx(fb, stage_bytes);
        const uint32_t dst = smem_u32(smem + size_t(s) * stage_bytes);
        bulk_g2s(dst, a_src + size_t(kt) * a_bytes, a_bytes, fb);
        bulk_g2s(dst + a_bytes, b_src + size_t(kt) * b_bytes, b_bytes, fb);
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t idesc = (2u << 4) | (0u << 7) | (0u << 10) | (uint32_t(p.N >> 3) << 17) | (uint32_t(kTcM >> 4) << 24);
      tc_fence_after();
      for (int kt = kt0; kt < kt1; ++kt) {
        const int c = it0 + (kt - kt0), s = c % kTcStages, u = c / kTcStages;
        mbar_wait(smem_u32(&full_bar[s]), u & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(smem + size_t(s) * stage_bytes);
        const uint32_t b_base = a_base + a_bytes;
#pragma unroll
        for (int ks = 0; ks < kTcKT / 32; ++ks) {
          const uint64_t da = umma_desc(a_base + ks * 256, 128, 1024);
          const uint64_t db = umma_desc(b_base + ks * 256, 128, 1024);
          umma_i8(tmem_base, da, db, idesc, ((kt - kt0) | ks) != 0);
        }
        umma_commit(smem_u32(&empty_bar[s]));
      }
      umma_commit(smem_u32(&done_bar));
    } else if (warp >= 4) {
      mbar_wait(smem_u32(&done_bar), uint32_t(i & 1));
      tc_fence_after();
      const int qd = warp & 3;
      const int row = qd * 32 + lane;
      const int m = mt * kTcM + row;
      const uint32_t trow = tmem_base + (uint32_t(qd * 32) << 16);
      for (int gq = 0; gq < p.Fc / 4; ++gq) {
        uint32_t v[16];
        tmem_ld16(trow + uint32_t(gq * 16), v);
        if (m < M) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int f = ch * p.Fc + gq * 4 + j;
            if (f < F) {
              const int64_t acc = int64_t(v[4 * j]) + (int64_t(v[4 * j + 1]) << 8) + (int64_t(v[4 * j + 2]) << 16) +
                                  (int64_t(v[4 * j + 3]) << 24);
              atomicAdd(q.part + int64_t(m) * F + f, (unsigned long long)acc);
            }
          }
        }
      }
    }
    it0 += nk;
    tc_fence_before();
    tc_grid_barrier(q.bar, gen);
    tc_fence_after();
    // ---------------- B: winner key (lat = T - 1 iff P > 0, v = fp32(P) desc, flat index asc) ----------------
    {
      const int per = int(ceil_div(MF, int(gridDim.x)));
      const int i0 = int(blockIdx.x) * per, i1 = min(MF, i0 + per);
      uint64_t bk = ~uint64_t(0);
      for (int e = i0 + tid; e < i1; e += blockDim.x) {
        const int64_t acc = int64_t(q.part[e]);
        q.part[e] = 0ull;
        if (acc > 0) {
          const int m = e / F, f = e - m * F;
          const uint64_t key = wta_key(uint8_t(q.T - 1), fixed_to_float(acc), uint32_t(f * M + m));
          bk = key < bk ? key : bk;
        }
      }
      bk = warp_min_u64(bk);
      if (lane == 0) wmin[warp] = bk;
      __syncthreads();
      if (tid == 0) {
        uint64_t x = ~uint64_t(0);
        for (int w = 0; w < kTcThreads / 32; ++w) x = wmin[w] < x ? wmin[w] : x;
        if (x != ~uint64_t(0)) atomicMin(&q.best[i & 1], (unsigned long long)x);
      }
    }
    tc_grid_barrier(q.bar, gen);
    // ---------------- C: decision and Eq. 4 on the winner (post = T - 1) ----------------
    {
      unsigned long long kb;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(kb) : "l"(q.best + (i & 1)) : "memory");
      int f = -1, y = -1, x = -1, d = -1;
      float rw = 0.0f;
      if (kb != ~0ull) {
        const int idx = int(kb & 0xFFFFFFu);
        f = idx / M;
        const int pos = idx - f * M;
        y = pos / q.Wo;
        x = pos - y * q.Wo;
        d = f / (F / q.n_classes);
        if (q.labels) rw = (d == q.labels[i]) ? 1.0f : -1.0f;
      }
      if (blockIdx.x == 0 && tid == 0) {
        q.winners[3 * i] = f; q.winners[3 * i + 1] = y; q.winners[3 * i + 2] = x;
        q.count[i] = f >= 0 ? 1 : 0;
        if (q.decision) q.decision[i] = d;
        if (q.reward) q.reward[i] = rw;
        q.best[(i + 1) & 1] = ~0ull;  // the next image's slot (last read before the previous barrier)
      }
      if (f >= 0 && rw != 0.0f) {
        const float ap = rw > 0.0f ? q.a_plus : -q.a_plus, am = rw > 0.0f ? q.a_minus : -q.a_minus;
        const uint8_t* lat_img = q.lat_in + int64_t(i) * CHW;
        bool bad = false;
        for (int g16 = int(blockIdx.x) * blockDim.x + tid; g16 < nk16; g16 += gridDim.x * blockDim.x)
          bad |= rstdp_eq4_group(g16, f, y, x, ap, am, post, lat_img, q.C, q.H, q.W, q.KH, q.KW, q.pad, q.w, q.bq, p,
                                 q.lb, q.ub, q.stabilizer);
        if (__any_sync(0xffffffffu, bad) && lane == 0) flag_error(q.err, kErrInexact);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the limbs are read by the next bulk copies
      }
    }
    tc_grid_barrier(q.bar, gen);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(q.tmem_cols) : "memory");
  }
}

size_t rstdp_inf_workspace(int C, int H, int W, int pad, int F, int KH, int KW) {
  const TcPlan p = tc_plan(1, C, H, W, pad, KH, KW, F, num_sms());
  return ((p.b_bytes + 1023) & ~size_t(1023)) + ((size_t(p.M) * F * sizeof(unsigned long long) + 255) & ~size_t(255)) +
         256 + 256 + 1024;  // + the persistent kernel's best keys and grid barrier
}

int rstdp_inf_sequence_launch(const void* prep, int b0, int N, int C, int H, int W, int pad, const uint8_t* lat_in,
                              float* w, int F, int KH, int KW, int T, const int32_t* labels, int n_classes,
                              float a_plus, float a_minus, float lb, float ub, int stabilizer, int32_t* winners,
                              int32_t* count, int32_t* decision, float* reward, void* ws, size_t ws_bytes,
                              cudaStream_t s) {
  TcPlan p = tc_plan(1, C, H, W, pad, KH, KW, F, num_sms());
  if (ws_bytes < rstdp_inf_workspace(C, H, W, pad, F, KH, KW))
    return set_error(SNN_EWORKSPACE, "snn_rstdp_inf_sequence: workspace too small");
  const int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1, R = C * KH * KW;
  uint8_t* bq = reinterpret_cast<uint8_t*>(ws);
  unsigned long long* part =
      reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + ((p.b_bytes + 1023) & ~size_t(1023)));
  int* err = error_word_ptr(s);
  {  // the B limbs of the initial weights (afterwards only the winner's feature is re-quantised)
    const int64_t total = int64_t(p.nch) * p.Fc * (p.Kp / 16);
    int64_t blocks = ceil_div(total, 256);
    if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
    launch_k(tc_prep_b16_kernel, dim3(int(blocks)), dim3(256), 0, s, w, F, R, KH * KW, p, bq, err);
    note_launch();
  }
  RstdpState* stp = reinterpret_cast<RstdpState*>(reinterpret_cast<uint8_t*>(part) +
                                                   ((size_t(p.M) * F * sizeof(unsigned long long) + 255) & ~size_t(255)));
  if (cudaMemsetAsync(part, 0, size_t(p.M) * F * sizeof(unsigned long long), s) != cudaSuccess ||
      cudaMemsetAsync(stp, 0xFF, sizeof(unsigned long long), s) != cudaSuccess ||
      cudaMemsetAsync(&stp->ticket, 0, sizeof(unsigned int), s) != cudaSuccess)
    return check_launch("snn_rstdp_inf_sequence memset");
  uint32_t cols = 32;
  while (cols < uint32_t(p.N)) cols <<= 1;
  const int smem = kTcStages * (kTcM * kTcKT + p.N * kTcKT) + 1024;
  cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_rstdp_inf_sequence: %s", cudaGetErrorString(e));
  const int64_t CHW = int64_t(C) * H * W;
  const int dbg = getenv("SNN_RSTDP_DBG") ? atoi(getenv("SNN_RSTDP_DBG")) : 0;  // timing experiments only
  {  // one persistent cooperative kernel for all N images when its CTAs fit the GPU -- opt-in
     // (SNN_RSTDP_PERSIST=1): measured on C4 at 26.6 us per image against 20.0 us for the per-image kernels
     // below (three software grid barriers per image cost more than two PDL-chained kernel boundaries)
    const int grid = p.Mt * p.nch * p.KS;
    int occ = 0;
    cudaFuncSetAttribute(rstdp_inf_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rstdp_inf_persist_kernel, kTcThreads, smem);
    const char* pe = getenv("SNN_RSTDP_PERSIST");
    if (N > 0 && pe && pe[0] == '1' && occ >= 1 && grid <= occ * num_sms()) {
      unsigned long long* best = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(stp) + 256);
      unsigned* bar = reinterpret_cast<unsigned*>(best + 2);
      if (cudaMemsetAsync(best, 0xFF, 2 * sizeof(unsigned long long), s) != cudaSuccess ||
          cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess)
        return check_launch("snn_rstdp_inf_sequence memset");
      PersistArgs q;
      q.prep = static_cast<const uint8_t*>(prep); q.b0 = b0; q.N = N; q.lat_in = lat_in;
      q.C = C; q.H = H; q.W = W; q.pad = pad; q.KH = KH; q.KW = KW; q.F = F; q.T = T; q.Ho = Ho; q.Wo = Wo;
      q.w = w; q.bq = bq; q.part = part; q.best = best; q.bar = bar; q.labels = labels; q.n_classes = n_classes;
      q.a_plus = a_plus; q.a_minus = a_minus; q.lb = lb; q.ub = ub; q.stabilizer = stabilizer;
      q.winners = winners; q.count = count; q.decision = decision; q.reward = reward; q.err = err; q.p = p;
      q.tmem_cols = cols;
      void* args[] = {&q};
      e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(rstdp_inf_persist_kernel), dim3(grid),
                                      dim3(kTcThreads), args, size_t(smem), s);
      if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_rstdp_inf_sequence: %s", cudaGetErrorString(e));
      note_launch();
      return check_launch("snn_rstdp_inf_sequence");
    }
  }
  const int MF = p.M * F;
  const int t1 = int(ceil_div(MF, 1024)) < num_sms() ? int(ceil_div(MF, 1024)) : num_sms();  // ~1K neurons per CTA
  const int nk16 = p.K / 16 + (p.K % 16 ? 1 : 0);
  for (int i = 0; i < N; ++i) {
    const uint8_t* aq = static_cast<const uint8_t*>(prep) + size_t(b0 + i) * p.a_bytes;
    if (!(dbg & 2)) launch_k(conv_tc_kernel, dim3(unsigned(int64_t(p.Mt) * p.nch * p.KS)), dim3(kTcThreads), smem, s, aq,
             (const uint8_t*)bq, p, F, Ho * Wo, T, cols, (uint8_t*)nullptr, (float*)nullptr, part, 0, TcImpl{});
    launch_k(rstdp_inf_tail1_kernel, dim3(t1 > 0 ? t1 : 1), dim3(256), 0, s, part, Ho * Wo, Wo, F, T, labels, i,
             n_classes, stp, winners + 3 * i, count + i, decision ? decision + i : nullptr,
             reward ? reward + i : nullptr, dbg);
    launch_k(rstdp_inf_tail2_kernel, dim3(int(ceil_div(nk16, 128))), dim3(128), 0, s, (const RstdpState*)stp, T,
             lat_in + int64_t(i) * CHW, C, H, W, KH, KW, pad, w, bq, p, a_plus, a_minus, lb, ub, stabilizer, err, i,
             dbg);
    note_launch(3);
  }
  return check_launch("snn_rstdp_inf_sequence");
}

}  // namespace snn
