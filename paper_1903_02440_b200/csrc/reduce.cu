// reduce.cu -- a4 pooling, a5 pointwise inhibition, a6 k-WTA, R-STDP decision.
// All of them order candidates by the packed 64-bit key (lat asc, v desc, flat index asc), so a
// single unsigned min gives the paper's "earliest spike, then maximum potential" rule (P:117, P:126,
// P:128) with the DESIGN.md R14 tie-break.  Pooling and inhibition are HBM-bound elementwise
// reductions (coalesced across the innermost spatial index); k-WTA runs one CTA per image over a
// per-position best-key map.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace snn {

// ------------------------------------------------------------------------------------- a4 pool
// Earliest spike in the window; the max v among the window entries that spiked at that time
// (per-time-step max-pooling of the thresholded potentials read at the pooled spike, R12).
// IDX = uint32_t when the output count fits 32 bits (the index arithmetic is then 32-bit: a 64-bit
// division per output made this HBM-light kernel instruction-bound), int64_t otherwise.
template <class IDX>
__global__ void __launch_bounds__(256) pool_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                   int64_t BF, int H, int W, int PH, int PW, int SH, int SW,
                                                   int DH, int DW, int Ho, int Wo, int vfinal,
                                                   uint8_t* __restrict__ lat_out, float* __restrict__ v_out) {
  pdl_begin();
  const IDX total = IDX(BF) * IDX(Ho) * IDX(Wo);
  const IDX HoWo = IDX(Ho) * IDX(Wo), HW = IDX(H) * IDX(W);
  for (IDX o = IDX(blockIdx.x) * IDX(blockDim.x) + threadIdx.x; o < total; o += IDX(gridDim.x) * blockDim.x) {
    const IDX bf = o / HoWo;
    const int rem = int(o - bf * HoWo);
    const int oy = rem / Wo, ox = rem - oy * Wo;
    const uint8_t* l = lat + bf * HW;
    const float* vv = v ? v + bf * HW : nullptr;
    int best = kNoSpike;
    float bv = 0.0f;
    const int y0 = oy * SH - DH, x0 = ox * SW - DW;
    for (int py = 0; py < PH; ++py) {
      const int yy = y0 + py;
      if (yy < 0 || yy >= H) continue;
      for (int px = 0; px < PW; ++px) {
        const int xx = x0 + px;
        if (xx < 0 || xx >= W) continue;
        const int li = l[yy * W + xx];
        if (li == kNoSpike || (li > best && !vfinal)) continue;
        const float vi = vv ? vv[yy * W + xx] : 0.0f;
        if (vfinal) {  // SNN_POOL_VFINAL: max over every spiking entry (the pooled potentials at T - 1)
          if (best == kNoSpike || vi > bv) bv = vi;
          if (li < best) best = li;
        } else if (li < best) { best = li; bv = vi; }
        else if (vi > bv) bv = vi;
      }
    }
    lat_out[o] = uint8_t(best);
    if (v_out) v_out[o] = best == kNoSpike ? 0.0f : bv;
  }
}

// 2 x 2 windows, stride 2, no padding, with potentials (C5's pool): one thread per pair of adjacent
// outputs, each input row read as one 4-byte latency word and one 16-byte potential vector
// (consecutive threads on consecutive column pairs: coalesced).  Requires W % 4 == 0.
__device__ __forceinline__ void pool4(uint32_t l0, uint32_t l1, uint32_t l2, uint32_t l3, float v0, float v1,
                                      float v2, float v3, int vfinal, uint32_t& lo, float& vo) {
  const uint32_t la[4] = {l0, l1, l2, l3};
  const float va[4] = {v0, v1, v2, v3};
  uint32_t best = kNoSpike;
#pragma unroll
  for (int j = 0; j < 4; ++j) best = la[j] < best ? la[j] : best;
  float bv = 0.0f;
  bool have = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool take = la[j] != kNoSpike && (vfinal || la[j] == best);
    if (take && (!have || va[j] > bv)) { bv = va[j]; have = true; }
  }
  lo = best;
  vo = best == kNoSpike ? 0.0f : bv;
}

__global__ void __launch_bounds__(256) pool2x2_v_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                        uint32_t pairs, int H, int W, int Ho, int Wo, int vfinal,
                                                        uint8_t* __restrict__ lat_out, float* __restrict__ v_out) {
  pdl_begin();
  const uint32_t Wo2 = uint32_t(Wo) >> 1, per_plane = uint32_t(Ho) * Wo2;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < pairs; q += gridDim.x * blockDim.x) {
    const uint32_t bf = q / per_plane, rem = q - bf * per_plane, oy = rem / Wo2, ox2 = rem - oy * Wo2;
    const uint32_t i0 = bf * uint32_t(H) * W + 2 * oy * W + 4 * ox2;
    const uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(lat + i0));
    const uint32_t c = __ldg(reinterpret_cast<const uint32_t*>(lat + i0 + W));
    const float4 va = __ldg(reinterpret_cast<const float4*>(v + i0));
    const float4 vc = __ldg(reinterpret_cast<const float4*>(v + i0 + W));
    uint32_t l0, l1;
    float o0, o1;
    pool4(a & 0xFF, (a >> 8) & 0xFF, c & 0xFF, (c >> 8) & 0xFF, va.x, va.y, vc.x, vc.y, vfinal, l0, o0);
    pool4((a >> 16) & 0xFF, a >> 24, (c >> 16) & 0xFF, c >> 24, va.z, va.w, vc.z, vc.w, vfinal, l1, o1);
    const uint32_t o = bf * per_plane * 2 + oy * uint32_t(Wo) + 2 * ox2;
    *reinterpret_cast<uint16_t*>(lat_out + o) = uint16_t(l0 | (l1 << 8));
    *reinterpret_cast<float2*>(v_out + o) = make_float2(o0, o1);
  }
}

// 2 x 2 / stride 2, latencies only, W % 4 == 0 (C2's first pool): one thread per 4-byte word of a
// row pair, the window minima by byte-wise SIMD (__vminu4), two outputs per 16-bit store; consecutive
// threads on consecutive words (coalesced).
__global__ void __launch_bounds__(256) pool2x2_lat_kernel(const uint8_t* __restrict__ lat, uint32_t words, int H,
                                                          int W, int Ho, uint8_t* __restrict__ lat_out) {
  pdl_begin();
  const uint32_t wpr = uint32_t(W) >> 2;  // words per input row
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < words; q += gridDim.x * blockDim.x) {
    const uint32_t row = q / wpr, w = q - row * wpr;  // row = bf * Ho + oy
    const uint32_t bf = row / uint32_t(Ho), oy = row - bf * uint32_t(Ho);
    const uint8_t* in = lat + (size_t(bf) * H + 2 * oy) * W + 4 * w;
    const uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(in));
    const uint32_t c = __ldg(reinterpret_cast<const uint32_t*>(in + W));
    const uint32_t m = __vminu4(a, c);
    const uint32_t p = __vminu4(m, m >> 8);  // bytes 0 and 2: the two windows' minima
    *reinterpret_cast<uint16_t*>(lat_out + size_t(row) * (W >> 1) + 2 * w) = uint16_t((p & 0xFFu) | ((p >> 8) & 0xFF00u));
  }
}

// Latency-only pooling (no v): one thread per output ROW of one plane walks its Wo windows left to
// right -- no per-output index arithmetic, every input byte of a stride = window layer loaded once
// (through L1), consecutive threads on consecutive rows.
__global__ void __launch_bounds__(256) pool_rows_kernel(const uint8_t* __restrict__ lat, uint32_t rows, int H, int W,
                                                        int PH, int PW, int SH, int SW, int DH, int DW, int Ho,
                                                        int Wo, uint8_t* __restrict__ lat_out) {
  pdl_begin();
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const uint32_t bf = r / uint32_t(Ho);
    const int oy = int(r - bf * uint32_t(Ho));
    const uint8_t* l = lat + size_t(bf) * H * W;
    uint8_t* out = lat_out + size_t(r) * Wo;
    const int y0 = oy * SH - DH;
    const int ya = y0 < 0 ? 0 : y0, yb = (y0 + PH < H ? y0 + PH : H);
    for (int ox = 0; ox < Wo; ++ox) {
      const int x0 = ox * SW - DW;
      const int xa = x0 < 0 ? 0 : x0, xb = (x0 + PW < W ? x0 + PW : W);
      unsigned best = kNoSpike;
      for (int yy = ya; yy < yb; ++yy)
        for (int xx = xa; xx < xb; ++xx) {
          const unsigned li = __ldg(l + yy * W + xx);
          best = li < best ? li : best;
        }
      out[ox] = uint8_t(best);
    }
  }
}

// Channels-last input (lat, v [B, H, W, F], the SNN_CONV_OUT_NHWC output of snn_conv_fire_ex).
// Window rule as pool_kernel (R10-R12; EQ3's truncated windows: entries past the input never spike),
// evaluated branch-free so a thread's window loads are all in flight together.
template <int VEC>
__device__ __forceinline__ void pool_window_nhwc(const uint8_t* limg, const float* vimg, int F, int H, int W, int PH,
                                                 int PW, int SH, int SW, int DH, int DW, int oy, int ox, int f,
                                                 int vfinal, unsigned (&best)[VEC], float (&bv)[VEC]) {
#pragma unroll
  for (int u = 0; u < VEC; ++u) { best[u] = kNoSpike; bv[u] = 0.0f; }
  const int y0 = oy * SH - DH, x0 = ox * SW - DW;
  const int ya = y0 < 0 ? 0 : y0, yb = (y0 + PH < H ? y0 + PH : H);
  const int xa = x0 < 0 ? 0 : x0, xb = (x0 + PW < W ? x0 + PW : W);
  for (int yy = ya; yy < yb; ++yy) {
    uint32_t i = (uint32_t(yy) * W + xa) * F + f;
#pragma unroll 4
    for (int xx = xa; xx < xb; ++xx, i += F) {
      unsigned lv[VEC];
      float vv[VEC];
      if constexpr (VEC == 4) {
        const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(limg + i));
        lv[0] = q & 0xFF; lv[1] = (q >> 8) & 0xFF; lv[2] = (q >> 16) & 0xFF; lv[3] = q >> 24;
        if (vimg) {
          const float4 w4 = __ldg(reinterpret_cast<const float4*>(vimg + i));
          vv[0] = w4.x; vv[1] = w4.y; vv[2] = w4.z; vv[3] = w4.w;
        } else {
          vv[0] = vv[1] = vv[2] = vv[3] = 0.0f;
        }
      } else {
        lv[0] = __ldg(limg + i);
        vv[0] = vimg ? __ldg(vimg + i) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < VEC; ++u) {
        const unsigned li = lv[u];
        const bool sp = li != kNoSpike;
        if (vfinal) {  // SNN_POOL_VFINAL: max over every spiking entry
          const bool tv = sp && (best[u] == kNoSpike || vv[u] > bv[u]);
          bv[u] = tv ? vv[u] : bv[u];
          best[u] = (sp && li < best[u]) ? li : best[u];
        } else {       // earliest spike, then the max potential among the entries at that time
          const bool tk = sp && (li < best[u] || (li == best[u] && vv[u] > bv[u]));
          bv[u] = tk ? vv[u] : bv[u];
          best[u] = tk ? li : best[u];
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < VEC; ++u) bv[u] = best[u] == kNoSpike ? 0.0f : bv[u];
}

// -> planar output [B, F, Ho, Wo].  CTA = (32 output columns, FT <= 32 * VEC features) of one output
// row of one image.  Pass 1: the tile's (column, VEC-feature slot) items over the CTA's threads,
// slots fastest (coalesced channels-last reads; a narrow layer -- C4's F = 20 -- still fills the
// warps); the results transpose through shared memory; pass 2: warps take features, lanes columns
// (coalesced planar rows).  blockIdx.x = column tile + ntx * feature chunk, y = output row, z = image.
template <int VEC>
__global__ void __launch_bounds__(256) pool_nhwc_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                        int F, int H, int W, int PH, int PW, int SH, int SW, int DH,
                                                        int DW, int Ho, int Wo, int ntx, int FT, int vfinal,
                                                        uint8_t* __restrict__ lat_out, float* __restrict__ v_out) {
  pdl_begin();
  constexpr int FTM = 32 * VEC;                       // the largest feature tile
  __shared__ __align__(16) uint8_t s_lat[32 * (FTM + 4)];   // [column][feature], row stride FT + 4
  __shared__ float s_v[32 * (FTM + 1)];                     // [column][feature], row stride FT + 1
  const int LS = FT + 4, VS = FT + 1, FV = FT / VEC;
  const int xt = blockIdx.x % ntx, fc = blockIdx.x / ntx, oy = blockIdx.y, b = blockIdx.z;
  const uint8_t* limg = lat + int64_t(b) * H * W * F;
  const float* vimg = v ? v + int64_t(b) * H * W * F : nullptr;
  for (int it = threadIdx.x; it < 32 * FV; it += blockDim.x) {
    const int p = FV == 32 ? (it >> 5) : it / FV, sl = it - p * FV;  // (a full tile: shifts)
    const int ox = xt * 32 + p, f = fc * FT + sl * VEC;
    unsigned best[VEC];
    float bv[VEC];
    if (ox < Wo && f < F) {
      pool_window_nhwc<VEC>(limg, vimg, F, H, W, PH, PW, SH, SW, DH, DW, oy, ox, f, vfinal, best, bv);
    } else {
#pragma unroll
      for (int u = 0; u < VEC; ++u) { best[u] = kNoSpike; bv[u] = 0.0f; }
    }
    if constexpr (VEC == 4)
      *reinterpret_cast<uint32_t*>(s_lat + p * LS + sl * 4) = best[0] | (best[1] << 8) | (best[2] << 16) | (best[3] << 24);
    else
      s_lat[p * LS + sl] = uint8_t(best[0]);
#pragma unroll
    for (int u = 0; u < VEC; ++u) s_v[p * VS + sl * VEC + u] = bv[u];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ox = xt * 32 + lane;
  if (ox >= Wo) return;
  for (int fl = warp; fl < FT; fl += 8) {
    const int ff = fc * FT + fl;
    if (ff >= F) break;
    const int64_t o = ((int64_t(b) * F + ff) * Ho + oy) * Wo + ox;
    lat_out[o] = s_lat[lane * LS + fl];
    if (v_out) v_out[o] = s_v[lane * VS + fl];
  }
}

// -> channels-last output [B, Ho, Wo, F]: one thread per (output pixel, VEC features), grid-stride;
// lat-only VEC = 4 windows reduce with byte-wise SIMD minima.
template <int VEC>
__global__ void __launch_bounds__(256) pool_nhwc2nhwc_kernel(const uint8_t* __restrict__ lat,
                                                             const float* __restrict__ v, int B, int F, int H, int W,
                                                             int PH, int PW, int SH, int SW, int DH, int DW, int Ho,
                                                             int Wo, int vfinal, uint8_t* __restrict__ lat_out,
                                                             float* __restrict__ v_out) {
  pdl_begin();
  const uint32_t FV = uint32_t(F / VEC), HoWo = uint32_t(Ho) * Wo;
  const uint32_t total = uint32_t(B) * HoWo * FV;  // < 2^32 (checked by the launcher): 32-bit index math
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
    const uint32_t pix = o / FV;
    const int f = int(o - pix * FV) * VEC;
    const uint32_t b = pix / HoWo, rem = pix - b * HoWo;
    const int oy = int(rem / uint32_t(Wo)), ox = int(rem - uint32_t(oy) * Wo);
    const uint8_t* limg = lat + int64_t(b) * H * W * F;
    const int64_t oi = int64_t(pix) * F + f;
    if (VEC == 4 && !v) {  // latencies only: min of the window's 4-byte words
      const int y0 = oy * SH - DH, x0 = ox * SW - DW;
      const int ya = y0 < 0 ? 0 : y0, yb = (y0 + PH < H ? y0 + PH : H);
      const int xa = x0 < 0 ? 0 : x0, xb = (x0 + PW < W ? x0 + PW : W);
      uint32_t m = 0xFFFFFFFFu;
      for (int yy = ya; yy < yb; ++yy) {
        uint32_t i = (uint32_t(yy) * W + xa) * F + f;
#pragma unroll 4
        for (int xx = xa; xx < xb; ++xx, i += F) m = __vminu4(m, __ldg(reinterpret_cast<const uint32_t*>(limg + i)));
      }
      *reinterpret_cast<uint32_t*>(lat_out + oi) = m;
      continue;
    }
    unsigned best[VEC];
    float bv[VEC];
    pool_window_nhwc<VEC>(limg, v ? v + int64_t(b) * H * W * F : nullptr, F, H, W, PH, PW, SH, SW, DH, DW, oy, ox, f,
                          vfinal, best, bv);
#pragma unroll
    for (int u = 0; u < VEC; ++u) {
      lat_out[oi + u] = uint8_t(best[u]);
      if (v_out) v_out[oi + u] = bv[u];
    }
  }
}

// Latencies only, channels-last in and out, F not a multiple of 4 (C2: F = 30 and 250): one warp per
// output pixel, lanes over its F contiguous features (coalesced byte runs, no per-byte index
// arithmetic), the min over the window's runs.  Windows inside the input (R10) or truncated (Eq. 3).
__global__ void __launch_bounds__(256) pool_nhwc_lat_rows_kernel(const uint8_t* __restrict__ lat, int B, int F,
                                                                 int H, int W, int PH, int PW, int SH, int SW, int DH,
                                                                 int DW, int Ho, int Wo,
                                                                 uint8_t* __restrict__ lat_out) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const uint32_t HoWo = uint32_t(Ho) * uint32_t(Wo);
  const uint32_t npix = uint32_t(B) * HoWo;  // < 2^32 (checked by the launcher): 32-bit index math
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5);
  for (uint32_t pix = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); pix < npix; pix += wstride) {
    const int b = int(pix / HoWo);
    const int rem = int(pix - uint32_t(b) * HoWo);
    const int oy = rem / Wo, ox = rem - (rem / Wo) * Wo;
    const int y0 = oy * SH - DH, x0 = ox * SW - DW;
    const int ya = y0 < 0 ? 0 : y0, yb = (y0 + PH < H ? y0 + PH : H);
    const int xa = x0 < 0 ? 0 : x0, xb = (x0 + PW < W ? x0 + PW : W);
    const uint8_t* img = lat + int64_t(b) * H * W * F;
    uint8_t* out = lat_out + int64_t(pix) * F;
    for (int f = lane; f < F; f += 32) {
      unsigned m = kNoSpike;
      for (int yy = ya; yy < yb; ++yy) {
        const uint8_t* row = img + (int64_t(yy) * W + xa) * F + f;
        for (int xx = xa; xx < xb; ++xx, row += F) m = min(m, unsigned(__ldg(row)));
      }
      out[f] = uint8_t(m);
    }
  }
}

int pool_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, int PH, int PW, int SH, int SW,
                int DH, int DW, int flags, uint8_t* lat_out, float* v_out, cudaStream_t s) {
  // R10 (windows inside the padded input), or Eq. 3 literally (last window truncated at the edge)
  const bool eq3 = flags & SNN_POOL_EQ3;
  const int Ho = eq3 ? (H + 2 * DH) / SH : (H + 2 * DH - PH) / SH + 1;
  const int Wo = eq3 ? (W + 2 * DW) / SW : (W + 2 * DW - PW) / SW + 1;
  const int64_t total = int64_t(B) * F * Ho * Wo;
  if (total == 0) return SNN_OK;
  if (flags & (SNN_POOL_IN_NHWC | SNN_POOL_OUT_NHWC)) {
    if (!(flags & SNN_POOL_IN_NHWC)) return set_error(SNN_EINVAL, "snn_pool: SNN_POOL_OUT_NHWC needs SNN_POOL_IN_NHWC");
    if (int64_t(H) * W * F >= (int64_t(1) << 32)) return set_error(SNN_ESHAPE, "snn_pool(NHWC input): H*W*F >= 2^32");
    const bool al = (reinterpret_cast<uintptr_t>(lat) & 3) == 0 && (reinterpret_cast<uintptr_t>(lat_out) & 3) == 0 &&
                    (!v_out || ((reinterpret_cast<uintptr_t>(v) & 15) == 0));
    const int vec = (F % 4 == 0 && al) ? 4 : 1;
    const float* vin = v_out ? v : nullptr;
    const int vf = (flags & SNN_POOL_VFINAL) ? 1 : 0;
    if (flags & SNN_POOL_OUT_NHWC) {
      if (total >= (int64_t(1) << 32)) return set_error(SNN_ESHAPE, "snn_pool(NHWC output): B*Ho*Wo*F >= 2^32");
      if (vec == 1 && !vin && !getenv("SNN_POOL_NOROWS")) {  // latencies only, F % 4 != 0: a warp per pixel
        int64_t nb = ceil_div(int64_t(B) * Ho * Wo, 8);  // a warp per output pixel (8 per CTA)
        if (nb > int64_t(num_sms()) * 64) nb = int64_t(num_sms()) * 64;
        launch_k(pool_nhwc_lat_rows_kernel, dim3(unsigned(nb)), dim3(256), 0, s, lat, B, F, H, W, PH, PW, SH, SW, DH,
                 DW, Ho, Wo, lat_out);
        note_launch();
        return check_launch("snn_pool(NHWC rows)");
      }
      int64_t nb = ceil_div(total / vec, 256);
      if (nb > int64_t(num_sms()) * 16) nb = int64_t(num_sms()) * 16;
      if (vec == 4)
        launch_k(pool_nhwc2nhwc_kernel<4>, dim3(unsigned(nb)), dim3(256), 0, s, lat, vin, B, F, H, W, PH, PW, SH, SW,
                 DH, DW, Ho, Wo, vf, lat_out, v_out);
      else
        launch_k(pool_nhwc2nhwc_kernel<1>, dim3(unsigned(nb)), dim3(256), 0, s, lat, vin, B, F, H, W, PH, PW, SH, SW,
                 DH, DW, Ho, Wo, vf, lat_out, v_out);
    } else {
      if (B > 65535 || Ho > 65535) return set_error(SNN_ESHAPE, "snn_pool(NHWC input): B or Ho > 65535");
      const int ntx = int(ceil_div(Wo, 32));
      const int FT = F < 32 * vec ? int(ceil_div(F, vec)) * vec : 32 * vec;  // features per tile
      const int nfc = int(ceil_div(F, FT));
      if (vec == 4)
        launch_k(pool_nhwc_kernel<4>, dim3(unsigned(ntx * nfc), unsigned(Ho), unsigned(B)), dim3(256), 0, s, lat, vin,
                 F, H, W, PH, PW, SH, SW, DH, DW, Ho, Wo, ntx, FT, vf, lat_out, v_out);
      else
        launch_k(pool_nhwc_kernel<1>, dim3(unsigned(ntx * nfc), unsigned(Ho), unsigned(B)), dim3(256), 0, s, lat, vin,
                 F, H, W, PH, PW, SH, SW, DH, DW, Ho, Wo, ntx, FT, vf, lat_out, v_out);
    }
    note_launch();
    return check_launch("snn_pool(NHWC input)");
  }
  int64_t blocks = ceil_div(total, 256);
  if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
  const bool small = total < (int64_t(1) << 32) && int64_t(B) * F * H * W < (int64_t(1) << 32);
  // the vector paths load 4-byte latency words / 16-byte potential vectors and store 2-byte / 8-byte
  // pairs: only for pointers with that alignment (a tensor view with an offset takes the scalar path)
  const auto al = [](const void* p, uintptr_t m) { return (reinterpret_cast<uintptr_t>(p) & (m - 1)) == 0; };
  const bool vec_ok = al(lat, 4) && al(lat_out, 2) && (!v_out || (al(v, 16) && al(v_out, 8)));
  if (small && vec_ok && v_out && PH == 2 && PW == 2 && SH == 2 && SW == 2 && DH == 0 && DW == 0 && W % 4 == 0 &&
      H % 2 == 0 && Wo % 2 == 0) {
    const uint32_t pairs = uint32_t(total / 2);
    int64_t pb = ceil_div(pairs, 256);
    if (pb > int64_t(num_sms()) * 16) pb = int64_t(num_sms()) * 16;
    launch_k(pool2x2_v_kernel, dim3(int(pb)), dim3(256), 0, s, lat, v, pairs, H, W, Ho, Wo, (flags & SNN_POOL_VFINAL) ? 1 : 0, lat_out,
                                              v_out);
  } else if (small && vec_ok && !v_out && PH == 2 && PW == 2 && SH == 2 && SW == 2 && DH == 0 && DW == 0 && W % 4 == 0 &&
             Wo * 2 == W) {
    const uint32_t words = uint32_t(int64_t(B) * F * Ho * (W / 4));
    int64_t wb = ceil_div(words, 256);
    if (wb > int64_t(num_sms()) * 16) wb = int64_t(num_sms()) * 16;
    launch_k(pool2x2_lat_kernel, dim3(int(wb)), dim3(256), 0, s, lat, words, H, W, Ho, lat_out);
  } else if (small && !v_out && PH * PW <= 16) {  // small windows: one thread per output row
    const uint32_t rows = uint32_t(int64_t(B) * F * Ho);
    int64_t rb = ceil_div(rows, 256);
    if (rb > int64_t(num_sms()) * 16) rb = int64_t(num_sms()) * 16;
    launch_k(pool_rows_kernel, dim3(int(rb)), dim3(256), 0, s, lat, rows, H, W, PH, PW, SH, SW, DH, DW, Ho, Wo, lat_out);
  } else if (small)
    launch_k(pool_kernel<uint32_t>, dim3(int(blocks)), dim3(256), 0, s, lat, v_out ? v : nullptr, int64_t(B) * F, H, W, PH, PW, SH, SW,
                                                      DH, DW, Ho, Wo, (flags & SNN_POOL_VFINAL) ? 1 : 0, lat_out, v_out);
  else
    launch_k(pool_kernel<int64_t>, dim3(int(blocks)), dim3(256), 0, s, lat, v_out ? v : nullptr, int64_t(B) * F, H, W, PH, PW, SH, SW,
                                                     DH, DW, Ho, Wo, (flags & SNN_POOL_VFINAL) ? 1 : 0, lat_out, v_out);
  note_launch();
  return check_launch("snn_pool");
}

// ------------------------------------------------------------------------------------- a5 inhibit
// Large maps: one thread per position, 8 features' loads in flight at a time (the v load only where
// the neuron spiked), then the write-back from the winning key alone (lat and v are recovered exactly
// from it, so nothing is read twice).  IDX = uint32_t when B*F*H*W < 2^32.
__device__ __forceinline__ float key_v(uint64_t key) {  // inverse of ordered_bits on the key's v field
  const uint32_t o = ~uint32_t(key >> 24);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

template <class IDX>
__global__ void __launch_bounds__(256) inhibit_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                      int B, int F, int64_t HW64, uint8_t* __restrict__ lat_out,
                                                      float* __restrict__ v_out, int16_t* __restrict__ winner_f) {
  pdl_begin();
  const IDX HW = IDX(HW64), total = IDX(B) * HW;
  for (IDX q = IDX(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += IDX(gridDim.x) * blockDim.x) {
    const IDX b = q / HW, p = q - b * HW;
    const IDX base = b * IDX(F) * HW + p;
    uint64_t best = ~uint64_t(0);
    for (int f0 = 0; f0 < F; f0 += 8) {
      uint32_t l[8];
      float vv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) l[j] = f0 + j < F ? lat[base + IDX(f0 + j) * HW] : kNoSpike;
#pragma unroll
      for (int j = 0; j < 8; ++j) vv[j] = l[j] != kNoSpike ? v[base + IDX(f0 + j) * HW] : 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (l[j] != kNoSpike) {
          const uint64_t k = wta_key(uint8_t(l[j]), vv[j], uint32_t(f0 + j));
          best = k < best ? k : best;
        }
    }
    const bool any = best != ~uint64_t(0);
    const int fw = any ? int(best & 0xFFFFFFu) : -1;
    const uint8_t lw = any ? uint8_t(best >> 56) : kNoSpike;
    const float vw = any ? key_v(best) : 0.0f;
    for (int f = 0; f < F; ++f) {
      const IDX i = base + IDX(f) * HW;
      lat_out[i] = f == fw ? lw : kNoSpike;
      v_out[i] = f == fw ? vw : 0.0f;
    }
    if (winner_f) winner_f[q] = int16_t(fw);
  }
}

// Small maps (batch-1 plasticity steps): one warp per position, lanes over features, so the
// per-position latency is one round of loads instead of F dependent ones.
constexpr int64_t kWarpPerPosMax = 16384;

__global__ void __launch_bounds__(256) inhibit_warp_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                           int B, int F, int64_t HW, uint8_t* __restrict__ lat_out,
                                                           float* __restrict__ v_out, int16_t* __restrict__ winner_f) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int64_t total = int64_t(B) * HW;
  for (int64_t q = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; q < total;
       q += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = q / HW, p = q - b * HW;
    const int64_t base = b * F * HW + p;
    uint64_t best = ~uint64_t(0);
    if (F <= 256) {  // all of the lane's (lat, v) loads in flight at once, kept for the write-back
      uint32_t l[8];
      float vv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int f = lane + 32 * j;
        l[j] = f < F ? lat[base + int64_t(f) * HW] : kNoSpike;
        vv[j] = f < F ? v[base + int64_t(f) * HW] : 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (l[j] != kNoSpike) {
          const uint64_t k = wta_key(uint8_t(l[j]), vv[j], uint32_t(lane + 32 * j));
          best = k < best ? k : best;
        }
      best = warp_min_u64(best);
      const int fw = best == ~uint64_t(0) ? -1 : int(best & 0xFFFFFFu);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int f = lane + 32 * j;
        if (f < F) {
          const int64_t i = base + int64_t(f) * HW;
          lat_out[i] = f == fw ? uint8_t(l[j]) : kNoSpike;
          v_out[i] = f == fw ? vv[j] : 0.0f;
        }
      }
      if (winner_f && lane == 0) winner_f[q] = int16_t(fw);
      continue;
    }
    for (int f = lane; f < F; f += 32) {
      const uint8_t l = lat[base + int64_t(f) * HW];
      if (l == kNoSpike) continue;
      const uint64_t k = wta_key(l, v[base + int64_t(f) * HW], uint32_t(f));
      best = k < best ? k : best;
    }
    best = warp_min_u64(best);
    const int fw = best == ~uint64_t(0) ? -1 : int(best & 0xFFFFFFu);
    for (int f = lane; f < F; f += 32) {
      const int64_t i = base + int64_t(f) * HW;
      const bool keep = f == fw;
      lat_out[i] = keep ? lat[i] : kNoSpike;
      v_out[i] = keep ? v[i] : 0.0f;
    }
    if (winner_f && lane == 0) winner_f[q] = int16_t(fw);
  }
}

// H*W % 4 == 0 (aligned maps): one thread per 4 consecutive positions -- 4-byte latency loads and
// stores, 16-byte potential loads (only for planes where one of the 4 spikes) and stores; 64-bit
// indexing (B*F*H*W may exceed 2^32: C5 is 2^28 neurons, larger batches are legal).
__global__ void __launch_bounds__(256) inhibit4_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                       int B, int F, int64_t HW, uint8_t* __restrict__ lat_out,
                                                       float* __restrict__ v_out, int16_t* __restrict__ winner_f) {
  pdl_begin();
  const int64_t HW4 = HW >> 2, total = int64_t(B) * HW4;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = q / HW4, p = (q - b * HW4) << 2;
    const int64_t base = b * F * HW + p;
    uint64_t best[4] = {~uint64_t(0), ~uint64_t(0), ~uint64_t(0), ~uint64_t(0)};
    for (int f0 = 0; f0 < F; f0 += 8) {
      uint32_t l[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        l[u] = f0 + u < F ? __ldg(reinterpret_cast<const uint32_t*>(lat + base + int64_t(f0 + u) * HW)) : 0xFFFFFFFFu;
      float4 vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        vv[u] = l[u] != 0xFFFFFFFFu ? __ldg(reinterpret_cast<const float4*>(v + base + int64_t(f0 + u) * HW))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (l[u] == 0xFFFFFFFFu) continue;
        const float vj[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint8_t lj = uint8_t(l[u] >> (8 * j));
          if (lj == kNoSpike) continue;
          const uint64_t k = wta_key(lj, vj[j], uint32_t(f0 + u));
          best[j] = k < best[j] ? k : best[j];
        }
      }
    }
    int fw[4];
    uint32_t lw[4];
    float vw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool any = best[j] != ~uint64_t(0);
      fw[j] = any ? int(best[j] & 0xFFFFFFu) : -1;
      lw[j] = any ? uint32_t(best[j] >> 56) : kNoSpike;
      vw[j] = any ? key_v(best[j]) : 0.0f;
    }
    for (int f = 0; f < F; ++f) {
      const int64_t i = base + int64_t(f) * HW;
      uint32_t lo = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) lo |= (f == fw[j] ? lw[j] : uint32_t(kNoSpike)) << (8 * j);
      *reinterpret_cast<uint32_t*>(lat_out + i) = lo;
      *reinterpret_cast<float4*>(v_out + i) =
          make_float4(f == fw[0] ? vw[0] : 0.f, f == fw[1] ? vw[1] : 0.f, f == fw[2] ? vw[2] : 0.f,
                      f == fw[3] ? vw[3] : 0.f);
    }
    if (winner_f)
#pragma unroll
      for (int j = 0; j < 4; ++j) winner_f[b * HW + p + j] = int16_t(fw[j]);
  }
}

int inhibit_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, uint8_t* lat_out, float* v_out,
                   int16_t* winner_f, cudaStream_t s) {
  const int64_t HW = int64_t(H) * W, total = int64_t(B) * HW;
  if (total == 0) return SNN_OK;
  if (total <= kWarpPerPosMax) {
    launch_k(inhibit_warp_kernel, dim3(int(ceil_div(total, 8))), dim3(256), 0, s, lat, v, B, F, HW, lat_out, v_out, winner_f);
    note_launch();
    return check_launch("snn_inhibit");
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(lat) & 3) == 0 && (reinterpret_cast<uintptr_t>(lat_out) & 3) == 0 &&
                       (reinterpret_cast<uintptr_t>(v) & 15) == 0 && (reinterpret_cast<uintptr_t>(v_out) & 15) == 0;
  if (HW % 4 == 0 && aligned && !getenv("SNN_INHIBIT1")) {
    int64_t b4 = ceil_div(total / 4, 256);
    if (b4 > int64_t(num_sms()) * 8) b4 = int64_t(num_sms()) * 8;
    launch_k(inhibit4_kernel, dim3(int(b4)), dim3(256), 0, s, lat, v, B, F, HW, lat_out, v_out, winner_f);
    note_launch();
    return check_launch("snn_inhibit");
  }
  int64_t blocks = ceil_div(total, 256);
  if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
  if (int64_t(B) * F * HW < (int64_t(1) << 32))
    launch_k(inhibit_kernel<uint32_t>, dim3(int(blocks)), dim3(256), 0, s, lat, v, B, F, HW, lat_out, v_out, winner_f);
  else
    launch_k(inhibit_kernel<int64_t>, dim3(int(blocks)), dim3(256), 0, s, lat, v, B, F, HW, lat_out, v_out, winner_f);
  note_launch();
  return check_launch("snn_inhibit");
}

// ------------------------------------------------------------------------------------- a6 k-WTA
// Stage 1 for H*W % 4 == 0: one thread per 4 consecutive positions, one 4-byte latency load per
// feature (a warp reads 128 contiguous bytes per feature plane), 8 features in flight -- the map is
// far larger than L2 on the throughput configs, so bytes in flight set the speed.
__global__ void __launch_bounds__(256) kwta_posbest4_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                            int B, int F, int HW, uint64_t* __restrict__ pos_best,
                                                            uint8_t* __restrict__ multi) {
  pdl_begin();
  const int HW4 = HW >> 2;
  const int64_t total = int64_t(B) * HW4;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(q / HW4), p = (int(q - int64_t(b) * HW4)) << 2;
    const uint32_t* lp = reinterpret_cast<const uint32_t*>(lat + int64_t(b) * F * HW + p);
    const float* vp = v + int64_t(b) * F * HW + p;
    uint64_t best[4] = {~uint64_t(0), ~uint64_t(0), ~uint64_t(0), ~uint64_t(0)};
    int nspk[4] = {0, 0, 0, 0};
    for (int f = 0; f < F; f += 8) {
      uint32_t l[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) l[u] = f + u < F ? __ldg(lp + (f + u) * HW4) : 0xFFFFFFFFu;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (l[u] == 0xFFFFFFFFu) continue;  // none of the 4 positions spikes in this plane
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint8_t lj = uint8_t(l[u] >> (8 * j));
          if (lj == kNoSpike) continue;
          const uint64_t k = wta_key(lj, vp[(f + u) * HW + j], uint32_t((f + u) * HW + p + j));
          best[j] = k < best[j] ? k : best[j];
          ++nspk[j];
        }
      }
    }
    uint64_t* out = pos_best + int64_t(b) * HW + p;
#pragma unroll
    for (int j = 0; j < 4; ++j) out[j] = best[j];
    if (multi)
      *reinterpret_cast<uint32_t*>(multi + int64_t(b) * HW + p) =
          uint32_t(nspk[0] > 1) | uint32_t(nspk[1] > 1) << 8 | uint32_t(nspk[2] > 1) << 16 | uint32_t(nspk[3] > 1) << 24;
  }
}

// Stage 1 (all SMs): best key over features for every position -> pos_best[b][p].
// 32-bit indexing (F*H*W <= 2^24 is checked at the ABI), 4 features in flight per thread.
__global__ void __launch_bounds__(256) kwta_posbest_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                           int B, int F, int HW, uint64_t* __restrict__ pos_best,
                                                           uint8_t* __restrict__ multi) {
  pdl_begin();
  const int64_t total = int64_t(B) * HW;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(q / HW), p = int(q - int64_t(b) * HW);
    const uint8_t* lp = lat + int64_t(b) * F * HW + p;
    const float* vp = v + int64_t(b) * F * HW + p;
    uint64_t best = ~uint64_t(0);
    int nspk = 0;
    int f = 0;
    for (; f + 4 <= F; f += 4) {
      uint8_t l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) l[u] = lp[(f + u) * HW];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (l[u] == kNoSpike) continue;
        const uint64_t k = wta_key(l[u], vp[(f + u) * HW], uint32_t((f + u) * HW + p));
        best = k < best ? k : best;
        ++nspk;
      }
    }
    for (; f < F; ++f) {
      const uint8_t l = lp[f * HW];
      if (l == kNoSpike) continue;
      const uint64_t k = wta_key(l, vp[f * HW], uint32_t(f * HW + p));
      best = k < best ? k : best;
      ++nspk;
    }
    pos_best[q] = best;
    if (multi) multi[q] = uint8_t(nspk > 1);
  }
}

__global__ void __launch_bounds__(256) kwta_posbest_warp_kernel(const uint8_t* __restrict__ lat,
                                                                const float* __restrict__ v, int B, int F, int HW,
                                                                uint64_t* __restrict__ pos_best) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int64_t total = int64_t(B) * HW;
  for (int64_t q = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; q < total;
       q += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int b = int(q / HW), p = int(q - int64_t(b) * HW);
    const uint8_t* lp = lat + int64_t(b) * F * HW + p;
    const float* vp = v + int64_t(b) * F * HW + p;
    uint64_t best = ~uint64_t(0);
#pragma unroll 4
    for (int f = lane; f < F; f += 32) {
      const uint8_t l = lp[f * HW];
      const float vf = vp[f * HW];
      if (l == kNoSpike) continue;
      const uint64_t k = wta_key(l, vf, uint32_t(f * HW + p));
      best = k < best ? k : best;
    }
    best = warp_min_u64(best);
    if (lane == 0) pos_best[q] = best;
  }
}

// Stage 1 with candidate lists (k + 1 <= kTopM, F <= 512, H*W <= kKwtaSmemPos): one warp per
// position keeps its features' keys in registers and extracts the M = k + 1 smallest in ascending
// order.  A position can lose at most k - 1 features to earlier winners before its last use, so its
// best remaining candidate is always in the list (or the list holds all its spiking features): the
// rounds never rescan the maps.
constexpr int kTopM = 17;
__global__ void __launch_bounds__(256) kwta_topk_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                        int B, int F, int HW, int M, uint64_t* __restrict__ pos_best,
                                                        uint64_t* __restrict__ topk) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int64_t total = int64_t(B) * HW;
  for (int64_t q = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; q < total;
       q += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int b = int(q / HW), p = int(q - int64_t(b) * HW);
    const uint8_t* lp = lat + int64_t(b) * F * HW + p;
    const float* vp = v + int64_t(b) * F * HW + p;
    uint64_t key[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int f = lane + 32 * j;
      key[j] = ~uint64_t(0);
      if (f < F) {  // lat and v loads independent: all in flight
        const uint8_t l = lp[int64_t(f) * HW];
        const float vf = vp[int64_t(f) * HW];
        if (l != kNoSpike) key[j] = wta_key(l, vf, uint32_t(f * HW + p));
      }
    }
    uint64_t prev = 0;
    bool first = true;
    for (int m = 0; m < M; ++m) {
      uint64_t mn = ~uint64_t(0);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if ((first || key[j] > prev) && key[j] < mn) mn = key[j];
      mn = warp_min_u64(mn);
      if (lane == 0) topk[q * M + m] = mn;
      if (m == 0 && lane == 0) pos_best[q] = mn;
      prev = mn;
      first = false;
      if (mn == ~uint64_t(0)) break;  // fewer than M spiking features: ~0 ends the list (read no further)
    }
  }
}

// Stage 2 (one CTA per image): k rounds of a block argmin over positions.  After each round the
// winner's (2r+1)^2 window is cleared (inhibited in all maps) and the positions whose best feature
// won are re-evaluated over the remaining features.  The per-image key map is staged in shared
// memory when it fits (<= 16384 positions).
constexpr int kKwtaThreads = 1024;
constexpr int kKwtaSmemPos = 16384;
constexpr int kKwtaQueue = 4096;

__global__ void __launch_bounds__(kKwtaThreads) kwta_rounds_kernel(const uint8_t* __restrict__ lat,
                                                                   const float* __restrict__ v, int F, int H, int W,
                                                                   int k, int r, uint64_t* __restrict__ pos_best,
                                                                   const uint64_t* __restrict__ topk, int M,
                                                                   int32_t* __restrict__ winners,
                                                                   int32_t* __restrict__ count, int use_smem,
                                                                   const uint8_t* __restrict__ multi) {
  pdl_begin();
  extern __shared__ uint64_t dyn[];  // [HW] current keys, then (topk) [HW] list cursors (u8)
  __shared__ uint32_t fexcl[256];  // bitmask of excluded features (F <= 8192)
  __shared__ uint64_t red[32];
  __shared__ int s_count, s_qn, s_wf, s_wy, s_wx;
  __shared__ int queue[kKwtaQueue];
  const int b = blockIdx.x;
  const int HW = H * W;
  uint64_t* pbg = pos_best + int64_t(b) * HW;
  uint64_t* pb = use_smem ? dyn : pbg;
  const uint8_t* lb = lat + int64_t(b) * F * HW;
  const float* vb = v + int64_t(b) * F * HW;
  const int nwords = (F + 31) >> 5;
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) fexcl[i] = 0;
  uint8_t* cur = reinterpret_cast<uint8_t*>(dyn + HW);
  const uint64_t* tk = topk ? topk + int64_t(b) * HW * M : nullptr;
  if (use_smem)
    for (int p = threadIdx.x; p < HW; p += blockDim.x) {
      dyn[p] = pbg[p];
      if (topk) cur[p] = 0;
    }
  if (threadIdx.x == 0) { s_count = 0; s_qn = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // Invariant between rounds: every live key in pb[] is a valid candidate -- its position is outside
  // the radius of every winner so far and its feature has not won.  The winner of a round therefore
  // is a plain argmin, and only the round's own winner has to be applied afterwards: its (2r+1)^2
  // window is killed directly and the positions whose key carries the winning feature (an index
  // range test, no division) move to their next candidate.  Those re-evaluations are folded into the
  // next round's argmin, so a round costs three barriers and O(H*W / threads) shared loads.
  for (int round = 0; round < k; ++round) {
    uint64_t best = ~uint64_t(0);
    {  // positions queued by the previous round: one warp each, lanes scan the features
      const int qn = s_qn < kKwtaQueue ? s_qn : kKwtaQueue;
      for (int qi = wid; qi < qn; qi += nwarps) {
        const int p = queue[qi];
        SNN_DCHECK(p >= 0 && p < HW);
        uint64_t key = ~uint64_t(0);
        for (int f0 = lane; f0 < F; f0 += 32 * 8) {  // 8 strided latency loads in flight per lane
          uint8_t l[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) l[u] = f0 + 32 * u < F ? lb[(f0 + 32 * u) * HW + p] : kNoSpike;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int ff = f0 + 32 * u;
            if (l[u] == kNoSpike || (fexcl[ff >> 5] >> (ff & 31) & 1)) continue;
            const uint64_t kk = wta_key(l[u], vb[ff * HW + p], uint32_t(ff * HW + p));
            key = kk < key ? kk : key;
          }
        }
        key = warp_min_u64(key);
        if (lane == 0) pb[p] = key;
        best = key < best ? key : best;
      }
    }
    for (int p = threadIdx.x; p < HW; p += blockDim.x) {
      const uint64_t key = pb[p];  // a queued position reads ~0 or its new key: both are counted
      best = key < best ? key : best;
    }
    best = warp_min_u64(best);
    if (lane == 0) red[wid] = best;
    __syncthreads();
    if (wid == 0) {
      uint64_t x = lane < nwarps ? red[lane] : ~uint64_t(0);
      x = warp_min_u64(x);
      if (lane == 0) {
        s_qn = 0;
        if (x != ~uint64_t(0)) {
          const int idx = int(x & 0xFFFFFFu);
          const int f = idx / HW, p = idx - f * HW;
          const int y = p / W, xx = p - y * W;
          const int c = s_count;
          winners[(int64_t(b) * k + c) * 3 + 0] = f;
          winners[(int64_t(b) * k + c) * 3 + 1] = y;
          winners[(int64_t(b) * k + c) * 3 + 2] = xx;
          s_wf = f; s_wy = y; s_wx = xx;
          fexcl[f >> 5] |= 1u << (f & 31);
          s_count = c + 1;
        }
      }
    }
    __syncthreads();
    if (s_count == round) break;  // no candidate left
    if (round + 1 == k) break;
    const int wf = s_wf, wyy = s_wy, wxx = s_wx;
    {  // the winner's window (clipped to the map) leaves every map
      const int y0 = max(wyy - r, 0), y1 = min(wyy + r, H - 1);
      const int x0 = max(wxx - r, 0), x1 = min(wxx + r, W - 1);
      const int ww = x1 - x0 + 1, n = (y1 - y0 + 1) * ww;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int dy = i / ww;
        pb[(y0 + dy) * W + x0 + (i - dy * ww)] = ~uint64_t(0);
      }
    }
    const uint32_t lo = uint32_t(wf) * uint32_t(HW);
    for (int p = threadIdx.x; p < HW; p += blockDim.x) {
      const uint64_t key = pb[p];
      if (key == ~uint64_t(0) || uint32_t(key & 0xFFFFFFu) - lo >= uint32_t(HW)) continue;
      const int y = p / W, x = p - y * W;
      if (abs(y - wyy) <= r && abs(x - wxx) <= r) continue;  // killed by the window above
      if (tk) {  // next entry of the position's candidate list whose feature has not won
        int c = cur[p];
        uint64_t kk;
        for (;;) {
          ++c;
          kk = c < M ? tk[int64_t(p) * M + c] : ~uint64_t(0);
          if (kk == ~uint64_t(0)) break;
          const int ff = int(uint32_t(kk & 0xFFFFFFu) / uint32_t(HW));
          if (!(fexcl[ff >> 5] >> (ff & 31) & 1)) break;
        }
        cur[p] = uint8_t(c < M ? c : M);
        pb[p] = kk;
        continue;
      }
      if (multi && !multi[int64_t(b) * HW + p]) {  // its only spiking feature won: nothing left
        pb[p] = ~uint64_t(0);
        continue;
      }
      const int slot = atomicAdd(&s_qn, 1);
      if (slot < kKwtaQueue) {
        pb[p] = ~uint64_t(0);
        queue[slot] = p;
      } else {  // queue overflow (rare): serial re-evaluation by this thread
        uint64_t kk2 = ~uint64_t(0);
        for (int ff = 0; ff < F; ++ff) {
          if (fexcl[ff >> 5] >> (ff & 31) & 1) continue;
          const uint8_t l = lb[ff * HW + p];
          if (l == kNoSpike) continue;
          const uint64_t kk = wta_key(l, vb[ff * HW + p], uint32_t(ff * HW + p));
          kk2 = kk < kk2 ? kk : kk2;
        }
        pb[p] = kk2;
      }
    }
    __syncthreads();
  }
  for (int i = s_count + threadIdx.x; i < k; i += blockDim.x) {
    winners[(int64_t(b) * k + i) * 3 + 0] = -1;
    winners[(int64_t(b) * k + i) * 3 + 1] = -1;
    winners[(int64_t(b) * k + i) * 3 + 2] = -1;
  }
  if (threadIdx.x == 0) count[b] = s_count;
}

size_t k_winners_workspace(int B, int F, int H, int W) {
  (void)F;
  // current key per position + (maps up to kKwtaSmemPos positions) candidate lists of up to kTopM keys
  const size_t per = (size_t(H) * W <= size_t(kKwtaSmemPos)) ? 1 + size_t(kTopM) : 1;
  // + one byte per position: "more than one feature spikes here" (a lone candidate is not rescanned)
  return size_t(B) * H * W * sizeof(uint64_t) * per + size_t(B) * H * W + 256;
}

// Stage 2 for small maps with candidate lists (H*W <= 1024: one position per thread): one barrier
// per round.  Every warp reduces the same per-warp minima (double-buffered, so the next round's writes
// cannot race a slow reader), every thread learns the winner and updates only its own position --
// killed inside the winner's Chebyshev-r neighbourhood (R15), else advanced along its list past features
// that have won (each thread keeps its own copy of that set by writing the same bits).
__global__ void __launch_bounds__(1024) kwta_rounds_small_kernel(int F, int H, int W, int k, int r,
                                                                 const uint64_t* __restrict__ pos_best,
                                                                 const uint64_t* __restrict__ topk, int M,
                                                                 int32_t* __restrict__ winners,
                                                                 int32_t* __restrict__ count) {
  pdl_begin();
  __shared__ uint64_t red[2][32];
  __shared__ uint32_t fexcl[256];  // F <= 8192
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  const int HW = H * W;
  for (int i = tid; i < 256; i += blockDim.x) fexcl[i] = 0;
  const int p = tid;
  uint64_t key = p < HW ? pos_best[int64_t(b) * HW + p] : ~uint64_t(0);
  const int py = p / W, px = p - (p / W) * W;
  int cur = 0, nwin = 0;
  __syncthreads();
  for (int round = 0; round < k; ++round) {
    uint64_t m = warp_min_u64(key);
    if (lane == 0) red[round & 1][wid] = m;
    __syncthreads();
    m = lane < nwarps ? red[round & 1][lane] : ~uint64_t(0);
    m = warp_min_u64(m);
    if (m == ~uint64_t(0)) break;  // block-uniform
    const int idx = int(m & 0xFFFFFFu), f = idx / HW, pw = idx - f * HW, wy = pw / W, wx = pw - (pw / W) * W;
    if (tid == 0) {
      int32_t* wr = winners + (int64_t(b) * k + nwin) * 3;
      wr[0] = f; wr[1] = wy; wr[2] = wx;
    }
    atomicOr(&fexcl[f >> 5], 1u << (f & 31));
    ++nwin;
    if (key == ~uint64_t(0)) continue;
    if (abs(py - wy) <= r && abs(px - wx) <= r) { key = ~uint64_t(0); continue; }
    int ff = int(uint32_t(key & 0xFFFFFFu) / uint32_t(HW));
    while (fexcl[ff >> 5] >> (ff & 31) & 1) {  // its feature has won: next list entry
      ++cur;
      key = cur < M ? topk[(int64_t(b) * HW + p) * M + cur] : ~uint64_t(0);
      if (key == ~uint64_t(0)) break;
      ff = int(uint32_t(key & 0xFFFFFFu) / uint32_t(HW));
    }
  }
  for (int i = nwin + tid; i < k; i += blockDim.x) {
    int32_t* wr = winners + (int64_t(b) * k + i) * 3;
    wr[0] = -1; wr[1] = -1; wr[2] = -1;
  }
  if (tid == 0) count[b] = nwin;
}

// k = 1 (C2's decision layer, C4's R-STDP winner): the single winner is the minimum key over every
// neuron of the image -- a plain reduction, spread over cpi CTAs per image for large maps (each writes
// its block minimum to the workspace), then one thread per image reduces them and decodes (f, y, x).
__global__ void __launch_bounds__(256) kwta_k1_min_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                          int n, int cpi, uint64_t* __restrict__ part_min) {
  pdl_begin();
  __shared__ uint64_t red[8];
  const int b = blockIdx.x / cpi, part = blockIdx.x - b * cpi;
  const uint8_t* lb = lat + int64_t(b) * n;
  const float* vb = v + int64_t(b) * n;
  uint64_t m = ~uint64_t(0);
  const int stride = cpi * 256;
  for (int i0 = part * 256 + threadIdx.x; i0 < n; i0 += 4 * stride) {  // 4 neurons' loads in flight
    uint32_t l[4];
    float vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) l[u] = i0 + u * stride < n ? lb[i0 + u * stride] : kNoSpike;
#pragma unroll
    for (int u = 0; u < 4; ++u) vv[u] = l[u] != kNoSpike ? vb[i0 + u * stride] : 0.0f;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (l[u] != kNoSpike) {
        const uint64_t k = wta_key(uint8_t(l[u]), vv[u], uint32_t(i0 + u * stride));  // flat index (R14)
        m = k < m ? k : m;
      }
  }
  m = warp_min_u64(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < 8 ? red[threadIdx.x] : ~uint64_t(0);
    m = warp_min_u64(m);
    if (threadIdx.x == 0) part_min[blockIdx.x] = m;
  }
}

__global__ void kwta_k1_emit_kernel(const uint64_t* __restrict__ part_min, int B, int cpi, int HW, int W,
                                    int32_t* __restrict__ winners, int32_t* __restrict__ count) {
  pdl_begin();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  uint64_t m = ~uint64_t(0);
  for (int c = 0; c < cpi; ++c) {
    const uint64_t x = part_min[int64_t(b) * cpi + c];
    m = x < m ? x : m;
  }
  if (m == ~uint64_t(0)) {
    winners[b * 3 + 0] = -1; winners[b * 3 + 1] = -1; winners[b * 3 + 2] = -1;
    count[b] = 0;
    return;
  }
  const int idx = int(m & 0xFFFFFFu), f = idx / HW, p = idx - f * HW;
  winners[b * 3 + 0] = f; winners[b * 3 + 1] = p / W; winners[b * 3 + 2] = p - (p / W) * W;
  count[b] = 1;
}

// k = 1 with one CTA per image (up to ~64 neurons per thread): reduction and decode in one kernel.
template <int NT>
__global__ void __launch_bounds__(NT) kwta_k1_block_kernel(const uint8_t* __restrict__ lat, const float* __restrict__ v,
                                                           int n, int HW, int W, int32_t* __restrict__ winners,
                                                           int32_t* __restrict__ count) {
  pdl_begin();
  __shared__ uint64_t red[NT / 32];
  const int b = blockIdx.x;
  const uint8_t* lb = lat + int64_t(b) * n;
  const float* vb = v + int64_t(b) * n;
  uint64_t m = ~uint64_t(0);
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * NT) {  // 4 neurons' loads in flight
    uint32_t l[4];
    float vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) l[u] = i0 + u * NT < n ? lb[i0 + u * NT] : kNoSpike;
#pragma unroll
    for (int u = 0; u < 4; ++u) vv[u] = l[u] != kNoSpike ? vb[i0 + u * NT] : 0.0f;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (l[u] != kNoSpike) {
        const uint64_t k = wta_key(uint8_t(l[u]), vv[u], uint32_t(i0 + u * NT));
        m = k < m ? k : m;
      }
  }
  m = warp_min_u64(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < NT / 32 ? red[threadIdx.x] : ~uint64_t(0);
    m = warp_min_u64(m);
    if (threadIdx.x == 0) {
      if (m == ~uint64_t(0)) {
        winners[b * 3 + 0] = -1; winners[b * 3 + 1] = -1; winners[b * 3 + 2] = -1;
        count[b] = 0;
      } else {
        const int idx = int(m & 0xFFFFFFu), f = idx / HW, p = idx - f * HW;
        winners[b * 3 + 0] = f; winners[b * 3 + 1] = p / W; winners[b * 3 + 2] = p - (p / W) * W;
        count[b] = 1;
      }
    }
  }
}

int k_winners_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, int k, int r, int32_t* winners,
                     int32_t* count, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (B == 0) return SNN_OK;
  const int64_t HW = int64_t(H) * W;
  if (ws_bytes < size_t(B) * HW * sizeof(uint64_t) || ws_bytes < size_t(B) * sizeof(uint64_t))
    return set_error(SNN_EWORKSPACE, "snn_k_winners: workspace too small");
  if (k == 1 && int64_t(F) * HW <= 1024 * 8) {  // one CTA per image suffices: no separate decode kernel
    // (larger maps of one image -- C4: 21,600 neurons -- are faster spread over several CTAs below)
    const int n = int(int64_t(F) * HW);
    if (n > 256 * 16 || B < num_sms())
      launch_k(kwta_k1_block_kernel<1024>, dim3(B), dim3(1024), 0, s, lat, v, n, int(HW), W, winners, count);
    else
      launch_k(kwta_k1_block_kernel<256>, dim3(B), dim3(256), 0, s, lat, v, n, int(HW), W, winners, count);
    note_launch();
    return check_launch("snn_k_winners(k=1)");
  }
  if (k == 1) {
    uint64_t* part_min = reinterpret_cast<uint64_t*>(ws);
    const int n = int(int64_t(F) * HW);
    int cpi = int(ceil_div(n, 256 * 4));  // ~4 neurons per thread, loaded together
    if (cpi < 1) cpi = 1;
    while (cpi > 1 && size_t(B) * cpi * sizeof(uint64_t) > ws_bytes) cpi /= 2;
    launch_k(kwta_k1_min_kernel, dim3(unsigned(int64_t(B) * cpi)), dim3(256), 0, s, lat, v, n, cpi, part_min);
    launch_k(kwta_k1_emit_kernel, dim3(int(ceil_div(B, 128))), dim3(128), 0, s, part_min, B, cpi, int(HW), W, winners, count);
    note_launch(2);
    return check_launch("snn_k_winners(k=1)");
  }
  uint64_t* pb = reinterpret_cast<uint64_t*>(ws);
  int64_t total = int64_t(B) * HW;
  int64_t blocks = ceil_div(total, 256);
  if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
  if (blocks < 1) blocks = 1;
  const int use_smem = HW <= kKwtaSmemPos;
  const int M = k + 1;
  const bool lists = k >= 2 && total <= kWarpPerPosMax && use_smem && M <= kTopM && F <= 512 &&
                     ws_bytes >= size_t(B) * HW * sizeof(uint64_t) * (1 + size_t(M));
  uint64_t* topk = lists ? pb + total : nullptr;
  const size_t multi_off = size_t(total) * sizeof(uint64_t) * (1 + (lists ? size_t(M) : 0));
  uint8_t* multi = !lists && ws_bytes >= multi_off + size_t(total) ? static_cast<uint8_t*>(ws) + multi_off : nullptr;
  if (lists) {
    int64_t wb = ceil_div(total, 8);
    if (wb > int64_t(num_sms()) * 32) wb = int64_t(num_sms()) * 32;
    launch_k(kwta_topk_kernel, dim3(int(wb)), dim3(256), 0, s, lat, v, B, F, int(HW), M, pb, topk);
  } else if (total <= kWarpPerPosMax) {
    launch_k(kwta_posbest_warp_kernel, dim3(int(ceil_div(total, 8))), dim3(256), 0, s, lat, v, B, F, int(HW), pb);
    multi = nullptr;  // (the warp-per-position stage does not count candidates)
  } else {
    if (HW % 4 == 0 && (reinterpret_cast<uintptr_t>(lat) & 3) == 0 && !getenv("SNN_KWTA_POSBEST1")) {
      int64_t b4 = ceil_div(total / 4, 256);
      if (b4 > int64_t(num_sms()) * 8) b4 = int64_t(num_sms()) * 8;
      launch_k(kwta_posbest4_kernel, dim3(int(b4)), dim3(256), 0, s, lat, v, B, F, int(HW), pb, multi);
    } else {
      launch_k(kwta_posbest_kernel, dim3(int(blocks)), dim3(256), 0, s, lat, v, B, F, int(HW), pb, multi);
    }
  }
  note_launch();
  if (lists && HW <= 1024 && !getenv("SNN_KWTA_NOSMALL")) {
    launch_k(kwta_rounds_small_kernel, dim3(B), dim3(int(ceil_div(HW, 32)) * 32), 0, s, F, H, W, k, r, pb, topk, M,
             winners, count);
    note_launch();
    return check_launch("snn_k_winners");
  }
  const size_t smem = use_smem ? size_t(HW) * sizeof(uint64_t) + (lists ? size_t(HW) : 0) : 0;
  cudaError_t e = cudaFuncSetAttribute(kwta_rounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_k_winners: %s", cudaGetErrorString(e));
  int nthr = kKwtaThreads;  // measured C1 (784 positions): 1024 threads 59 us step, 512 67, 256 70
  if (const char* e = getenv("SNN_KWTA_THREADS")) nthr = atoi(e);  // tuning experiments
  launch_k(kwta_rounds_kernel, dim3(B), dim3(nthr), smem, s, lat, v, F, H, W, k, r, pb, topk, M, winners, count, use_smem,
           const_cast<const uint8_t*>(multi));
  note_launch();
  return check_launch("snn_k_winners");
}

// ------------------------------------------------------------------------------------- decision
__global__ void decide_kernel(const int32_t* __restrict__ winners, const int32_t* __restrict__ count, int B, int k,
                              int F, int n_classes, const int32_t* __restrict__ labels, int32_t* __restrict__ decision,
                              float* __restrict__ reward) {
  pdl_begin();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int d = -1;
  float rw = 0.0f;
  if (count[b] > 0) {
    d = winners[int64_t(b) * k * 3] / (F / n_classes);
    if (labels) rw = (d == labels[b]) ? 1.0f : -1.0f;
  }
  if (decision) decision[b] = d;
  if (reward) reward[b] = rw;
}

int decide_launch(const int32_t* winners, const int32_t* count, int B, int k, int F, int n_classes,
                  const int32_t* labels, int32_t* decision, float* reward, cudaStream_t s) {
  if (B == 0) return SNN_OK;
  launch_k(decide_kernel, dim3(int(ceil_div(B, 256))), dim3(256), 0, s, winners, count, B, k, F, n_classes, labels, decision, reward);
  note_launch();
  return check_launch("snn_decide");
}

}  // namespace snn
