// stdp.cu -- a7: STDP / R-STDP weight update of one image, in place (Eq. 4, P:161;
// DESIGN.md R17-R23).  One CTA per (winner slot, slice of 256 synapses), one thread per synapse:
// a gather of the winner's receptive field (pre spike times) and an elementwise fp32 update.
// The winners of k-WTA have distinct features, so their kernels are disjoint (no write races).
// Arithmetic is fp32 round-to-nearest with explicit intrinsics so no FMA is contracted:
//   dW = (a * (W - lb)) * (ub - W)   (stabilizer on, Eq. 4 left to right)  or  dW = a
//   W  = min(max(W + dW, lb), ub)   (no clamp for stabilizer == 2, the A20 variant)
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace snn {

__global__ void __launch_bounds__(256) stdp_kernel(float* __restrict__ w, int C, int KH, int KW,
                                                   const uint8_t* __restrict__ lat_in, int H, int W, int pad,
                                                   const uint8_t* __restrict__ lat_out, int Ho, int Wo,
                                                   const int32_t* __restrict__ winners,
                                                   const int32_t* __restrict__ count, float a_plus, float a_minus,
                                                   float lb, float ub, int stabilizer,
                                                   const float* __restrict__ reward, int f0, int Floc, int sharded,
                                                   int* err) {
  pdl_begin();
  const int i = blockIdx.x;  // winner slot; blockIdx.y = slice of its synapses (gridDim.y slices)
  if (i >= count[0]) return;
  {  // a winner outside the map (or, unsharded, outside the layer's features) is skipped and reported
    const int wf = winners[i * 3], wy = winners[i * 3 + 1], wx = winners[i * 3 + 2];
    const bool bad = wf < 0 || wy < 0 || wy >= Ho || wx < 0 || wx >= Wo || (!sharded && wf >= Floc);
    if (bad) {
      if (blockIdx.y == 0 && threadIdx.x == 0) flag_error(err, kErrWinner);
      return;
    }
  }
  if (winners[i * 3] < f0 || winners[i * 3] >= f0 + Floc) return;  // another rank's feature (f4 sharding)
  float rw = reward ? reward[0] : 1.0f;
  if (rw == 0.0f) return;  // silent sample: no plasticity
  const float ap = rw > 0.0f ? a_plus : -a_plus;   // anti-STDP = negated rates
  const float am = rw > 0.0f ? a_minus : -a_minus;
  const int f = winners[i * 3 + 0] - f0, y = winners[i * 3 + 1], x = winners[i * 3 + 2];
  const int post = lat_out[(int64_t(f) * Ho + y) * Wo + x];
  const int KK = KH * KW, R = C * KK;
  float* wf = w + int64_t(f) * R;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < R; e += gridDim.y * blockDim.x) {
    const int c = e / KK, rr = e - c * KK, ky = rr / KW, kx = rr - ky * KW;
    const int yy = y + ky - pad, xx = x + kx - pad;
    int pre = kNoSpike;
    if (yy >= 0 && yy < H && xx >= 0 && xx < W) pre = lat_in[(int64_t(c) * H + yy) * W + xx];
    const float a = (pre != kNoSpike && pre <= post) ? ap : am;  // T_j <= T_i -> LTP (Eq. 4)
    const float w0 = wf[e];
    const float dw = stabilizer ? __fmul_rn(__fmul_rn(a, __fsub_rn(w0, lb)), __fsub_rn(ub, w0)) : a;
    float w1 = __fadd_rn(w0, dw);
    if (stabilizer != 2) {  // 2 = stabilized without the clamp (A20 variant, "clamp only when the stabilizer is off")
      w1 = w1 < lb ? lb : w1;
      w1 = w1 > ub ? ub : w1;
    }
    wf[e] = w1;
  }
}

int stdp_launch(float* w, int F, int C, int KH, int KW, const uint8_t* lat_in, int H, int W, int pad,
                const uint8_t* lat_out, int Ho, int Wo, const int32_t* winners, const int32_t* count, int k,
                float a_plus, float a_minus, float lb, float ub, int stabilizer, const float* reward,
                int f0, int sharded, cudaStream_t s) {
  if (k == 0) return SNN_OK;
  // one CTA per (winner, slice of 256 synapses): a large kernel (C4: 5,780 synapses) is updated by many
  // SMs at once instead of one CTA looping over it
  const int R = C * KH * KW;
  int slices = int(ceil_div(R, 256));
  if (slices > 64) slices = 64;
  launch_k(stdp_kernel, dim3(dim3(k, slices)), dim3(256), 0, s, w, C, KH, KW, lat_in, H, W, pad, lat_out, Ho, Wo, winners, count, a_plus, a_minus,
                                lb, ub, stabilizer, reward, f0, F, sharded, error_word_ptr(s));
  note_launch();
  return check_launch("snn_stdp_update");
}

}  // namespace snn
