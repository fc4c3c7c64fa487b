// events.cu -- synaptic-event counters for the throughput metric (off the hot path).
// One warp per output position: a per-warp histogram of the receptive field's spike times, its
// prefix over t, then per feature the number of inputs that spiked at or before the neuron's own
// first spike (all spiking inputs if it never fired).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace snn {

__global__ void __launch_bounds__(256) count_events_kernel(const uint8_t* __restrict__ lat_in, int B, int C, int H,
                                                           int W, int pad, int F, int KH, int KW, int T, int Ho,
                                                           int Wo, const uint8_t* __restrict__ lat_out,
                                                           unsigned long long* __restrict__ out) {
  pdl_begin();
  extern __shared__ uint32_t hist[];  // [warps][T + 1]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  uint32_t* h = hist + warp * (T + 1);
  const int64_t HoWo = int64_t(Ho) * Wo, npos = int64_t(B) * HoWo;
  const int KK = KH * KW, R = C * KK;
  unsigned long long paper = 0, need = 0;
  for (int64_t p = int64_t(blockIdx.x) * nwarps + warp; p < npos; p += int64_t(gridDim.x) * nwarps) {
    const int b = int(p / HoWo);
    const int rem = int(p - int64_t(b) * HoWo);
    const int y = rem / Wo, x = rem - (rem / Wo) * Wo;
    for (int t = lane; t <= T; t += 32) h[t] = 0;
    __syncwarp();
    for (int e = lane; e < R; e += 32) {
      const int c = e / KK, r = e - c * KK, ky = r / KW, kx = r - ky * KW;
      const int yy = y + ky - pad, xx = x + kx - pad;
      if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
      const uint8_t l = lat_in[((int64_t(b) * C + c) * H + yy) * W + xx];
      if (l < T) atomicAdd(&h[l], 1u);
    }
    __syncwarp();
    if (lane == 0) {  // inclusive prefix over t; h[T] = total spiking inputs
      uint32_t run = 0;
      for (int t = 0; t < T; ++t) { run += h[t]; h[t] = run; }
      h[T] = run;
    }
    __syncwarp();
    const uint32_t total = h[T];
    if (lane == 0) paper += (unsigned long long)total * F;
    if (lat_out)
      for (int f = lane; f < F; f += 32) {
        const uint8_t lo = lat_out[(int64_t(b) * F + f) * HoWo + rem];
        need += lo < T ? h[lo] : total;
      }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) {
    paper += __shfl_xor_sync(0xffffffffu, paper, o);
    need += __shfl_xor_sync(0xffffffffu, need, o);
  }
  if (lane == 0) {
    atomicAdd(&out[0], paper);
    atomicAdd(&out[1], need);
  }
}

int count_events_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                        const uint8_t* lat_out, unsigned long long* out, cudaStream_t s) {
  if (cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess) return check_launch("snn_count_events");
  const int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
  const int64_t npos = int64_t(B) * Ho * Wo;
  if (npos == 0) return SNN_OK;
  int64_t blocks = ceil_div(npos, 8);
  if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
  launch_k(count_events_kernel, dim3(int(blocks)), dim3(256), 8 * (T + 1) * sizeof(uint32_t), s, lat_in, B, C, H, W, pad, F, KH, KW, T,
                                                                                Ho, Wo, lat_out, out);
  note_launch();
  return check_launch("snn_count_events");
}

}  // namespace snn
