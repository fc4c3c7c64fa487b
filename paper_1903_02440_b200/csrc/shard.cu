// shard.cu -- f4: feature-sharded plasticity across GPUs.
//
// Each rank owns a contiguous slice of the features.  Pointwise inhibition (R13/R14) keeps,
// at every position, the feature with the minimum key (lat asc, v desc, f asc); that minimum over
// ALL features is the minimum over ranks of each rank's own minimum, so one all-reduce(MIN) of a
// packed 63-bit key per position is the only exchange (NCCL, int64).  k-WTA (R15) then runs
// identically on every rank on the reduced key map -- after inhibition a position holds at most one
// candidate -- and every rank applies STDP (Eq. 4) to the winners it owns.
//
// Position key (int64, non-negative, so a signed MIN reduces it):
//   bits 55..62 lat (0..253), bits 23..54 ~ordered_bits(v), bits 0..22 the global feature index;
//   SNN_KEY_NONE = INT64_MAX when no feature of the position spikes.
#include "common.cuh"

namespace snn {
namespace {

constexpr int kKeyThreads = 256;
constexpr int kWtaThreads = 512;

__device__ __forceinline__ int64_t pos_key(uint8_t lat, float v, int f) {
  return int64_t((uint64_t(lat) << 55) | (uint64_t(~ordered_bits(v)) << 23) | uint64_t(f));
}

// One thread per (image, position): the minimum key over the rank's F features (coalesced along the
// position index for every feature plane).
__global__ void __launch_bounds__(kKeyThreads) position_keys_kernel(const uint8_t* __restrict__ lat,
                                                                    const float* __restrict__ v, int64_t B, int F,
                                                                    int HW, int f0, int64_t* __restrict__ keys) {
  pdl_begin();
  const int64_t total = B * HW;
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < total; o += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = o / HW;
    const int p = int(o - b * HW);
    const uint8_t* lb = lat + b * F * HW + p;
    const float* vb = v + b * F * HW + p;
    int64_t best = INT64_MAX;
    for (int f = 0; f < F; ++f) {
      const uint8_t l = lb[int64_t(f) * HW];
      if (l == kNoSpike) continue;
      const int64_t k = pos_key(l, vb[int64_t(f) * HW], f0 + f);
      best = k < best ? k : best;
    }
    keys[o] = best;
  }
}

// One CTA per image: k rounds over the inhibited map.  Candidate order = the k-WTA key (lat asc,
// v desc, flat index f*H*W + p asc) rebuilt from the position key; a winner removes its feature and
// every position within Chebyshev distance r (R15).  The map lives in shared memory when it fits,
// else in the workspace.
__global__ void __launch_bounds__(kWtaThreads) k_winners_keys_kernel(const int64_t* __restrict__ keys, int H, int W,
                                                                     int k, int r, uint64_t* __restrict__ scratch,
                                                                     int use_smem, int32_t* __restrict__ winners,
                                                                     int32_t* __restrict__ count) {
  pdl_begin();
  extern __shared__ uint64_t skey[];
  __shared__ uint64_t red[kWtaThreads / 32];
  const int b = blockIdx.x, HW = H * W;
  uint64_t* kk = use_smem ? skey : scratch + int64_t(b) * HW;
  const int64_t* kb = keys + int64_t(b) * HW;
  for (int p = threadIdx.x; p < HW; p += kWtaThreads) {
    const int64_t pk = kb[p];
    if (pk == INT64_MAX) { kk[p] = ~uint64_t(0); continue; }
    const uint64_t f = uint64_t(pk) & 0x7FFFFFu;
    kk[p] = ((uint64_t(pk) >> 23) << 24) | (f * uint64_t(HW) + uint64_t(p));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int n = 0;
  for (; n < k; ++n) {
    uint64_t best = ~uint64_t(0);
    for (int p = threadIdx.x; p < HW; p += kWtaThreads) best = kk[p] < best ? kk[p] : best;
    best = warp_min_u64(best);
    if (lane == 0) red[wid] = best;
    __syncthreads();
    best = lane < kWtaThreads / 32 ? red[lane] : ~uint64_t(0);
    best = warp_min_u64(best);  // every warp reduces the same partials: a block-uniform result
    if (best == ~uint64_t(0)) break;
    const int idx = int(best & 0xFFFFFFu), f = idx / HW, p = idx - f * HW, y = p / W, x = p - y * W;
    if (threadIdx.x == 0) {
      winners[(int64_t(b) * k + n) * 3 + 0] = f;
      winners[(int64_t(b) * k + n) * 3 + 1] = y;
      winners[(int64_t(b) * k + n) * 3 + 2] = x;
    }
    for (int q = threadIdx.x; q < HW; q += kWtaThreads) {
      const uint64_t c = kk[q];
      if (c == ~uint64_t(0)) continue;
      const int qy = q / W, qx = q - qy * W;
      const bool same_f = int((c & 0xFFFFFFu) / uint64_t(HW)) == f;
      if (same_f || (abs(qy - y) <= r && abs(qx - x) <= r)) kk[q] = ~uint64_t(0);
    }
    __syncthreads();
  }
  for (int i = n + int(threadIdx.x); i < k; i += kWtaThreads) {  // -1 padding of the unused slots
    winners[(int64_t(b) * k + i) * 3 + 0] = -1;
    winners[(int64_t(b) * k + i) * 3 + 1] = -1;
    winners[(int64_t(b) * k + i) * 3 + 2] = -1;
  }
  if (threadIdx.x == 0) count[b] = n;
}

}  // namespace

int position_keys_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, int f0, int64_t* keys,
                         cudaStream_t s) {
  const int64_t total = int64_t(B) * H * W;
  int64_t blocks = ceil_div(total, kKeyThreads);
  if (blocks > int64_t(num_sms()) * 16) blocks = int64_t(num_sms()) * 16;
  launch_k(position_keys_kernel, dim3(unsigned(blocks)), dim3(kKeyThreads), 0, s, lat, v, B, F, H * W, f0, keys);
  note_launch();
  return check_launch("snn_position_keys");
}

size_t k_winners_keys_workspace(int B, int H, int W) { return size_t(B) * H * W * sizeof(uint64_t) + 256; }

int k_winners_keys_launch(const int64_t* keys, int B, int H, int W, int k, int r, int32_t* winners, int32_t* count,
                          void* ws, size_t ws_bytes, cudaStream_t s) {
  const size_t smem = size_t(H) * W * sizeof(uint64_t);
  const int use_smem = smem <= 200 * 1024;
  if (!use_smem && ws_bytes < k_winners_keys_workspace(B, H, W))
    return set_error(SNN_EWORKSPACE, "snn_k_winners_keys: workspace %zu < %zu bytes", ws_bytes,
                     k_winners_keys_workspace(B, H, W));
  const size_t dyn = use_smem ? smem : 0;
  if (dyn > 48 * 1024 &&
      cudaFuncSetAttribute(k_winners_keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn)) != cudaSuccess)
    return set_error(SNN_ECUDA, "snn_k_winners_keys: cannot opt in to %zu B of shared memory", dyn);
  launch_k(k_winners_keys_kernel, dim3(B), dim3(kWtaThreads), dyn, s, keys, H, W, k, r, static_cast<uint64_t*>(ws), use_smem, winners,
                                                    count);
  note_launch();
  return check_launch("snn_k_winners_keys");
}

}  // namespace snn
