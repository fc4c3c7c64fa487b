// common.cuh -- shared device helpers of libsnn (sm_100a).  Product code; never includes oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/snn.h"

namespace snn {

constexpr uint8_t kNoSpike = SNN_NO_SPIKE;

// Device error word (bit 0 = inexact weight), defined in conv_fire.cu (the only device writer);
// read and cleared by snn_sync_status() through read_clear_error_word().
constexpr int kErrInexact = 1;
constexpr int kErrInternal = 2;  // a kernel's internal consistency trap fired (a library bug)
constexpr int kErrWinner = 4;    // snn_stdp_update: a winner outside the map / the layer (skipped)
int read_clear_error_word(cudaStream_t s, int* word);
int* error_word_ptr(cudaStream_t s);  // device address of the stream's error word (current device)
__device__ __forceinline__ void flag_error(int* err, int bit) { atomicOr(err, bit); }

// Host-side error reporting (thread-local message), defined in api.cu.
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
int num_sms();  // multiprocessor count of the current device (cached per device)
void note_launch(int n = 1);  // diagnostic kernel-launch counter (snn_launch_count)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Device bounds checks of the checked build (python -m paper_1903_02440_b200.build --checked ->
// libsnn_checked.so, run by tools/gpu_checked.sh): an index outside its buffer prints the condition
// and traps the launch.  Compiled out of the product library.  (Stands in for compute-sanitizer,
// which is closed on this GPU pool.)
#ifdef SNN_CHECKED
#define SNN_DCHECK(cond)                                                                         \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("SNN_CHECKED %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,         \
             int(blockIdx.x), int(threadIdx.x));                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define SNN_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// Total-order key of a float (ascending order of value), then complemented by callers that want
// descending order.  v >= 0 for every potential this library produces.
__device__ __forceinline__ uint32_t ordered_bits(float v) {
  uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Candidate key used by pooling ties, inhibition and k-WTA (R13/R14):
// ascending key = (lat ascending, v descending, idx ascending); idx < 2^24.
__device__ __forceinline__ uint64_t wta_key(uint8_t lat, float v, uint32_t idx) {
  return (uint64_t(lat) << 56) | (uint64_t(~ordered_bits(v)) << 24) | uint64_t(idx & 0xFFFFFFu);
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y < x ? y : x;
  }
  return x;
}

// Programmatic dependent launch: every chained kernel first waits for its predecessor grid (so no
// read or write can race it), then lets its own dependent start launching; launches go through
// launch_k with the programmatic-serialization attribute (SNN_PDL=0 turns it off).  Without the
// attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Large resident kernels (the walk and the sort, one CTA per SM with most of the shared memory) only
// wait: letting their dependents launch early would park waiting CTAs next to them (C5: -1.6 %).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// Exact fixed-point potential (units of 2^-31) -> fp32, round to nearest (N1).
__device__ __forceinline__ float fixed_to_float(int64_t acc) {
  return __ll2float_rn(acc) * 4.656612873077392578125e-10f;  // 2^-31, exact scaling
}

}  // namespace snn
