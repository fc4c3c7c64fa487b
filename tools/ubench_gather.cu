// Microbenchmark (tools only, not product code): throughput of the walk's shared-memory weight
// gather on one B200 -- every lane reads VEC*4 contiguous bytes of a row chosen by a warp-uniform
// list entry, rows of 32*VEC*4 bytes (conflict-free), sums them in 32 bits.  Reports wavefronts per
// clock per SM (128 B per wavefront) for several warp counts and gathers in flight per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_gather.cu && /tmp/ubench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

template <int VEC> struct V;
template <> struct V<1> { static __device__ __forceinline__ uint32_t ld(uint32_t a) { uint32_t x; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a)); return x; } };
template <> struct V<2> { static __device__ __forceinline__ uint32_t ld(uint32_t a) { uint32_t x, y; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a)); return x + y; } };
template <> struct V<4> { static __device__ __forceinline__ uint32_t ld(uint32_t a) { uint32_t x, y, z, w; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a)); return (x + y) + (z + w); } };

constexpr int kRows = 256;
template <int VEC, int UNR, bool UNIF>
__global__ void gather(int iters, uint32_t* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int rb = 32 * VEC * 4;
  uint32_t* w = reinterpret_cast<uint32_t*>(sm);
  uint32_t* ent = reinterpret_cast<uint32_t*>(sm + kRows * rb);  // 4096 entries
  for (int i = threadIdx.x; i < kRows * rb / 4; i += blockDim.x) w[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) ent[i] = ((i * 40503u) % kRows) * rb;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t base;
  asm volatile("mov.u32 %0, %1;" : "=r"(base) : "r"((uint32_t)__cvta_generic_to_shared(sm + lane * VEC * 4)));
  const uint32_t ebase = (uint32_t)__cvta_generic_to_shared(ent);
  uint32_t acc = 0;
  long long t0 = clock64();
  int e = (warp * 96) & 4092;
  for (int it = 0; it < iters; ++it) {
    uint32_t off[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u += 4) {
      uint4 q;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(ebase + ((e + u) & 4095) * 4));
      off[u] = q.x; off[u + 1] = q.y; off[u + 2] = q.z; off[u + 3] = q.w;
    }
    uint32_t s = 0;
#pragma unroll
    for (int u = 0; u < UNR; ++u) s += V<VEC>::ld(base + off[u]);
    acc += s;
    e = (e + UNR) & 4092;
  }
  long long t1 = clock64();
  if (acc == 0x12345) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// walk-like: blocks of 8 LDS.128 gathers, 32-bit block sums per feature, 64-bit accumulators, a
// threshold test and one warp vote per block (the fast path of walk_block)
template <int MODE>
__global__ void walkish(int iters, uint32_t* out, long long* cyc, long long thr) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int rb = 512;
  uint32_t* w = reinterpret_cast<uint32_t*>(sm);
  uint32_t* ent = reinterpret_cast<uint32_t*>(sm + kRows * rb);
  for (int i = threadIdx.x; i < kRows * rb / 4; i += blockDim.x) w[i] = (i * 2654435761u) >> 8;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) ent[i] = ((i * 40503u) % kRows) * rb;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t base;
  asm volatile("mov.u32 %0, %1;" : "=r"(base) : "r"((uint32_t)__cvta_generic_to_shared(sm + lane * 16)));
  const uint32_t ebase = (uint32_t)__cvta_generic_to_shared(ent);
  unsigned long long acc[4] = {0, 0, 0, 0};
  int fired = 0;
  long long t0 = clock64();
  int e = (warp * 96) & 4092;
  for (int it = 0; it < iters; ++it) {
    uint4 q0, q1;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w) : "r"(ebase + e * 4));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w) : "r"(ebase + e * 4 + 16));
    const uint32_t off[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    uint32_t wv[8][4];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(wv[k][0]), "=r"(wv[k][1]), "=r"(wv[k][2]), "=r"(wv[k][3]) : "r"(base + off[k]));
    bool hit = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t b = ((wv[0][j] + wv[1][j]) + (wv[2][j] + wv[3][j])) + ((wv[4][j] + wv[5][j]) + (wv[6][j] + wv[7][j]));
      acc[j] += b;
      hit |= (long long)acc[j] > thr;
    }
    if (MODE >= 1) {
      if (__ballot_sync(0xffffffffu, hit)) { fired++; acc[0] = 0; }
    } else {
      fired += hit;
    }
    e = (e + 8) & 4088;
  }
  long long t1 = clock64();
  if (fired == 0x12345 || acc[1] + acc[2] + acc[3] == 7) out[0] = fired;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void runw(int warps) {
  const int smem = kRows * 512 + 4096 * 4;
  auto k = walkish<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<<<148, warps * 32, smem>>>(iters, out, cyc, 1ll << 40);
  k<<<148, warps * 32, smem>>>(iters, out, cyc, 1ll << 40);
  cudaDeviceSynchronize();
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); exit(1); }
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double wf = double(iters) * 8 * warps * 4;
  printf("walkish MODE %d warps %2d: gather wavefronts/clk/SM %.3f\n", MODE, warps, wf / double(c[0]));
  cudaFree(out); cudaFree(cyc);
}

template <int VEC, int UNR>
void run(int warps) {
  const int rb = 32 * VEC * 4;
  const int smem = kRows * rb + 4096 * 4;
  auto k = gather<VEC, UNR, true>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096 / UNR * 8;
  k<<<148, warps * 32, smem>>>(iters, out, cyc);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, warps * 32, smem>>>(iters, out, cyc);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); exit(1); }
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double wf = double(iters) * UNR * warps * VEC;  // wavefronts per SM (VEC wavefronts per warp-gather)
  double wfe = double(iters) * (UNR / 4) * warps;    // entry loads (1 wavefront each, broadcast)
  printf("VEC %d UNR %2d warps %2d: %.3f ms  gather wavefronts/clk/SM %.3f (+entries %.3f)  err=%s\n", VEC, UNR, warps, ms,
         wf / double(c[0]), wfe / double(c[0]), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int n = 0; cudaError_t e0 = cudaGetDeviceCount(&n); printf("devices %d %s\n", n, cudaGetErrorString(e0));
  for (int w : {8, 16, 24, 32}) { run<4, 8>(w); runw<0>(w); runw<1>(w); }
  return 0;
}
