// encode.cu -- a1: intensity -> latency rank-order encoding (R1/R2, K1).
//
// Per image, the N positive intensities are ranked by the unique 55-bit key
//     K = ((0x7FFFFFFF - bits(x)) << 24) | flat_index          (x > 0, flat_index < 2^24)
// whose ascending order is (value descending, index ascending).  Bin b (b = 1..T-1) starts at rank
// start_b = b*q + min(b, m).  Instead of sorting, an MSB radix SELECT finds, for every cut b, the key
// prefix of the element of rank start_b; every element's latency is then the number of cuts whose
// prefix it reaches: lat = #{b : (K >> shift_b) >= prefix_b}.  Large images: two levels (12 + 8 bits,
// per-image histograms; level 1 in shared memory), then pass 3 writes every element's latency except
// those sharing a still unresolved cut's 20-bit prefix (the candidates, a few thousand per image),
// which one CTA per image sorts by key to place the cuts exactly (enc_finish_kernel).  Three reads of
// x in all.  An image with more than kEncCandCap candidates (heavy ties) takes levels 2-4 (12/12/11
// bits) and the full assign instead, gated on the device.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace snn {

constexpr int kEncLevels = 5;
constexpr int kEncBins = 4096;
// level 1 takes 8 bits so that its histograms (one per unresolved prefix) fit shared memory
__constant__ int c_enc_bits[kEncLevels] = {12, 8, 12, 12, 11};
__constant__ int c_enc_shift[kEncLevels] = {43, 35, 23, 11, 0};  // prefix after level L = K >> shift[L]
constexpr int kEncL1Bins = 256, kEncL1MaxSlots = 32;
// pass-3 tables per image: lat0[4096] (cuts passed by every key of a level-0 digit, 0xFF = depends on
// the level-1 digit), slot0[4096] (that digit's row in lat1, 0xFF = none), lat1[32][256] (cuts passed by
// every key of a 20-bit prefix, 0xFF = a still unresolved cut's prefix: a candidate)
constexpr int kEncTabBytes = 4096 + 4096 + kEncL1MaxSlots * kEncL1Bins;
constexpr int kEncThreads = 256;
constexpr int kEncPerThread = 16;
constexpr int kEncChunk = kEncThreads * kEncPerThread;
constexpr int kEncCandCap = 8192;  // candidates per image after level 1 (20-bit prefixes; U(0,1) data: ~4K)

struct EncodeWS {
  uint32_t* hist0;      // [G][4096]
  uint32_t* hist;       // [G][S][4096]   S = T (>= the number of cuts)
  uint64_t* cut_prefix; // [G][S]
  int32_t* cut_shift;   // [G][S]  -1 = empty cut (never passed); >=0 when resolved
  uint32_t* cut_resid;  // [G][S]
  int32_t* cut_slot;    // [G][S]  slot of an unresolved cut, -1 when resolved / empty
  uint64_t* slot_prefix;// [G][S]
  int32_t* n_slots;     // [G]
  uint64_t* cand;       // [G][kEncCandCap] keys of the elements whose 20-bit prefix is an unresolved cut's
  int32_t* ncand;       // [G] candidate count (may exceed the capacity: overflow -> the full-level fallback)
  int32_t* ovf;         // [G] 1 = the image takes the level 2-4 fallback
  uint8_t* tab;         // [G][kEncTabBytes] pass-3 tables (enc_build_tables): lat0, slot0, lat1
  int32_t* tabok;       // [G] the tables are valid (at most kEncL1MaxSlots level-0 cut digits)
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t encode_ws_layout(int G, int T, EncodeWS* ws, char* base) {
  int S = T, NC = S;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return base ? base + o : nullptr; };
  EncodeWS w;
  w.hist0 = (uint32_t*)take(sizeof(uint32_t) * size_t(G) * kEncBins);
  w.hist = (uint32_t*)take(sizeof(uint32_t) * size_t(G) * S * kEncBins);
  w.cut_prefix = (uint64_t*)take(sizeof(uint64_t) * size_t(G) * NC);
  w.cut_shift = (int32_t*)take(sizeof(int32_t) * size_t(G) * NC);
  w.cut_resid = (uint32_t*)take(sizeof(uint32_t) * size_t(G) * NC);
  w.cut_slot = (int32_t*)take(sizeof(int32_t) * size_t(G) * NC);
  w.slot_prefix = (uint64_t*)take(sizeof(uint64_t) * size_t(G) * S);
  w.n_slots = (int32_t*)take(sizeof(int32_t) * size_t(G));
  w.cand = (uint64_t*)take(sizeof(uint64_t) * size_t(G) * kEncCandCap);
  w.ncand = (int32_t*)take(sizeof(int32_t) * size_t(G));
  w.ovf = (int32_t*)take(sizeof(int32_t) * size_t(G));
  w.tab = (uint8_t*)take(size_t(G) * kEncTabBytes);
  w.tabok = (int32_t*)take(sizeof(int32_t) * size_t(G));
  if (ws) *ws = w;
  return off;
}

// Group size: whole batch unless the per-image histograms exceed ~256 MB.
static int encode_group(int B, int T) {
  size_t per = encode_ws_layout(1, T, nullptr, nullptr);
  size_t g = (size_t(256) << 20) / (per ? per : 1);
  if (g < 1) g = 1;
  return int(g < size_t(B) ? g : size_t(B));
}

size_t encode_workspace(int B, int C, int H, int W, int T) {
  (void)C; (void)H; (void)W;
  if (B <= 0) return 256;
  return encode_ws_layout(encode_group(B, T), T, nullptr, nullptr);
}

__device__ __forceinline__ uint64_t enc_key(float x, uint32_t idx) {
  return (uint64_t(0x7FFFFFFFu - __float_as_uint(x)) << 24) | idx;
}

// Number of cuts and the rank at which bin b (b = 1..ncuts) starts, per bin-size rule (snn_encode_ex):
// 0 (R1) q + 1 ranks for the first N % T bins, q for the rest; 1 proportional, bin = floor(r T / N);
// 2 floor, q ranks per bin and a T-th cut at T q past which nothing spikes (lat = T -> no spike).
__host__ __device__ __forceinline__ int enc_ncuts(int T, int bins) { return T - 1 + (bins == 2 ? 1 : 0); }
__device__ __forceinline__ uint32_t enc_cut_start(uint32_t b, uint32_t N, uint32_t T, int bins) {
  const uint32_t q = N / T, m = N % T;
  if (bins == 1) return uint32_t((uint64_t(b) * N + T - 1) / T);
  if (bins == 2) return b * q;
  return b * q + (b < m ? b : m);
}

// The 16 elements of a thread's share of a 4096-element chunk: element 4 (j kEncThreads + tid) + u of the
// chunk in v[4 j + u] (j, u < 4), loaded as four float4 (vec: every image 16-byte aligned, n % 4 == 0)
// or element by element; all loads issued before any use.  Out of range: 0 (never positive).
__device__ __forceinline__ void enc_load16(const float* __restrict__ xg, int64_t n, int64_t base, bool vec,
                                           float (&v)[16]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = base + 4 * (int64_t(j) * kEncThreads + tid);
    if (vec && i + 3 < n) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(xg + i));
      v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[4 * j + u] = (i + u < n) ? __ldg(xg + i + u) : 0.0f;
    }
  }
}
__device__ __forceinline__ int64_t enc_elem(int64_t base, int k) {
  return base + 4 * (int64_t(k >> 2) * kEncThreads + threadIdx.x) + (k & 3);
}

// Level 0: histogram of the top 12 bits of every positive key (all images of the group).  A CTA walks
// several 4096-element chunks of its image (grid-stride), counting in one shared histogram with plain
// shared atomics, then adds its non-zero bins to the image's histogram once.
__global__ void __launch_bounds__(kEncThreads) enc_hist0_kernel(const float* __restrict__ x, int64_t n, bool vec,
                                                                 EncodeWS ws) {
  pdl_begin();
  __shared__ uint32_t sh[kEncBins];
  for (int i = threadIdx.x; i < kEncBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int g = blockIdx.y;
  const float* xg = x + int64_t(g) * n;
  const int64_t nch = (n + kEncChunk - 1) / kEncChunk;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    float v[16];
    enc_load16(xg, n, ch * kEncChunk, vec, v);
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (v[k] > 0.0f) atomicAdd(&sh[(0x7FFFFFFFu - __float_as_uint(v[k])) >> 19], 1u);  // key bits 54..43
  }
  __syncthreads();
  uint32_t* hg = ws.hist0 + int64_t(g) * kEncBins;
  for (int i = threadIdx.x; i < kEncBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hg[i], sh[i]);
}

// Sorted unresolved prefixes of image g in shared memory (sp) and a 4096-bit mask of their low 12 bits.
__device__ __forceinline__ int enc_slots_smem(const EncodeWS& ws, int g, int S, uint64_t* sp, uint32_t* dmask) {
  const int ns = ws.n_slots[g];
  for (int i = threadIdx.x; i < kEncBins / 32; i += blockDim.x) dmask[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const uint64_t q = ws.slot_prefix[int64_t(g) * S + i];
    sp[i] = q;
    atomicOr(&dmask[uint32_t(q >> 5) & (kEncBins / 32 - 1)], 1u << (uint32_t(q) & 31));
  }
  __syncthreads();
  return ns;
}
// Slot of prefix p (lower bound in the sorted sp), or -1.
__device__ __forceinline__ int enc_slot_of(uint64_t p, const uint64_t* sp, const uint32_t* dmask, int ns) {
  const uint32_t dg = uint32_t(p) & (kEncBins - 1);  // a 12-bit digit: most elements leave here
  if (!(dmask[dg >> 5] >> (dg & 31) & 1)) return -1;
  int lo = 0, hi = ns;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sp[mid] < p) lo = mid + 1; else hi = mid;
  }
  return (lo < ns && sp[lo] == p) ? lo : -1;
}

// Levels 1..4: histogram of the next digit for elements whose prefix matches an unresolved cut.
// gate != NULL: only images with gate[g] != 0 (the fallback levels of overflowed images).
__global__ void __launch_bounds__(kEncThreads) enc_hist_kernel(const float* __restrict__ x, int64_t n, bool vec, int T,
                                                                int level, EncodeWS ws, const int32_t* gate) {
  pdl_begin();
  const int g = blockIdx.y;
  if (gate && !gate[g]) return;
  const int S = T;
  if (ws.n_slots[g] == 0) return;
  __shared__ uint64_t sp[256];
  __shared__ uint32_t dmask[kEncBins / 32];  // previous-level digits of the unresolved prefixes
  const int ns = enc_slots_smem(ws, g, S, sp, dmask);
  const int shp = c_enc_shift[level - 1], sh = c_enc_shift[level];
  const uint64_t mask = (uint64_t(1) << c_enc_bits[level]) - 1;
  const float* xg = x + int64_t(g) * n;
  uint32_t* hg = ws.hist + int64_t(g) * S * kEncBins;
  // level 1 (8-bit digits, at most kEncL1MaxSlots prefixes): the CTA counts in shared memory and adds
  // its non-zero bins to the image's histograms once; otherwise one global atomic per element
  extern __shared__ uint32_t hs[];  // [ns][kEncL1Bins] (dynamic, level 1 only)
  const bool sm = level == 1 && ns <= kEncL1MaxSlots;
  __shared__ uint8_t slot_of[kEncBins];  // level 1: a level-0 digit's slot (the prefixes are the digits)
  if (sm) {
    for (int i = threadIdx.x; i < ns * kEncL1Bins; i += blockDim.x) hs[i] = 0;
    for (int i = threadIdx.x; i < kEncBins; i += blockDim.x) slot_of[i] = 0xFF;
    __syncthreads();
    for (int i = threadIdx.x; i < ns; i += blockDim.x) slot_of[uint32_t(sp[i]) & (kEncBins - 1)] = uint8_t(i);
    __syncthreads();
  }
  const int64_t nch = (n + kEncChunk - 1) / kEncChunk;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {  // grid-stride over the image's chunks
    const int64_t base = ch * kEncChunk;
    float v[16];
    enc_load16(xg, n, base, vec, v);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (!(v[k] > 0.0f)) continue;
      const uint64_t K = enc_key(v[k], uint32_t(enc_elem(base, k)));
      int sl;
      if (sm) {
        const uint32_t s8 = slot_of[uint32_t(K >> shp)];  // K >> 43: exactly the 12-bit level-0 digit
        sl = s8 == 0xFF ? -1 : int(s8);
      } else {
        sl = enc_slot_of(K >> shp, sp, dmask, ns);
      }
      if (sl < 0) continue;
      const uint32_t dg = uint32_t((K >> sh) & mask);
      if (sm) atomicAdd(&hs[sl * kEncL1Bins + dg], 1u);
      else atomicAdd(&hg[int64_t(sl) * kEncBins + dg], 1u);
    }
  }
  if (sm) {
    __syncthreads();
    for (int i = threadIdx.x; i < ns * kEncL1Bins; i += blockDim.x)
      if (hs[i]) atomicAdd(&hg[int64_t(i / kEncL1Bins) * kEncBins + (i % kEncL1Bins)], hs[i]);
  }
}

// Per-image selection after level L: locate every unresolved cut's digit (one warp per cut: the slot's
// 4096-bin histogram scanned as 32 runs of 128 bins), resolve or descend, rebuild the sorted list of
// distinct prefixes for level L+1 and zero their histograms.  gate: as enc_hist_kernel.
__global__ void __launch_bounds__(1024) enc_select_kernel(int T, int bins, int level, EncodeWS ws,
                                                          const int32_t* gate, int zero_next) {
  pdl_begin();
  const int g = blockIdx.x;
  if (gate && !gate[g]) return;
  const int S = T;
  const int NC = enc_ncuts(T, bins);
  __shared__ int s_nslots;
  uint64_t* cp = ws.cut_prefix + int64_t(g) * S;
  int32_t* csh = ws.cut_shift + int64_t(g) * S;
  uint32_t* cr = ws.cut_resid + int64_t(g) * S;
  int32_t* cs = ws.cut_slot + int64_t(g) * S;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (level == 0) {  // initialise the cuts from N = total positives
    __shared__ uint32_t s_n;
    if (wid == 0) {
      const uint4* h4 = reinterpret_cast<const uint4*>(ws.hist0 + int64_t(g) * kEncBins);
      uint32_t sum = 0;
      for (int i = lane; i < kEncBins / 4; i += 32) { const uint4 q = h4[i]; sum += q.x + q.y + q.z + q.w; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) s_n = sum;
    }
    __syncthreads();
    const uint32_t N = s_n;
    for (int b = tid; b < NC; b += blockDim.x) {
      const uint32_t start = enc_cut_start(uint32_t(b + 1), N, uint32_t(T), bins);
      cp[b] = 0;
      if (start >= N) { csh[b] = -1; cs[b] = -1; cr[b] = 0; }
      else { csh[b] = -2; cs[b] = 0; cr[b] = start; }
    }
    __syncthreads();
  }
  for (int b = wid; b < NC; b += nw) {
    const int sl = cs[b];
    if (sl < 0 || csh[b] == -1) continue;  // resolved or empty (warp-uniform)
    const uint32_t* h = (level == 0) ? ws.hist0 + int64_t(g) * kEncBins : ws.hist + (int64_t(g) * S + sl) * kEncBins;
    const uint32_t r = cr[b];
    const int rl = level == 1 ? kEncL1Bins / 32 : 128;  // bins per lane run (level 1: 256 bins in use)
    const uint4* h4 = reinterpret_cast<const uint4*>(h + lane * rl);
    uint32_t run = 0;
#pragma unroll 2
    for (int q = 0; q < rl / 4; ++q) {
      const uint4 x4 = h4[q];
      run += x4.x + x4.y + x4.z + x4.w;
    }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    // the digit holding rank r: the run whose inclusive sum first exceeds r; then the warp loads that
    // run's 128 bins (4 per lane, one 16-byte load each) and finds the digit by a second scan
    const unsigned over = __ballot_sync(0xffffffffu, inc > r);
    const int L = __ffs(over) - 1;  // exists: r < the slot's total
    const uint32_t rbase = __shfl_sync(0xffffffffu, inc - run, L);  // exclusive base of run L
    const uint4 q4 = lane * 4 < rl ? reinterpret_cast<const uint4*>(h + L * rl)[lane] : make_uint4(0, 0, 0, 0);
    const uint32_t s4 = q4.x + q4.y + q4.z + q4.w;
    uint32_t inc2 = s4;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc2, o);
      if (lane >= o) inc2 += y;
    }
    const unsigned over2 = __ballot_sync(0xffffffffu, rbase + inc2 > r);
    const int L2 = __ffs(over2) - 1;
    if (lane == L2) {
      uint32_t c = rbase + inc2 - s4;  // exclusive base of these 4 bins
      const uint32_t hb[4] = {q4.x, q4.y, q4.z, q4.w};
      int d = 0;
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (cnt == 0 && c + hb[k] > r) { d = L2 * 4 + k; cnt = hb[k]; }
        else if (cnt == 0) c += hb[k];
      }
      const int dig = L * rl + d;
      cp[b] = (cp[b] << c_enc_bits[level]) | uint64_t(dig);
      cr[b] = r - c;
      if (cnt == 1 || level == kEncLevels - 1) { csh[b] = c_enc_shift[level]; cs[b] = -1; }
      else cs[b] = -3;  // unresolved, slot assigned below
    }
  }
  __syncthreads();
  // rebuild slots for the next level: cuts are in rank order, so their prefixes are sorted
  if (tid == 0) {
    int n = 0;
    uint64_t* spg = ws.slot_prefix + int64_t(g) * S;
    for (int b = 0; b < NC; ++b) {
      if (cs[b] != -3) continue;
      if (n == 0 || spg[n - 1] != cp[b]) spg[n++] = cp[b];
      cs[b] = n - 1;
    }
    ws.n_slots[g] = n;
    s_nslots = n;
  }
  __syncthreads();
  // zero the next level's histograms: level 1 uses 256 bins per slot; the level-2 histograms are needed
  // only by the gated fallback, whose images enc_finish_kernel zeroes (zero_next = 0 here)
  if (level + 1 < kEncLevels && zero_next) {
    const int nb = level + 1 == 1 ? kEncL1Bins : kEncBins;
    for (int64_t i = tid; i < int64_t(s_nslots) * nb; i += blockDim.x) {
      const int64_t sl = i / nb;
      ws.hist[(int64_t(g) * S + sl) * kEncBins + (i - sl * nb)] = 0;
    }
  }
}

// Output index of flat input element i: planar (hw = 0) or channels-last [H, W, C] (SNN_ENCODE_OUT_NHWC).
struct EncOut {
  int hw, c;
  __device__ __forceinline__ uint32_t idx(uint32_t i) const {
    if (!hw) return i;
    const uint32_t ch = i / uint32_t(hw);
    return (i - ch * uint32_t(hw)) * uint32_t(c) + ch;
  }
};

// The cuts of image g in shared memory for the latency count: sp = prefix, ssh = its shift (-1 = never
// passed).  unres_shift >= 0: cuts still unresolved (after level 1) compare at that shift -- exact for
// every element whose prefix is not theirs (those are the candidates).
__device__ __forceinline__ void enc_cuts_smem(const EncodeWS& ws, int g, int S, int NC, int unres_shift,
                                              uint64_t* sp, int* ssh) {
  for (int b = threadIdx.x; b < NC; b += blockDim.x) {
    sp[b] = ws.cut_prefix[int64_t(g) * S + b];
    const int sh = ws.cut_shift[int64_t(g) * S + b];
    ssh[b] = (sh == -2 && unres_shift >= 0) ? unres_shift : sh;
  }
}
// Number of cuts passed by key K (pass(b) is monotone non-increasing in b).
__device__ __forceinline__ int enc_passed(uint64_t K, const uint64_t* sp, const int* ssh, int NC) {
  int lo = 0, hi = NC;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool pass = ssh[mid] >= 0 && (K >> ssh[mid]) >= sp[mid];
    if (pass) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Fallback assign (all levels resolved): lat = number of cuts whose prefix the key reaches.
__global__ void __launch_bounds__(kEncThreads) enc_assign_kernel(const float* __restrict__ x, int64_t n, int T,
                                                                  int bins, uint8_t* __restrict__ lat, EncodeWS ws,
                                                                  EncOut eo, const int32_t* gate) {
  pdl_begin();
  const int g = blockIdx.y;
  if (gate && !gate[g]) return;
  const int S = T;
  const int NC = enc_ncuts(T, bins);
  __shared__ uint64_t sp[256];
  __shared__ int ssh[256];
  enc_cuts_smem(ws, g, S, NC, -1, sp, ssh);
  __syncthreads();
  const float* xg = x + int64_t(g) * n;
  uint8_t* lg = lat + int64_t(g) * n;
  const int64_t nch = (n + kEncChunk - 1) / kEncChunk;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {  // grid-stride over the image's chunks
    const int64_t base = ch * kEncChunk;
    for (int j = 0; j < kEncPerThread; ++j) {
      int64_t i = base + int64_t(j) * kEncThreads + threadIdx.x;
      if (i >= n) break;
      float v = xg[i];
      uint8_t out = kNoSpike;
      if (v > 0.0f) {
        const int lo = enc_passed(enc_key(v, uint32_t(i)), sp, ssh, NC);
        out = lo >= T ? kNoSpike : uint8_t(lo);
      }
      lg[eo.idx(uint32_t(i))] = out;
    }
  }
}

// Per image after level 1: the pass-3 lookup tables (kEncTabBytes).  A key range (a level-0 digit, or a
// 20-bit prefix) passes cut b entirely, not at all, or either way (ambiguous); a table entry is the number
// of cuts the whole range passes, 0xFF if any cut is ambiguous there.  Cut b compares at its resolved
// shift, a cut still unresolved after level 1 at shift 35 (its 20-bit prefix: ambiguous on that prefix,
// whose elements become candidates).  More than kEncL1MaxSlots ambiguous level-0 digits: tabok = 0 and
// pass 3 searches the cuts per element instead.
// Cuts passed by every key of [kmin, kmax] (cuts are in rank order, so "passed" is monotone in b): all =
// the cuts passed already at kmin (an unresolved cut only strictly above its prefix), any = the cuts
// passed at kmax; all < any: some cut is ambiguous on the range -> 0xFF.
__device__ __forceinline__ int enc_range_lat(uint64_t kmin, uint64_t kmax, const uint64_t* cp, const int* csh, int NC) {
  const int shu = c_enc_shift[1];
  auto count = [&](uint64_t K, bool strict_unres) {
    int lo = 0, hi = NC;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int c = csh[mid];
      bool pass;
      if (c == -1) pass = false;  // empty cut: never passed
      else if (c >= 0) pass = (K >> c) >= cp[mid];
      else pass = strict_unres ? (K >> shu) > cp[mid] : (K >> shu) >= cp[mid];
      if (pass) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int all = count(kmin, true), any = count(kmax, false);
  return any > all ? 0xFF : all;
}
__global__ void __launch_bounds__(1024) enc_tables_kernel(int T, int bins, EncodeWS ws) {
  pdl_begin();
  const int g = blockIdx.x, tid = threadIdx.x;
  const int S = T, NC = enc_ncuts(T, bins);
  __shared__ uint64_t cp[256];
  __shared__ int csh[256];
  __shared__ uint8_t lat0[kEncBins], slot0[kEncBins];
  __shared__ uint16_t dig[kEncL1MaxSlots];
  __shared__ int s_nk;
  for (int b = tid; b < NC; b += blockDim.x) {
    cp[b] = ws.cut_prefix[int64_t(g) * S + b];
    csh[b] = ws.cut_shift[int64_t(g) * S + b];
  }
  __syncthreads();
  const int sh0 = c_enc_shift[0], sh1 = c_enc_shift[1];
  for (int d = tid; d < kEncBins; d += blockDim.x) {
    const uint64_t kmin = uint64_t(d) << sh0, kmax = kmin + ((uint64_t(1) << sh0) - 1);
    lat0[d] = uint8_t(enc_range_lat(kmin, kmax, cp, csh, NC));
  }
  __syncthreads();
  if (tid < 32) {  // the ambiguous level-0 digits in ascending order -> rows of lat1
    int nk = 0;
    for (int d0 = 0; d0 < kEncBins; d0 += 32) {
      const bool a = lat0[d0 + tid] == 0xFF;
      const unsigned m = __ballot_sync(0xffffffffu, a);
      const int k = nk + __popc(m & ((1u << tid) - 1u));
      slot0[d0 + tid] = (a && k < kEncL1MaxSlots) ? uint8_t(k) : 0xFF;
      if (a && k < kEncL1MaxSlots) dig[k] = uint16_t(d0 + tid);
      nk += __popc(m);
    }
    if (tid == 0) s_nk = nk;
  }
  __syncthreads();
  const int nk = s_nk;
  uint8_t* tg = ws.tab + int64_t(g) * kEncTabBytes;
  if (nk > kEncL1MaxSlots) {
    if (tid == 0) ws.tabok[g] = 0;
    return;
  }
  for (int i = tid; i < nk * kEncL1Bins; i += blockDim.x) {
    const int k = i / kEncL1Bins, d1 = i - k * kEncL1Bins;
    const uint64_t kmin = ((uint64_t(dig[k]) << c_enc_bits[1]) | uint64_t(d1)) << sh1;
    const uint64_t kmax = kmin + ((uint64_t(1) << sh1) - 1);
    tg[2 * kEncBins + i] = uint8_t(enc_range_lat(kmin, kmax, cp, csh, NC));
  }
  for (int i = tid; i < kEncBins; i += blockDim.x) { tg[i] = lat0[i]; tg[kEncBins + i] = slot0[i]; }
  if (tid == 0) ws.tabok[g] = 1;
}

// Pass 3 (after level 1): the latency of every element whose 20-bit prefix no unresolved cut shares,
// written in the output layout; the others (candidates, ~200 per U(0,1) image) are appended to the
// image's candidate list for enc_finish_kernel.  Planar output: a 4096-element chunk per CTA, 4
// consecutive latencies per 32-bit store.  Channels-last output (C <= 256): a tile of 128 positions x
// all C channels per CTA (coalesced float4 reads of each channel's 128 positions), transposed in shared
// memory and written as one contiguous 128 C-byte run.
constexpr int kEncTileP = 128;
__device__ __forceinline__ void enc_candidate(const EncodeWS& ws, int g, uint64_t K) {
  const int slot = atomicAdd(&ws.ncand[g], 1);
  if (slot < kEncCandCap) ws.cand[int64_t(g) * kEncCandCap + slot] = K;
}
__global__ void __launch_bounds__(kEncThreads) enc_assign2_kernel(const float* __restrict__ x, int64_t n, bool vec,
                                                                   int T, int bins, uint8_t* __restrict__ lat,
                                                                   EncodeWS ws, EncOut eo) {
  pdl_begin();
  const int g = blockIdx.y;
  const int S = T;
  const int NC = enc_ncuts(T, bins);
  __shared__ uint64_t sp[256], slp[256];
  __shared__ int ssh[256];
  __shared__ uint32_t dmask[kEncBins / 32];
  __shared__ __align__(16) uint8_t tab[kEncTabBytes];
  extern __shared__ __align__(16) uint8_t tile[];  // [kEncTileP * C] (channels-last output only)
  const bool tabok = ws.tabok[g] != 0;
  if (tabok) {
    const uint4* src = reinterpret_cast<const uint4*>(ws.tab + int64_t(g) * kEncTabBytes);
    for (int i = threadIdx.x; i < kEncTabBytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(tab)[i] = src[i];
  }
  enc_cuts_smem(ws, g, S, NC, c_enc_shift[1], sp, ssh);
  const int ns = enc_slots_smem(ws, g, S, slp, dmask);  // (syncs)
  const float* xg = x + int64_t(g) * n;
  uint8_t* lg = lat + int64_t(g) * n;
  const int shp = c_enc_shift[1];
  uint32_t tab_a;  // the tables' shared-window address, kept in a register
  asm volatile("mov.u32 %0, %1;" : "=r"(tab_a) : "r"(smem_u32(tab)));
  auto ld8 = [&](uint32_t off) {
    uint16_t r;
    asm("ld.shared.u8 %0, [%1];" : "=h"(r) : "r"(tab_a + off));
    return uint32_t(r);
  };
  auto lat_of = [&](float v, uint32_t i) -> uint8_t {
    if (!(v > 0.0f)) return kNoSpike;
    int c;
    if (tabok) {  // two table lookups (level-0 digit, then its 20-bit prefix): value bits only (32-bit)
      const uint32_t v31 = 0x7FFFFFFFu - __float_as_uint(v);  // key bits 54..24
      const uint32_t d0 = v31 >> 19;                           // key bits 54..43
      c = int(ld8(d0));
      SNN_DCHECK(d0 < uint32_t(kEncBins));
      if (c == 0xFF) {
        SNN_DCHECK(ld8(kEncBins + d0) < uint32_t(kEncL1MaxSlots));
        c = int(ld8(2 * kEncBins + ld8(kEncBins + d0) * kEncL1Bins + ((v31 >> 11) & 0xFFu)));
      }
      if (c == 0xFF) {
        enc_candidate(ws, g, enc_key(v, i));
        return kNoSpike;  // placeholder, rewritten by enc_finish_kernel
      }
      return c >= T ? kNoSpike : uint8_t(c);
    }
    const uint64_t K = enc_key(v, i);
    {
      if (ns > 0 && enc_slot_of(K >> shp, slp, dmask, ns) >= 0) {
        enc_candidate(ws, g, K);
        return kNoSpike;
      }
      c = enc_passed(K, sp, ssh, NC);
    }
    return c >= T ? kNoSpike : uint8_t(c);
  };
  if (!eo.hw) {
    const int64_t nch = (n + kEncChunk - 1) / kEncChunk;
    for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {  // grid-stride over the image's chunks
      const int64_t base = ch * kEncChunk;
      float v[16];
      enc_load16(xg, n, base, vec, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t i = base + 4 * (int64_t(j) * kEncThreads + threadIdx.x);
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) w |= uint32_t(lat_of(v[4 * j + u], uint32_t(i + u))) << (8 * u);
        if (vec && i + 3 < n) {
          *reinterpret_cast<uint32_t*>(lg + i) = w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i + u < n) lg[i + u] = uint8_t(w >> (8 * u));
        }
      }
    }
    return;
  }
  // channels-last: tiles of positions [p0, p0 + 128) x channels [0, C), grid-stride.  C % 4 == 0 (and a
  // 4-byte aligned output): a lane reads 4 channels at one position (each load coalesced across the
  // warp's 32 positions), packs their latencies in one word and stores it to a tile row padded to an odd
  // word count (conflict-free); the tile then leaves as whole words.  Otherwise byte-wise, rows of C + 1.
  const int HW = eo.hw, C = eo.c;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool w4 = (C % 4 == 0) && (reinterpret_cast<uintptr_t>(lg) & 3) == 0;
  // w4: a warp covers 128 positions of one 4-channel group; with fewer groups than warps the tile grows
  // to 128 x (warps per group) positions so every warp has work (C4: C = 4, 1024-position tiles)
  const int ncg4 = C / 4, nwarp4 = int(blockDim.x >> 5);
  const int wpg = (w4 && ncg4 < nwarp4) ? nwarp4 / ncg4 : 1;
  const int TP = kEncTileP * wpg;
  const int ntiles = (HW + TP - 1) / TP;
  const int rw = w4 ? C / 4 + 1 : 0;                 // tile row stride in words (w4)
  uint32_t* tile32 = reinterpret_cast<uint32_t*>(tile);
  for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int p0 = tl * TP;
    const int np = min(TP, HW - p0);
    if (w4) {
      const int ncg = C / 4, nwarp = blockDim.x >> 5;
      // one warp per 4-channel group: lane l takes positions 4l .. 4l + 3 of the tile, one float4 per
      // channel (vec) -- 16 elements from 4 loads, 4 packed words to the tile
      const bool v4 = vec && (HW % 4 == 0);
      for (int it = wid; it < ncg * wpg; it += nwarp) {
        const int cg = it / wpg, q = (it - cg * wpg) * kEncTileP + lane * 4;
        if (q < np) {
          float v[4][4];  // [channel][position]
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float* src = xg + int64_t(4 * cg + u) * HW + p0 + q;
            if (v4 && q + 3 < np) {
              const float4 f = __ldg(reinterpret_cast<const float4*>(src));
              v[u][0] = f.x; v[u][1] = f.y; v[u][2] = f.z; v[u][3] = f.w;
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) v[u][j] = (q + j < np) ? __ldg(src + j) : 0.0f;
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (q + j < np) {
              uint32_t w = 0;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                w |= uint32_t(lat_of(v[u][j], uint32_t(int64_t(4 * cg + u) * HW + p0 + q + j))) << (8 * u);
              tile32[(q + j) * rw + cg] = w;
            }
          }
        }
      }
      __syncthreads();
      uint32_t* dst = reinterpret_cast<uint32_t*>(lg + int64_t(p0) * C);
      if (int(blockDim.x) % ncg == 0) {  // (position, word) advanced by a constant step: no division per word
        const int wdx = threadIdx.x % ncg, pstep = blockDim.x / ncg;
        for (int p = threadIdx.x / ncg; p < np; p += pstep) dst[p * ncg + wdx] = tile32[p * rw + wdx];
      } else {
        for (int k = threadIdx.x; k < np * ncg; k += blockDim.x) {
          const int p = k / ncg, wdx = k - p * ncg;
          dst[k] = tile32[p * rw + wdx];
        }
      }
    } else {
      for (int it = threadIdx.x; it < C * kEncTileP; it += blockDim.x) {
        const int c = it / kEncTileP, q = it - c * kEncTileP;
        if (q < np) {
          const int64_t i = int64_t(c) * HW + p0 + q;
          tile[q * (C + 1) + c] = lat_of(__ldg(xg + i), uint32_t(i));
        }
      }
      __syncthreads();
      uint8_t* dst = lg + int64_t(p0) * C;
      for (int k = threadIdx.x; k < np * C; k += blockDim.x) {
        const int p = k / C, c = k - p * C;
        dst[k] = tile[p * (C + 1) + c];
      }
    }
    __syncthreads();  // the tile is rewritten by the next iteration
  }
}

// Per image: the candidates of pass 3 sorted by key in shared memory (bitonic), each one's rank j among
// the elements of its 20-bit prefix (all of them are candidates), and its latency: a cut still
// unresolved with that prefix is passed iff j >= the cut's residual rank in the prefix (cut_resid);
// every other cut compares as in pass 3.  More than kEncCandCap candidates: the image is flagged for
// the level 2-4 fallback (ovf) and nothing is written here.
constexpr int kEncFinThreads = 1024;
__global__ void __launch_bounds__(kEncFinThreads) enc_finish_kernel(int T, int bins, uint8_t* __restrict__ lat,
                                                                     int64_t n, EncodeWS ws, EncOut eo) {
  pdl_begin();
  extern __shared__ uint64_t ck[];  // [np2]
  __shared__ uint64_t sp[256];
  __shared__ int ssh[256];
  __shared__ uint32_t cres[256];
  const int g = blockIdx.x, tid = threadIdx.x;
  const int S = T, NC = enc_ncuts(T, bins);
  const int nc = ws.ncand[g];  // (zeroed by the launcher before pass 3)
  if (tid == 0) ws.ovf[g] = nc > kEncCandCap ? 1 : 0;
  if (nc > kEncCandCap) {  // the fallback's level-2 histograms (one per slot of enc_select level 1)
    const int ns = ws.n_slots[g];
    uint4* hg = reinterpret_cast<uint4*>(ws.hist + int64_t(g) * S * kEncBins);
    for (int64_t i = tid; i < int64_t(ns) * kEncBins / 4; i += blockDim.x) hg[i] = make_uint4(0, 0, 0, 0);
    return;
  }
  if (nc == 0) return;
  const int shp = c_enc_shift[1];
  for (int b = tid; b < NC; b += blockDim.x) {
    sp[b] = ws.cut_prefix[int64_t(g) * S + b];
    ssh[b] = ws.cut_shift[int64_t(g) * S + b];  // -2: unresolved at level 1 (prefix at shift shp)
    cres[b] = ws.cut_resid[int64_t(g) * S + b];
  }
  int np2 = 1;
  while (np2 < nc) np2 <<= 1;
  SNN_DCHECK(np2 <= kEncCandCap);
  for (int i = tid; i < np2; i += blockDim.x) ck[i] = i < nc ? ws.cand[int64_t(g) * kEncCandCap + i] : ~uint64_t(0);
  __syncthreads();
  for (int k = 2; k <= np2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < np2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const uint64_t a = ck[i], b = ck[p];
          if (((i & k) == 0) == (a > b)) { ck[i] = b; ck[p] = a; }
        }
      }
      __syncthreads();
    }
  uint8_t* lg = lat + int64_t(g) * n;
  for (int q = tid; q < nc; q += blockDim.x) {
    const uint64_t K = ck[q];
    const uint64_t pfx = K >> shp;
    int lo = 0, hi = q;  // first candidate of this prefix
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((ck[mid] >> shp) < pfx) lo = mid + 1; else hi = mid;
    }
    const uint32_t j = uint32_t(q - lo);
    int a = 0, z = NC;  // cuts passed (monotone)
    while (a < z) {
      const int mid = (a + z) >> 1;
      bool pass;
      if (ssh[mid] == -2) pass = pfx > sp[mid] || (pfx == sp[mid] && j >= cres[mid]);
      else pass = ssh[mid] >= 0 && (K >> ssh[mid]) >= sp[mid];
      if (pass) a = mid + 1; else z = mid;
    }
    lg[eo.idx(uint32_t(K & 0xFFFFFFu))] = a >= T ? kNoSpike : uint8_t(a);
  }
}

// Small images (C*H*W <= 16384, e.g. C1-C3): one CTA per image runs the same radix select with
// everything in shared memory -- the image's 31-bit value keys, a 4096-bin level-0 histogram, then
// 8-bit digit levels with one 256-bin histogram per distinct unresolved cut prefix.  Levels: key bits
// 54..43 (12), then 8, 8, 8, 8, 8 and the last 3 (the index part of the key included).
constexpr int kSmLevels = 7;
__constant__ int c_sm_bits[kSmLevels] = {12, 8, 8, 8, 8, 8, 3};
__constant__ int c_sm_shift[kSmLevels] = {43, 35, 27, 19, 11, 3, 0};
constexpr int kSmThreads = 512;

__device__ __forceinline__ uint64_t sm_key(uint32_t vk, int i) { return (uint64_t(vk) << 24) | uint32_t(i); }

__global__ void __launch_bounds__(kSmThreads) enc_small_kernel(const float* __restrict__ x, int n, int T, int bins,
                                                                uint8_t* __restrict__ lat, EncOut eo) {
  pdl_begin();
  extern __shared__ uint32_t vk[];              // [n] 0x7FFFFFFF - bits(x), or ~0 for x <= 0; then [n] u16 candidates
  uint16_t* cand = reinterpret_cast<uint16_t*>(vk + n);
  __shared__ uint8_t bin_lat[4096];             // level-0 bin -> latency of its elements, 0xFF = a cut inside
  __shared__ int s_ncand;
  __shared__ uint32_t hist[4096];               // level 0: 4096 bins; later: slot * 256 + digit
  __shared__ uint32_t slot_tot[16];
  __shared__ uint64_t cut_prefix[256], slot_prefix[256];
  __shared__ int cut_shift[256], cut_slot[256];
  __shared__ uint32_t cut_resid[256];
  __shared__ int s_nslots, s_N;
  __shared__ uint32_t wsum[kSmThreads / 32];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float* xb = x + int64_t(b) * n;
  uint8_t* lb = lat + int64_t(b) * n;
  const int NC = enc_ncuts(T, bins);
  for (int i = tid; i < 4096; i += kSmThreads) hist[i] = 0;
  __syncthreads();
  // ---- level 0: load keys, histogram of the top 12 bits ----
  for (int i0 = 0; i0 < n; i0 += kSmThreads) {
    const int i = i0 + tid;
    bool pos = false;
    uint32_t d = 0;
    if (i < n) {
      const float v = xb[i];
      pos = v > 0.0f;
      const uint32_t k = pos ? 0x7FFFFFFFu - __float_as_uint(v) : 0xFFFFFFFFu;
      vk[i] = k;
      if (pos) d = uint32_t(sm_key(k, i) >> 43);
    }
    const unsigned act = __ballot_sync(0xffffffffu, pos);
    if (pos) {
      const unsigned peers = __match_any_sync(act, d);
      if (lane == __ffs(peers) - 1) atomicAdd(&hist[d], uint32_t(__popc(peers)));
    }
  }
  __syncthreads();
  {  // exclusive scan of 4096 bins (8 per thread) in place; N = total
    uint32_t loc[8], run = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { loc[j] = hist[tid * 8 + j]; run += loc[j]; }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    uint32_t base = 0, tot = 0;
    for (int w = 0; w < kSmThreads / 32; ++w) { if (w < wid) base += wsum[w]; tot += wsum[w]; }
    uint32_t e = base + inc - run;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) { hist[tid * 8 + j] = e; e += loc[j]; }
    if (tid == 0) s_N = int(tot);
  }
  __syncthreads();
  const uint32_t N = uint32_t(s_N);
  for (int c = tid; c < NC; c += kSmThreads) {
    const uint32_t start = enc_cut_start(uint32_t(c + 1), N, uint32_t(T), bins);
    if (start >= N) { cut_shift[c] = -1; cut_slot[c] = -1; continue; }
    int lo = 0, hi = 4095;  // largest d with cum[d] <= start
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (hist[mid] <= start) lo = mid; else hi = mid - 1; }
    const uint32_t next = lo == 4095 ? N : hist[lo + 1];
    cut_prefix[c] = uint64_t(lo);
    cut_resid[c] = start - hist[lo];
    if (next - hist[lo] == 1) { cut_shift[c] = 43; cut_slot[c] = -1; }
    else { cut_shift[c] = -2; cut_slot[c] = -3; }
  }
  __syncthreads();
  // ---- per-bin latencies: an element of a level-0 bin without a cut passes exactly the cuts of the
  // lower bins; only elements of bins holding a cut (the candidates) take part in the finer levels ----
  for (int d = tid; d < 4096; d += kSmThreads) {
    int lo = 0, hi = NC;  // cuts with digit < d (empty cuts, never passed, count as digit +inf)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int dm = cut_shift[mid] == -1 ? 4096 : int(cut_prefix[mid]);
      if (dm < d) lo = mid + 1; else hi = mid;
    }
    const bool inside = lo < NC && cut_shift[lo] != -1 && int(cut_prefix[lo]) == d;
    bin_lat[d] = inside ? uint8_t(0xFF) : uint8_t(lo);
  }
  if (tid == 0) s_ncand = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += kSmThreads) {  // warp-uniform trip count (the ballot needs every lane)
    const int i = i0 + tid;
    const uint32_t k32 = i < n ? vk[i] : 0xFFFFFFFFu;
    const bool c = k32 != 0xFFFFFFFFu && bin_lat[uint32_t(sm_key(k32, i) >> 43)] == 0xFF;
    const unsigned m = __ballot_sync(0xffffffffu, c);  // warp-aggregated append
    int base = 0;
    if ((tid & 31) == 0 && m) base = atomicAdd(&s_ncand, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (c) cand[base + __popc(m & ((1u << (tid & 31)) - 1u))] = uint16_t(i);
  }
  __syncthreads();
  const int ncand = s_ncand;
  // ---- levels 1..6 (a level is repeated while more than 16 distinct prefixes are pending) ----
  for (int L = 1; L < kSmLevels;) {
    if (tid == 0) {  // distinct prefixes of unresolved cuts (sorted, since cuts are in rank order)
      int ns = 0;
      for (int c = 0; c < NC; ++c) {
        if (cut_slot[c] != -3) continue;
        if (ns == 0 || slot_prefix[ns - 1] != cut_prefix[c]) slot_prefix[ns++] = cut_prefix[c];
        cut_slot[c] = ns - 1 + 1000;  // tagged: slot index + 1000
      }
      s_nslots = ns;
    }
    __syncthreads();
    const int ns = s_nslots;
    if (ns == 0) break;
    const int nsl = ns < 16 ? ns : 16;
    for (int i = tid; i < nsl * 256; i += kSmThreads) hist[i] = 0;
    __syncthreads();
    const int shp = c_sm_shift[L - 1], sh = c_sm_shift[L];
    const uint32_t mask = (1u << c_sm_bits[L]) - 1u;
    for (int j = tid; j < ncand; j += kSmThreads) {
      const int i = cand[j];
      const uint32_t k32 = vk[i];
      const uint64_t K = sm_key(k32, i), pfx = K >> shp;
      int lo = 0, hi = nsl;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (slot_prefix[mid] < pfx) lo = mid + 1; else hi = mid; }
      if (lo < nsl && slot_prefix[lo] == pfx) atomicAdd(&hist[lo * 256 + uint32_t((K >> sh) & mask)], 1u);
    }
    __syncthreads();
    for (int sl = wid; sl < nsl; sl += kSmThreads / 32) {  // per-slot exclusive scan, one warp per slot
      uint32_t loc[8], run = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { loc[j] = hist[sl * 256 + lane * 8 + j]; run += loc[j]; }
      uint32_t inc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      uint32_t e = inc - run;
#pragma unroll
      for (int j = 0; j < 8; ++j) { hist[sl * 256 + lane * 8 + j] = e; e += loc[j]; }
      if (lane == 31) slot_tot[sl] = inc;
    }
    __syncthreads();
    for (int c = tid; c < NC; c += kSmThreads) {
      if (cut_slot[c] < 1000) continue;
      const int sl = cut_slot[c] - 1000;
      if (sl >= nsl) { cut_slot[c] = -3; continue; }  // beyond the first 16 prefixes: repeat the level
      const uint32_t* h = hist + sl * 256;
      const uint32_t r = cut_resid[c];
      int lo = 0, hi = 255;
      while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (h[mid] <= r) lo = mid; else hi = mid - 1; }
      const uint32_t next = lo == 255 ? slot_tot[sl] : h[lo + 1];
      cut_prefix[c] = (cut_prefix[c] << c_sm_bits[L]) | uint64_t(lo);
      cut_resid[c] = r - h[lo];
      if (next - h[lo] == 1 || L == kSmLevels - 1) { cut_shift[c] = c_sm_shift[L]; cut_slot[c] = -1; }
      else cut_slot[c] = -4;  // descends to the next level
    }
    __syncthreads();
    if (nsl == ns) {  // every pending prefix was handled at this level: advance
      for (int c = tid; c < NC; c += kSmThreads)
        if (cut_slot[c] == -4) cut_slot[c] = -3;
      ++L;
    }
    __syncthreads();
  }
  // ---- assign: lat = number of cuts whose prefix the key reaches ----
  for (int i = tid; i < n; i += kSmThreads) {
    const uint32_t k32 = vk[i];
    if (k32 == 0xFFFFFFFFu) { lb[eo.idx(i)] = kNoSpike; continue; }
    const uint64_t K = sm_key(k32, i);
    const int bl = bin_lat[uint32_t(K >> 43)];
    if (bl != 0xFF) { lb[eo.idx(i)] = bl >= T ? kNoSpike : uint8_t(bl); continue; }
    int lo = 0, hi = NC;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const bool pass = cut_shift[mid] >= 0 && (K >> cut_shift[mid]) >= cut_prefix[mid];
      if (pass) lo = mid + 1; else hi = mid;
    }
    lb[eo.idx(i)] = lo >= T ? kNoSpike : uint8_t(lo);
  }
}

// Latency path for a handful of small images (C1: one image per plasticity step): one CTA of 1024
// threads per image sorts the image's unique 55-bit keys (value desc, index asc) with a shared-memory
// bitonic network, then every sorted rank r maps to its bin directly -- a few microseconds where the
// multi-level select, built for throughput over many images, needs tens of them for one.
constexpr int kBtThreads = 1024;
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(v), m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(v >> 32), m);
  return (uint64_t(hi) << 32) | lo;
}

// EPT keys per thread (np2 = 1024 EPT): each warp owns 32 EPT consecutive keys, lane l keys
// [l EPT, l EPT + EPT); compare-exchange partners closer than 32 EPT are in the same thread or a
// shuffle away (no barrier), farther ones go through shared memory (one barrier per stride).
template <int EPT, int NT = kBtThreads>
__global__ void __launch_bounds__(NT) enc_bitonic_kernel(const float* __restrict__ x, int n, int T, int bins,
                                                         uint8_t* __restrict__ lat, EncOut eo) {
  pdl_begin();
  constexpr int np2 = NT * EPT, WCH = 32 * EPT;
  extern __shared__ uint64_t bk[];  // [np2] keys for the long strides
  __shared__ int s_n;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int base = (tid >> 5) * WCH + lane * EPT;
  const float* xb = x + int64_t(b) * n;
  uint8_t* lb = lat + int64_t(b) * n;
  if (tid == 0) s_n = 0;
  __syncthreads();
  uint64_t v[EPT];
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int i = base + k;
    v[k] = ~uint64_t(0);  // not positive / padding: sorts last
    if (i < n) {
      const float xv = xb[i];
      if (xv > 0.0f) { v[k] = (uint64_t(0x7FFFFFFFu - __float_as_uint(xv)) << 24) | uint32_t(i); ++cnt; }
      else lb[eo.idx(i)] = kNoSpike;
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0 && cnt) atomicAdd(&s_n, cnt);
  for (int size = 2; size <= np2; size <<= 1) {  // bitonic sort, ascending
    int stride = size >> 1;
    if (stride >= WCH) {  // long strides: through shared memory
#pragma unroll
      for (int k = 0; k < EPT; ++k) bk[base + k] = v[k];
      __syncthreads();
      for (; stride >= WCH; stride >>= 1) {
        for (int i = tid; i < (np2 >> 1); i += NT) {
          const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          const bool up = (lo & size) == 0;
          const uint64_t a = bk[lo], c = bk[hi];
          if ((a > c) == up) { bk[lo] = c; bk[hi] = a; }
        }
        __syncthreads();
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k) v[k] = bk[base + k];
      __syncthreads();  // bk is rewritten by the next size's long strides
    }
    for (; stride >= EPT; stride >>= 1) {  // partner in lane ^ (stride / EPT), same slot
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int i = base + k;
        const uint64_t o = shfl_xor_u64(v[k], stride / EPT);
        const bool up = (i & size) == 0, lower = (i & stride) == 0;
        const uint64_t mn = v[k] < o ? v[k] : o, mx = v[k] < o ? o : v[k];
        v[k] = (lower == up) ? mn : mx;
      }
    }
    for (; stride > 0; stride >>= 1) {  // partner in the same thread
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int pk = k ^ stride;
        if (pk > k) {
          const bool up = ((base + k) & size) == 0;
          const uint64_t a = v[k], c = v[pk];
          if ((a > c) == up) { v[k] = c; v[pk] = a; }
        }
      }
    }
  }
  __syncthreads();  // s_n complete
  const uint32_t N = uint32_t(s_n), q = N / uint32_t(T), m = N % uint32_t(T);
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const uint32_t r = uint32_t(base + k);
    if (r >= N) continue;
    uint32_t bin;
    if (bins == 1) bin = uint32_t((uint64_t(r) * T) / N);
    else if (bins == 2) bin = q ? (r < q * uint32_t(T) ? r / q : 255u) : 255u;
    else bin = r < m * (q + 1) ? r / (q + 1) : m + (r - m * (q + 1)) / q;  // R1
    lb[eo.idx(uint32_t(v[k] & 0xFFFFFFu))] = bin >= uint32_t(T) ? kNoSpike : uint8_t(bin);
  }
}

int encode_launch(const float* x, int B, int C, int H, int W, int T, int bins, uint8_t* lat, void* wsp,
                  size_t ws_bytes, cudaStream_t s) {
  int64_t n = int64_t(C) * H * W;
  EncOut eo;  // SNN_ENCODE_OUT_NHWC: latency of flat element i = c H W + p stored at p C + c
  eo.hw = (bins & SNN_ENCODE_OUT_NHWC) ? H * W : 0;
  eo.c = C;
  bins &= 0xFF;
  if (B == 0 || n == 0) return SNN_OK;
  if (n <= 8192 && B * 2 <= num_sms()) {  // a few small images: latency path
    // keys per thread x threads = the padded key count (measured C1: 1024 threads 53 us per step, 512 56,
    // 256 63; SNN_BITONIC_NT = 256 / 512 / 1024 for tuning)
    int nt = 1024;
    if (const char* e = getenv("SNN_BITONIC_NT")) nt = atoi(e);
    const int keys = n <= 2048 ? 2048 : n <= 4096 ? 4096 : 8192;
    if (nt != 256 && nt != 512 && nt != 1024) nt = 1024;
    if (keys / nt > 16) nt = keys / 16;
    const int ept = keys / nt;
    void (*k)(const float*, int, int, int, uint8_t*, EncOut) = nullptr;
    if (nt == 256) k = ept == 8 ? enc_bitonic_kernel<8, 256> : enc_bitonic_kernel<16, 256>;
    else if (nt == 512) k = ept == 4 ? enc_bitonic_kernel<4, 512> : ept == 8 ? enc_bitonic_kernel<8, 512> : enc_bitonic_kernel<16, 512>;
    else k = ept == 2 ? enc_bitonic_kernel<2, 1024> : ept == 4 ? enc_bitonic_kernel<4, 1024> : enc_bitonic_kernel<8, 1024>;
    const size_t smem = size_t(keys) * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_encode: %s", cudaGetErrorString(e));
    launch_k(k, dim3(B), dim3(nt), smem, s, x, int(n), T, bins, lat, eo);
    note_launch();
    return check_launch("snn_encode(bitonic)");
  }
  if (n <= 16384) {
    const size_t smem = size_t(n) * (sizeof(uint32_t) + sizeof(uint16_t)) + 16;
    cudaError_t e = cudaFuncSetAttribute(enc_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_encode: %s", cudaGetErrorString(e));
    launch_k(enc_small_kernel, dim3(B), dim3(kSmThreads), smem, s, x, int(n), T, bins, lat, eo);
    note_launch();
    return check_launch("snn_encode(small)");
  }
  int G = encode_group(B, T);
  EncodeWS ws;
  size_t need = encode_ws_layout(G, T, &ws, (char*)wsp);
  if (ws_bytes < need) return set_error(SNN_EWORKSPACE, "snn_encode: workspace %zu < %zu bytes", ws_bytes, need);
  const int nchunks = int(ceil_div(n, kEncChunk));
  const bool vec = (n % 4 == 0) && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  // two radix levels over the image, then pass 3 (latencies + the few candidates) and a per-image
  // finish; the level 2-4 passes run only for images with more than kEncCandCap candidates (gated
  // on the device: no host round trip).  SNN_ENCODE_LEVELS=5 forces the all-level path (experiments).
  const bool all_levels = (eo.hw && eo.c > 256) || (getenv("SNN_ENCODE_LEVELS") && atoi(getenv("SNN_ENCODE_LEVELS")) == 5);
  int fin_smem = int(sizeof(uint64_t)) * kEncCandCap;
  if (cudaFuncSetAttribute(enc_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fin_smem) != cudaSuccess)
    return check_launch("snn_encode(finish attr)");
  for (int g0 = 0; g0 < B; g0 += G) {
    int gn = B - g0 < G ? B - g0 : G;
    const float* xg = x + int64_t(g0) * n;
    uint8_t* lg = lat + int64_t(g0) * n;
    if (cudaMemsetAsync(ws.hist0, 0, sizeof(uint32_t) * size_t(gn) * kEncBins, s) != cudaSuccess ||
        cudaMemsetAsync(ws.ncand, 0, sizeof(int32_t) * size_t(gn), s) != cudaSuccess)
      return check_launch("snn_encode memset");
    dim3 grid(nchunks, gn);
    // grid-stride kernels: about 16 chunks per CTA for level 0 (fewer flushes of the CTA histograms);
    // the gated fallback kernels at most 16 CTAs per image (an image not taking them exits at once)
    const dim3 grid0(unsigned(nchunks < 16 ? 1 : nchunks / 16), gn), gridg(unsigned(nchunks < 16 ? nchunks : 16), gn);
    launch_k(enc_hist0_kernel, dim3(grid0), dim3(kEncThreads), 0, s, xg, n, vec, ws);
    launch_k(enc_select_kernel, dim3(gn), dim3(1024), 0, s, T, bins, 0, ws, (const int32_t*)nullptr, 1);
    launch_k(enc_hist_kernel, dim3(grid0), dim3(kEncThreads), kEncL1MaxSlots * kEncL1Bins * 4, s, xg, n, vec, T, 1, ws,
             (const int32_t*)nullptr);
    launch_k(enc_select_kernel, dim3(gn), dim3(1024), 0, s, T, bins, 1, ws, (const int32_t*)nullptr, all_levels ? 1 : 0);
    note_launch(4);
    if (!all_levels) {
      launch_k(enc_tables_kernel, dim3(gn), dim3(1024), 0, s, T, bins, ws);
      note_launch();
    }
    const int32_t* gate = nullptr;
    if (!all_levels) {
      // grid-stride pass 3: about 8 chunks (or tiles) per CTA, so the per-CTA table loads stay small
      const int wpg = (eo.c % 4 == 0 && eo.c / 4 < kEncThreads / 32) ? (kEncThreads / 32) / (eo.c / 4) : 1;
      const int64_t units = eo.hw ? ceil_div(eo.hw, int64_t(kEncTileP) * wpg) : nchunks;
      dim3 g3(unsigned(units < 8 ? 1 : units / 8), gn);
      // the channels-last tile: rows padded (see enc_assign2_kernel), 128 x wpg positions when C % 4 == 0
      const int tile_bytes = eo.hw ? (eo.c % 4 == 0 ? kEncTileP * wpg * (eo.c + 4) : kEncTileP * (eo.c + 1)) : 0;
      if (cudaFuncSetAttribute(enc_assign2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_bytes) != cudaSuccess)
        return check_launch("snn_encode(assign attr)");
      launch_k(enc_assign2_kernel, dim3(g3), dim3(kEncThreads), tile_bytes, s, xg, n, vec, T, bins, lg, ws, eo);
      launch_k(enc_finish_kernel, dim3(gn), dim3(kEncFinThreads), fin_smem, s, T, bins, lg, n, ws, eo);
      note_launch(2);
      gate = ws.ovf;
    }
    for (int L = 2; L < kEncLevels; ++L) {
      launch_k(enc_hist_kernel, dim3(gate ? gridg : grid), dim3(kEncThreads), 0, s, xg, n, vec, T, L, ws, gate);
      launch_k(enc_select_kernel, dim3(gn), dim3(1024), 0, s, T, bins, L, ws, gate, 1);
      note_launch(2);
    }
    launch_k(enc_assign_kernel, dim3(gate ? gridg : grid), dim3(kEncThreads), 0, s, xg, n, T, bins, lg, ws, eo, gate);
    note_launch();
    int rc = check_launch("snn_encode");
    if (rc) return rc;
  }
  return SNN_OK;
}

// ------------------------------------------------------------------------------------ expand / validate
__global__ void expand_kernel(const uint8_t* __restrict__ lat, int64_t n, int T, float* __restrict__ wave) {
  pdl_begin();
  int b = blockIdx.y;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint8_t l = lat[int64_t(b) * n + i];
    for (int t = 0; t < T; ++t)
      wave[(int64_t(b) * T + t) * n + i] = (l != kNoSpike && t >= int(l)) ? 1.0f : 0.0f;
  }
}

int expand_launch(const uint8_t* lat, int B, int n, int T, float* wave, cudaStream_t s) {
  if (B == 0 || n == 0) return SNN_OK;
  int blocks = int(ceil_div(n, 256));
  if (blocks > 4096) blocks = 4096;
  launch_k(expand_kernel, dim3(dim3(blocks, B)), dim3(256), 0, s, lat, n, T, wave);
  note_launch();
  return check_launch("snn_expand");
}

__global__ void validate_kernel(const uint8_t* __restrict__ lat, size_t n, int T, int32_t* n_bad) {
  pdl_begin();
  int bad = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint8_t l = lat[i];
    bad += (l != kNoSpike && int(l) >= T);
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(n_bad, bad);
}

int validate_launch(const uint8_t* lat, size_t n, int T, int32_t* n_bad, cudaStream_t s) {
  if (cudaMemsetAsync(n_bad, 0, sizeof(int32_t), s) != cudaSuccess) return check_launch("snn_validate_lat");
  if (n == 0) return SNN_OK;
  size_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  launch_k(validate_kernel, dim3(unsigned(blocks)), dim3(256), 0, s, lat, n, T, n_bad);
  note_launch();
  return check_launch("snn_validate_lat");
}

}  // namespace snn
