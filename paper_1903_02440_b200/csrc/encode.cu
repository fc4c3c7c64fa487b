// encode.cu -- a1: intensity -> latency rank-order encoding (R1/R2, K1).
//
// Per image, the N positive intensities are ranked by the unique 55-bit key
//     K = ((0x7FFFFFFF - bits(x)) << 24) | flat_index          (x > 0, flat_index < 2^24)
// whose ascending order is (value descending, index ascending).  Bin b (b = 1..T-1) starts at rank
// start_b = b*q + min(b, m).  Instead of sorting, a multi-level MSB radix SELECT finds, for every
// cut b, the key prefix of the element of rank start_b (levels of 12/12/12/12/7 bits; a cut stops
// as soon as its digit bucket holds a single element).  Then every element's latency is the number
// of cuts whose prefix it reaches: lat = #{b : (K >> shift_b) >= prefix_b}.  HBM traffic is one read
// of x per level (L2-resident for a group of images) plus one write of lat.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace snn {

constexpr int kEncLevels = 5;
constexpr int kEncBins = 4096;
__constant__ int c_enc_bits[kEncLevels] = {12, 12, 12, 12, 7};
__constant__ int c_enc_shift[kEncLevels] = {43, 31, 19, 7, 0};  // prefix after level L = K >> shift[L]
constexpr int kEncThreads = 256;
constexpr int kEncPerThread = 16;
constexpr int kEncChunk = kEncThreads * kEncPerThread;

struct EncodeWS {
  uint32_t* hist0;      // [G][4096]
  uint32_t* hist;       // [G][S][4096]   S = T (>= the number of cuts)
  uint64_t* cut_prefix; // [G][S]
  int32_t* cut_shift;   // [G][S]  -1 = empty cut (never passed); >=0 when resolved
  uint32_t* cut_resid;  // [G][S]
  int32_t* cut_slot;    // [G][S]  slot of an unresolved cut, -1 when resolved / empty
  uint64_t* slot_prefix;// [G][S]
  int32_t* n_slots;     // [G]
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

// Level 0: histogram of the top 12 bits of every positive key (all images of the group).
__global__ void __launch_bounds__(kEncThreads) enc_hist0_kernel(const float* __restrict__ x, int64_t n,
                                                                 EncodeWS ws) {
  pdl_begin();
  __shared__ uint32_t sh[kEncBins];
  for (int i = threadIdx.x; i < kEncBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int g = blockIdx.y;
  const float* xg = x + int64_t(g) * n;
  int64_t base = int64_t(blockIdx.x) * kEncChunk;
  for (int j = 0; j < kEncPerThread; ++j) {
    int64_t i = base + int64_t(j) * kEncThreads + threadIdx.x;
    bool pos = false;
    uint32_t d = 0;
    if (i < n) {
      float v = xg[i];
      pos = v > 0.0f;
      if (pos) d = uint32_t(enc_key(v, uint32_t(i)) >> 43);
    }
    // warp-aggregated shared atomics: intensities cluster in few bins (e.g. one exponent)
    unsigned act = __ballot_sync(0xffffffffu, pos);
    if (pos) {
      unsigned peers = __match_any_sync(act, d);
      int leader = __ffs(peers) - 1;
      if ((threadIdx.x & 31) == leader) atomicAdd(&sh[d], __popc(peers));
    }
  }
  __syncthreads();
  uint32_t* hg = ws.hist0 + int64_t(g) * kEncBins;
  for (int i = threadIdx.x; i < kEncBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hg[i], sh[i]);
}

// Levels 1..4: histogram of the next digit for elements whose prefix matches an unresolved cut.
__global__ void __launch_bounds__(kEncThreads) enc_hist_kernel(const float* __restrict__ x, int64_t n, int T,
                                                                int level, EncodeWS ws) {
  pdl_begin();
  const int g = blockIdx.y;
  const int S = T;
  const int ns = ws.n_slots[g];
  if (ns == 0) return;
  __shared__ uint64_t sp[256];
  __shared__ uint32_t dmask[kEncBins / 32];  // previous-level digits of the unresolved prefixes
  for (int i = threadIdx.x; i < kEncBins / 32; i += blockDim.x) dmask[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const uint64_t q = ws.slot_prefix[int64_t(g) * S + i];
    sp[i] = q;
    atomicOr(&dmask[uint32_t(q >> 5) & (kEncBins / 32 - 1)], 1u << (uint32_t(q) & 31));
  }
  __syncthreads();
  const int shp = c_enc_shift[level - 1], sh = c_enc_shift[level];
  const uint64_t mask = (uint64_t(1) << c_enc_bits[level]) - 1;
  const float* xg = x + int64_t(g) * n;
  uint32_t* hg = ws.hist + int64_t(g) * S * kEncBins;
  int64_t base = int64_t(blockIdx.x) * kEncChunk;
  for (int j = 0; j < kEncPerThread; ++j) {
    int64_t i = base + int64_t(j) * kEncThreads + threadIdx.x;
    if (i >= n) break;
    float v = xg[i];
    if (!(v > 0.0f)) continue;
    uint64_t K = enc_key(v, uint32_t(i));
    uint64_t p = K >> shp;
    const uint32_t dg = uint32_t(p) & (kEncBins - 1);  // a 12-bit digit: most elements leave here
    if (!(dmask[dg >> 5] >> (dg & 31) & 1)) continue;
    int lo = 0, hi = ns;  // lower_bound
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (sp[mid] < p) lo = mid + 1; else hi = mid;
    }
    if (lo < ns && sp[lo] == p) atomicAdd(&hg[int64_t(lo) * kEncBins + ((K >> sh) & mask)], 1u);
  }
}

// Per-image selection after level L: locate every unresolved cut's digit, resolve or descend,
// rebuild the sorted list of distinct prefixes for level L+1 and zero their histograms.
__global__ void __launch_bounds__(256) enc_select_kernel(int T, int bins, int level, EncodeWS ws) {
  pdl_begin();
  const int g = blockIdx.x;
  const int S = T;
  const int NC = enc_ncuts(T, bins);
  __shared__ uint32_t cum[kEncBins + 1];
  __shared__ uint32_t wsum[8];
  __shared__ int s_nslots;
  uint64_t* cp = ws.cut_prefix + int64_t(g) * S;
  int32_t* csh = ws.cut_shift + int64_t(g) * S;
  uint32_t* cr = ws.cut_resid + int64_t(g) * S;
  int32_t* cs = ws.cut_slot + int64_t(g) * S;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  int nslots = (level == 0) ? 1 : ws.n_slots[g];
  for (int s = 0; s < nslots; ++s) {
    const uint32_t* h = (level == 0) ? ws.hist0 + int64_t(g) * kEncBins
                                     : ws.hist + (int64_t(g) * S + s) * kEncBins;
    // block exclusive scan of 4096 bins: 16 consecutive bins per thread
    uint32_t loc[16], run = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) { loc[j] = h[tid * 16 + j]; run += loc[j]; }
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    uint32_t wbase = 0;
    for (int w = 0; w < wid; ++w) wbase += wsum[w];
    uint32_t e = wbase + inc - run;
#pragma unroll
    for (int j = 0; j < 16; ++j) { cum[tid * 16 + j] = e; e += loc[j]; }
    if (tid == 255) cum[kEncBins] = e;
    __syncthreads();
    if (level == 0) {
      // initialise the cuts from N = total positives
      uint32_t N = cum[kEncBins];
      for (int b = tid; b < NC; b += blockDim.x) {
        uint32_t start = enc_cut_start(uint32_t(b + 1), N, uint32_t(T), bins);
        cp[b] = 0;
        if (start >= N) { csh[b] = -1; cs[b] = -1; cr[b] = 0; }
        else { csh[b] = -2; cs[b] = 0; cr[b] = start; }
      }
      __syncthreads();
    }
    for (int b = tid; b < NC; b += blockDim.x) {
      if (cs[b] != s || csh[b] == -1) continue;
      uint32_t r = cr[b];
      int lo = 0, hi = kEncBins - 1;  // largest d with cum[d] <= r
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (cum[mid] <= r) lo = mid; else hi = mid - 1;
      }
      uint32_t cnt = cum[lo + 1] - cum[lo];
      uint64_t np = (cp[b] << c_enc_bits[level]) | uint64_t(lo);
      cp[b] = np;
      cr[b] = r - cum[lo];
      if (cnt == 1 || level == kEncLevels - 1) { csh[b] = c_enc_shift[level]; cs[b] = -1; }
      else cs[b] = -3;  // unresolved, slot assigned below
    }
    __syncthreads();
  }
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
  if (level + 1 < kEncLevels) {
    uint32_t* hg = ws.hist + int64_t(g) * S * kEncBins;
    for (int64_t i = tid; i < int64_t(s_nslots) * kEncBins; i += blockDim.x) hg[i] = 0;
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

__global__ void __launch_bounds__(kEncThreads) enc_assign_kernel(const float* __restrict__ x, int64_t n, int T,
                                                                  int bins, uint8_t* __restrict__ lat, EncodeWS ws,
                                                                  EncOut eo) {
  pdl_begin();
  const int g = blockIdx.y;
  const int S = T;
  const int NC = enc_ncuts(T, bins);
  __shared__ uint64_t sp[256];
  __shared__ int ssh[256];
  for (int b = threadIdx.x; b < NC; b += blockDim.x) {
    sp[b] = ws.cut_prefix[int64_t(g) * S + b];
    ssh[b] = ws.cut_shift[int64_t(g) * S + b];
  }
  __syncthreads();
  const float* xg = x + int64_t(g) * n;
  uint8_t* lg = lat + int64_t(g) * n;
  int64_t base = int64_t(blockIdx.x) * kEncChunk;
  for (int j = 0; j < kEncPerThread; ++j) {
    int64_t i = base + int64_t(j) * kEncThreads + threadIdx.x;
    if (i >= n) break;
    float v = xg[i];
    uint8_t out = kNoSpike;
    if (v > 0.0f) {
      uint64_t K = enc_key(v, uint32_t(i));
      int lo = 0, hi = NC;  // number of cuts passed (pass(b) is monotone non-increasing in b)
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        bool pass = ssh[mid] >= 0 && (K >> ssh[mid]) >= sp[mid];
        if (pass) lo = mid + 1; else hi = mid;
      }
      out = lo >= T ? kNoSpike : uint8_t(lo);
    }
    lg[eo.idx(uint32_t(i))] = out;
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
  int nchunks = int(ceil_div(n, kEncChunk));
  for (int g0 = 0; g0 < B; g0 += G) {
    int gn = B - g0 < G ? B - g0 : G;
    const float* xg = x + int64_t(g0) * n;
    if (cudaMemsetAsync(ws.hist0, 0, sizeof(uint32_t) * size_t(gn) * kEncBins, s) != cudaSuccess)
      return check_launch("snn_encode memset");
    dim3 grid(nchunks, gn);
    launch_k(enc_hist0_kernel, dim3(grid), dim3(kEncThreads), 0, s, xg, n, ws);
    note_launch();
    if (enc_ncuts(T, bins) > 0) {
      launch_k(enc_select_kernel, dim3(gn), dim3(256), 0, s, T, bins, 0, ws);
      note_launch();
      for (int L = 1; L < kEncLevels; ++L) {
        launch_k(enc_hist_kernel, dim3(grid), dim3(kEncThreads), 0, s, xg, n, T, L, ws);
        note_launch();
        launch_k(enc_select_kernel, dim3(gn), dim3(256), 0, s, T, bins, L, ws);
        note_launch();
      }
    }
    launch_k(enc_assign_kernel, dim3(grid), dim3(kEncThreads), 0, s, xg, n, T, bins, lat + int64_t(g0) * n, ws, eo);
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
