// conv_fire.cu -- a2 + a3: spiking convolution fused with threshold firing (Eq. 2,
// P:122, Eq. 5; R3-R9, N1, K2).
//
// The one-spike property turns the T convolutions of the paper (conv2d with time as the batch,
// P:93) into a single pass over each receptive field in spike-time order:
//   P[t] = P[t-1] + sum of the weights of the inputs whose spike time is exactly t
// (the onset delta, prefix-scanned along t).  One warp owns one output position; its receptive
// field (R = C*KH*KW inputs) is counting-sorted into T latency buckets in shared memory, then the
// warp walks the buckets in order.  Lanes are output features: each lane gathers FPL consecutive
// fixed-point weights per input from the shared-memory weight slice [R+1][32*FPL] and accumulates
// them exactly in int64 (units of 2^-31).  After every non-empty bucket the lane compares with the
// threshold; the first crossing gives (lat_out, v_out = fp32(P[lat_out])).  The warp exits as soon
// as all its features have fired (early exit), so only the inputs up to the last crossing are read.
//
// theta = +inf with a receptive field too large for shared memory (C2 L3, C4 L2) goes to
// conv_dense_kernel: a masked sum of the spike-wave at T-1 with weights read from L2.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace snn {

// Device error words, one per stream (snn_sync_status(stream) reads and clears its stream's word):
// streams are given slots of this per-device array in order of first use; past kErrSlots streams of
// one device, slots are shared (documented in snn.h).  The array is a module global, so every device
// has its own copy; its address is looked up per device.
constexpr int kErrSlots = 64;
constexpr int kMaxDevices = 64;
__device__ int g_error_words[kErrSlots];

namespace {
std::mutex g_err_mu;
std::unordered_map<uint64_t, int> g_err_slot;  // (device << 48) ^ stream -> slot
int g_err_next[kMaxDevices];
int* g_err_base[kMaxDevices];
}  // namespace

int* error_word_ptr(cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  std::lock_guard<std::mutex> lk(g_err_mu);
  if (!g_err_base[dev]) cudaGetSymbolAddress(reinterpret_cast<void**>(&g_err_base[dev]), g_error_words);
  const uint64_t key = (uint64_t(dev) << 48) ^ uint64_t(reinterpret_cast<uintptr_t>(s));
  auto it = g_err_slot.find(key);
  int slot;
  if (it != g_err_slot.end()) {
    slot = it->second;
  } else {
    slot = g_err_next[dev]++ % kErrSlots;
    g_err_slot.emplace(key, slot);
  }
  return g_err_base[dev] + slot;
}

int read_clear_error_word(cudaStream_t s, int* word) {
  int* p = error_word_ptr(s);
  cudaError_t e = cudaMemcpyAsync(word, p, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(int), s);
  return e == cudaSuccess ? SNN_OK : set_error(SNN_ECUDA, "snn_sync_status: %s", cudaGetErrorString(e));
}

constexpr int kSmemLimit = 227 * 1024;

struct ConvArgs {
  const uint8_t* lat_in;
  int B, C, H, W, pad;
  int F, KH, KW, T, Ho, Wo, R;
  int FGS, n_groups;
  uint32_t* wq;        // [n_groups][R+1][FGS] fixed-point weights, row R = 0
  int64_t thr;         // fire iff acc > thr
  int inf;             // theta = +inf (Eq. 5)
  uint8_t* lat_out;
  float* v_out;
  float* pot_out;      // nullable [B][T][F][Ho][Wo]
  int nhwc;            // lat_out / v_out layout: 0 = [B, F, Ho, Wo], 1 = [B, Ho, Wo, F]
  int ws_off_eoff, ws_off_ekk, ws_off_warps, warp_bytes;
  int cnt_off, start_off, size_off, list_off;
};

static inline int align16(int x) { return (x + 15) & ~15; }

// ------------------------------------------------------------------------- weight preparation
// w [F][R] fp32 -> wq [g][R+1][FGS] uint32 fixed point (w * 2^31).  Flags weights whose value is
// not an integer multiple of 2^-31 in [0, 1] (outside the exact domain, N1).
__global__ void weight_prep_kernel(const float* __restrict__ w, int F, int R, int FGS, int n_groups,
                                   uint32_t* __restrict__ wq, int nhwc_C, int KK, int* err) {
  pdl_begin();
  int64_t total = int64_t(n_groups) * (R + 1) * FGS;
  int bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    int j = int(i % FGS);
    int64_t rest = i / FGS;
    int e = int(rest % (R + 1));
    int g = int(rest / (R + 1));
    int f = g * FGS + j;
    uint32_t u = 0;
    if (f < F && e < R) {
      int se = e;  // nhwc_C > 0: rows ordered (ky, kx, c) for channels-last input (SNN_CONV_IN_NHWC)
      if (nhwc_C) { const int kk = e / nhwc_C; se = (e - kk * nhwc_C) * KK + kk; }
      float x = w[int64_t(f) * R + se];
      float s = x * 2147483648.0f;  // exact power-of-two scaling
      if (!(x >= 0.0f && x <= 1.0f) || s != truncf(s)) bad = 1;
      else u = uint32_t(s);
    }
    wq[i] = u;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrInexact);
}

// ------------------------------------------------------------------------- fused sort + walk
template <int FPL> struct WVec;
template <> struct WVec<1> { typedef uint32_t T; };
template <> struct WVec<2> { typedef uint2 T; };
template <> struct WVec<4> { typedef uint4 T; };

template <int FPL>
__device__ __forceinline__ void wload(const uint32_t* p, uint32_t (&o)[FPL]) {
  typedef typename WVec<FPL>::T V;
  V v = *reinterpret_cast<const V*>(p);
  if constexpr (FPL == 1) { o[0] = v; }
  else if constexpr (FPL == 2) { o[0] = v.x; o[1] = v.y; }
  else { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
}

template <int FPL>
__global__ void __launch_bounds__(1024, 1) conv_fire_kernel(const ConvArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int FGS = 32 * FPL;
  const int R = a.R, T = a.T;
  uint32_t* Ws = reinterpret_cast<uint32_t*>(smem);
  int32_t* eoff = reinterpret_cast<int32_t*>(smem + a.ws_off_eoff);
  uint16_t* ekk = reinterpret_cast<uint16_t*>(smem + a.ws_off_ekk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  unsigned char* wb = smem + a.ws_off_warps + warp * a.warp_bytes;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(wb + a.cnt_off);      // [T][34]
  uint16_t* start = reinterpret_cast<uint16_t*>(wb + a.start_off);  // [T+1]
  uint16_t* bsize = reinterpret_cast<uint16_t*>(wb + a.size_off);   // [T]
  uint16_t* list = reinterpret_cast<uint16_t*>(wb + a.list_off);    // [R+T+2]
  const int g = blockIdx.y;

  {  // stage the weight slice of this feature group and the receptive-field offset table
    const uint4* src = reinterpret_cast<const uint4*>(a.wq + int64_t(g) * (R + 1) * FGS);
    uint4* dst = reinterpret_cast<uint4*>(Ws);
    const int n4 = (R + 1) * FGS / 4;
    for (int i = tid; i < n4; i += blockDim.x) dst[i] = src[i];
    const int KK = a.KH * a.KW;
    for (int e = tid; e < R; e += blockDim.x) {
      int c = e / KK, r = e - c * KK, ky = r / a.KW, kx = r - ky * a.KW;
      eoff[e] = c * a.H * a.W + ky * a.W + kx;
      ekk[e] = uint16_t((ky << 8) | kx);
    }
  }
  __syncthreads();

  const int64_t HoWo = int64_t(a.Ho) * a.Wo;
  const int64_t npos = int64_t(a.B) * HoWo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  const int fbase = g * FGS + lane * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < a.F) ? (1u << j) : 0u;
  constexpr unsigned kAll = (1u << FPL) - 1;

  for (int64_t p = int64_t(blockIdx.x) * nwarps + warp; p < npos; p += int64_t(gridDim.x) * nwarps) {
    const int b = int(p / HoWo);
    const int rem = int(p - int64_t(b) * HoWo);
    const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in = a.lat_in + int64_t(b) * CHW + int64_t(y0) * a.W + x0;
    const bool interior = y0 >= 0 && x0 >= 0 && y0 + a.KH <= a.H && x0 + a.KW <= a.W;

    // ---- counting sort of the receptive field by spike time (lane-private columns) ----
    for (int t = 0; t < T; ++t) cnt[t * 34 + lane] = 0;
    __syncwarp();
    for (int e = lane; e < R; e += 32) {
      uint8_t l;
      if (interior) l = in[eoff[e]];
      else {
        int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
        bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
        l = ok ? in[eoff[e]] : kNoSpike;
      }
      if (l < T) cnt[l * 34 + lane] += 1;
    }
    __syncwarp();
    int carry = 0;
    for (int tb = 0; tb < T; tb += 32) {
      const int t = tb + lane;
      int tot = 0;
      if (t < T)
        for (int j = 0; j < 32; ++j) tot += cnt[t * 34 + j];
      const int padded = tot + (tot & 1);  // buckets padded to an even length (pair loads)
      int inc = padded;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      const int st = carry + inc - padded;
      if (t < T) {
        start[t] = uint16_t(st);
        bsize[t] = uint16_t(tot);
        int run = st;
        for (int j = 0; j < 32; ++j) { int c = cnt[t * 34 + j]; cnt[t * 34 + j] = uint16_t(run); run += c; }
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) start[T] = uint16_t(carry);
    __syncwarp();
    for (int e = lane; e < R; e += 32) {
      uint8_t l;
      if (interior) l = in[eoff[e]];
      else {
        int kk = ekk[e], ky = kk >> 8, kx = kk & 0xFF;
        bool ok = (y0 + ky >= 0) && (y0 + ky < a.H) && (x0 + kx >= 0) && (x0 + kx < a.W);
        l = ok ? in[eoff[e]] : kNoSpike;
      }
      if (l < T) {
        int c = cnt[l * 34 + lane];
        cnt[l * 34 + lane] = uint16_t(c + 1);
        list[c] = uint16_t(e);
      }
    }
    for (int t = lane; t < T; t += 32)
      if (bsize[t] & 1) list[start[t] + bsize[t]] = uint16_t(R);  // zero-weight dummy entry
    __syncwarp();

    // ---- walk the buckets in time order ----
    uint64_t acc[FPL];
    uint8_t lo[FPL];
    float vo[FPL];
#pragma unroll
    for (int j = 0; j < FPL; ++j) { acc[j] = 0; lo[j] = kNoSpike; vo[j] = 0.0f; }
    unsigned fired = ~valid & kAll;
    const uint32_t* wl = Ws + lane * FPL;
    const int total = start[T];
    int s = 0;
    for (int t = 0; t < T; ++t) {
      const int e_end = start[t + 1];
      const bool nonempty = s < e_end;
      for (int i = s; i < e_end; i += 2) {
        const uint32_t pr = *reinterpret_cast<const uint32_t*>(list + i);
        uint32_t w0[FPL], w1[FPL];
        wload<FPL>(wl + (pr & 0xFFFFu) * FGS, w0);
        wload<FPL>(wl + (pr >> 16) * FGS, w1);
#pragma unroll
        for (int j = 0; j < FPL; ++j) acc[j] += uint64_t(w0[j]) + uint64_t(w1[j]);
      }
      s = e_end;
      if (a.pot_out) {
#pragma unroll
        for (int j = 0; j < FPL; ++j)
          if (valid >> j & 1)
            a.pot_out[((int64_t(b) * T + t) * a.F + fbase + j) * HoWo + rem] = fixed_to_float(int64_t(acc[j]));
      }
      if (!a.inf && (nonempty || t == 0)) {
#pragma unroll
        for (int j = 0; j < FPL; ++j) {
          if (!(fired >> j & 1) && int64_t(acc[j]) > a.thr) {
            fired |= 1u << j;
            lo[j] = uint8_t(t);
            vo[j] = fixed_to_float(int64_t(acc[j]));
          }
        }
        if (!a.pot_out && __all_sync(0xffffffffu, fired == kAll)) break;
      }
      if (!a.pot_out && s >= total && t > 0) break;  // no input left: nothing changes any more
    }
    if (a.inf) {
#pragma unroll
      for (int j = 0; j < FPL; ++j) {
        lo[j] = acc[j] > 0 ? uint8_t(T - 1) : kNoSpike;
        vo[j] = fixed_to_float(int64_t(acc[j]));
      }
    }
#pragma unroll
    for (int j = 0; j < FPL; ++j) {
      if (valid >> j & 1) {
        const int64_t o = a.nhwc ? (int64_t(b) * HoWo + rem) * a.F + fbase + j : (int64_t(b) * a.F + fbase + j) * HoWo + rem;
        a.lat_out[o] = lo[j];
        if (a.v_out) a.v_out[o] = vo[j];
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------- dense theta = inf
// P[T-1] for receptive fields too large for the shared-memory slice: warp = (position, 32 features),
// weights [R+1][32] per group read through L1/L2 (coalesced 128 B rows).
__global__ void __launch_bounds__(256) conv_dense_kernel(const ConvArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t HoWo = int64_t(a.Ho) * a.Wo;
  const int64_t npos = int64_t(a.B) * HoWo;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;
  const int KK = a.KH * a.KW;
  const int64_t nwarps_total = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t items = npos * a.n_groups;
  for (int64_t it = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += nwarps_total) {
    const int g = int(it % a.n_groups);
    const int64_t p = it / a.n_groups;
    const int b = int(p / HoWo);
    const int rem = int(p - int64_t(b) * HoWo);
    const int y = rem / a.Wo, x = rem - (rem / a.Wo) * a.Wo;
    const int y0 = y - a.pad, x0 = x - a.pad;
    const uint8_t* in = a.lat_in + int64_t(b) * CHW;
    const uint32_t* wg = a.wq + int64_t(g) * (a.R + 1) * 32 + lane;
    uint64_t acc = 0;
    for (int e0 = 0; e0 < a.R; e0 += 32) {
      const int e = e0 + lane;
      bool spk = false;
      if (e < a.R) {
        int c = e / KK, r = e - c * KK, ky = r / a.KW, kx = r - ky * a.KW;
        int yy = y0 + ky, xx = x0 + kx;
        if (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W) spk = in[(int64_t(c) * a.H + yy) * a.W + xx] < a.T;
      }
      unsigned m = __ballot_sync(0xffffffffu, spk);
      while (m) {
        int j = __ffs(m) - 1;
        m &= m - 1;
        acc += wg[int64_t(e0 + j) * 32];
      }
    }
    const int f = g * 32 + lane;
    if (f < a.F) {
      const int64_t o = a.nhwc ? (int64_t(b) * HoWo + rem) * a.F + f : (int64_t(b) * a.F + f) * HoWo + rem;
      a.lat_out[o] = acc > 0 ? uint8_t(a.T - 1) : kNoSpike;
      if (a.v_out) a.v_out[o] = fixed_to_float(int64_t(acc));
    }
    if (a.pot_out) {  // validation mode: P[t] for every t (one masked pass per time step)
      for (int t = 0; t < a.T; ++t) {
        uint64_t pt = 0;
        for (int e0 = 0; e0 < a.R; e0 += 32) {
          const int e = e0 + lane;
          bool spk = false;
          if (e < a.R) {
            int c = e / KK, r = e - c * KK, ky = r / a.KW, kx = r - ky * a.KW;
            int yy = y0 + ky, xx = x0 + kx;
            if (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W) spk = in[(int64_t(c) * a.H + yy) * a.W + xx] <= t;
          }
          unsigned m = __ballot_sync(0xffffffffu, spk);
          while (m) {
            int j = __ffs(m) - 1;
            m &= m - 1;
            pt += wg[int64_t(e0 + j) * 32];
          }
        }
        if (f < a.F) a.pot_out[((int64_t(b) * a.T + t) * a.F + f) * HoWo + rem] = fixed_to_float(int64_t(pt));
      }
    }
  }
}

// ------------------------------------------------------------------------- host side
struct ConvPlan {
  int fpl, FGS, n_groups, nwarps, smem, dense;
  size_t wq_bytes;
  ConvArgs a;
};

static int warp_bytes_for(int T, int R, int* cnt_off, int* start_off, int* size_off, int* list_off) {
  int o = 0;
  *cnt_off = o; o += align16(T * 34 * 2);
  *start_off = o; o += align16((T + 1) * 2);
  *size_off = o; o += align16(T * 2);
  *list_off = o; o += align16((R + T + 2) * 2);
  return o;
}

static void make_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, bool inf, ConvPlan* pl) {
  ConvArgs& a = pl->a;
  a = ConvArgs{};
  a.B = B; a.C = C; a.H = H; a.W = W; a.pad = pad; a.F = F; a.KH = KH; a.KW = KW; a.T = T;
  a.Ho = H + 2 * pad - KH + 1; a.Wo = W + 2 * pad - KW + 1; a.R = C * KH * KW;
  a.inf = inf;
  const int R = a.R;
  const int wb = warp_bytes_for(T, R, &a.cnt_off, &a.start_off, &a.size_off, &a.list_off);
  a.warp_bytes = wb;
  pl->dense = 1;
  int best_fpl = 0, best_warps = 0, best_groups = 1 << 30;
  const int fpls[3] = {4, 2, 1};
  for (int k = 0; k < 3; ++k) {
    int fpl = fpls[k], FGS = 32 * fpl;
    if (fpl > 1 && F <= 32 * (fpl / 2)) continue;  // lanes would idle
    long ws_b = long(R + 1) * FGS * 4;
    long fixed = align16(int(ws_b)) + align16(R * 4) + align16(R * 2);
    if (ws_b > kSmemLimit) continue;
    long warps = (kSmemLimit - fixed) / wb;
    if (warps > 32) warps = 32;
    if (warps < 4) continue;
    int groups = int(ceil_div(F, FGS));
    // prefer fewer groups while keeping >= 8 warps per CTA
    bool better = best_fpl == 0 || (warps >= 8 && (best_warps < 8 || groups < best_groups));
    if (better) { best_fpl = fpl; best_warps = int(warps); best_groups = groups; }
  }
  if (best_fpl) {
    pl->dense = 0;
    pl->fpl = best_fpl;
    pl->FGS = 32 * best_fpl;
    pl->n_groups = best_groups;
    pl->nwarps = best_warps;
    long ws_b = long(R + 1) * pl->FGS * 4;
    a.ws_off_eoff = align16(int(ws_b));
    a.ws_off_ekk = a.ws_off_eoff + align16(R * 4);
    a.ws_off_warps = a.ws_off_ekk + align16(R * 2);
    pl->smem = a.ws_off_warps + best_warps * wb;
  } else {
    pl->fpl = 1; pl->FGS = 32; pl->n_groups = int(ceil_div(F, 32)); pl->nwarps = 8; pl->smem = 0;
  }
  a.FGS = pl->FGS;
  a.n_groups = pl->n_groups;
  pl->wq_bytes = size_t(pl->n_groups) * (R + 1) * pl->FGS * 4;
}

size_t conv_tc_workspace(int B, int C, int H, int W, int pad, int KH, int KW, int F);
int conv_tc_launches(int B, int C, int H, int W, int pad, int KH, int KW, int F);
size_t conv_walk_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T);
size_t conv_tct_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T);
int conv_tct_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                    int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                    cudaStream_t s, int nhwc);

// Finite-threshold path selection.  Default: the SIMT delta walk (conv_walk.cu).  SNN_CONV_PATH=tct
// selects the tensor-core time-stepped kernel (conv_tct.cu; exact, parity-tested, but slower than the
// walk on every config so far: its epilogue re-reads 16 bytes of TMEM per neuron and step, DESIGN.md
// §7), SNN_CONV_PATH=ref the validation kernel below.
static int conv_path_override() {
  const char* e = getenv("SNN_CONV_PATH");
  if (!e) return 1;
  if (!strcmp(e, "tct")) return 0;
  if (!strcmp(e, "ref")) return 2;
  return 1;
}
int conv_walk_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                     cudaStream_t s, int nhwc, int in_nhwc, int pool2 = 0);

static int conv_path_override();
int conv_walk_describe(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, int* pre, int* chunks,
                       int* launches);
bool conv_tct_applies(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta);

// Which kernels one snn_conv_fire call (pot_out == NULL) launches, for measurement: path 0 = fused
// sort+walk, 1 = presorted walk (sort + walk per list chunk), 2 = tensor-core Eq. 5 (theta = inf),
// 3 = tensor-core time-stepped (SNN_CONV_PATH=tct), 4 = validation kernel.
int conv_fire_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta, int* path,
                   int* launches, int* chunks) {
  const bool inf = isinf(theta) && theta > 0;
  *chunks = 1;
  if (inf) { *path = 2; *launches = conv_tc_launches(B, C, H, W, pad, KH, KW, F); return SNN_OK; }
  const int ov = conv_path_override();
  if (ov == 0 && conv_tct_applies(B, C, H, W, pad, F, KH, KW, T, theta)) { *path = 3; *launches = 2; return SNN_OK; }
  int pre = 0, ch = 1, nl = 0;
  if (ov <= 1 && conv_walk_describe(B, C, H, W, pad, F, KH, KW, T, &pre, &ch, &nl)) {
    *path = pre == 2 ? 5 : pre ? 1 : 0;
    *chunks = ch;
    *launches = nl;  // weight prep + walk (latency mode: the walk converts the weights itself), or per chunk
    return SNN_OK;
  }
  *path = 4; *launches = 2;
  return SNN_OK;
}

int weight_prep_launch(const float* w, int F, int R, int FGS, int n_groups, uint32_t* wq, cudaStream_t s,
                       int nhwc_C, int KK) {
  const int64_t total = int64_t(n_groups) * (R + 1) * FGS;
  int blocks = int(ceil_div(total, 256));
  if (blocks > 2048) blocks = 2048;
  if (blocks < 1) blocks = 1;
  launch_k(weight_prep_kernel, dim3(blocks), dim3(256), 0, s, w, F, R, FGS, n_groups, wq, nhwc_C, KK, error_word_ptr(s));
  note_launch();
  return check_launch("snn_conv_fire(weight prep)");
}
int conv_tc_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH, int KW,
                   int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes, cudaStream_t s,
                   const uint8_t* aq_pre = nullptr, int nhwc = 0, int in_nhwc = 0);

size_t conv_fire_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta) {
  const bool inf = isinf(theta) && theta > 0;
  ConvPlan pl;
  make_plan(B, C, H, W, pad, F, KH, KW, T, inf, &pl);
  size_t m = pl.wq_bytes;
  if (inf) {  // tensor-core path (and the SIMT dense path for validation mode)
    size_t t = conv_tc_workspace(B, C, H, W, pad, KH, KW, F);
    m = m > t ? m : t;
  } else {
    size_t t = conv_walk_workspace(B, C, H, W, pad, F, KH, KW, T);
    m = m > t ? m : t;
    t = conv_tct_workspace(B, C, H, W, pad, F, KH, KW, T);
    m = m > t ? m : t;
  }
  return ((m + 255) & ~size_t(255)) + 256;
}

int conv_fire_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, float* pot_out, void* ws,
                     size_t ws_bytes, cudaStream_t s, int nhwc, int in_nhwc, int pool2) {
  const bool inf = isinf(theta) && theta > 0;
  ConvPlan pl;
  make_plan(B, C, H, W, pad, F, KH, KW, T, inf, &pl);
  ConvArgs a = pl.a;
  if (ws_bytes < pl.wq_bytes) return set_error(SNN_EWORKSPACE, "snn_conv_fire: workspace %zu < %zu", ws_bytes, pl.wq_bytes);
  a.lat_in = lat_in; a.lat_out = lat_out; a.v_out = v_out; a.pot_out = pot_out; a.nhwc = nhwc;
  a.wq = reinterpret_cast<uint32_t*>(ws);
  if (!inf) {
    double t = floor(double(theta) * 2147483648.0);
    a.thr = t >= 9.0e18 ? INT64_MAX : (t < -1.0 ? -1 : (int64_t)t);
  } else a.thr = INT64_MAX;
  const int64_t npos = int64_t(B) * a.Ho * a.Wo;
  if (npos == 0 || F == 0) return SNN_OK;
  if (pool2) {  // SNN_CONV_POOL2: only the row-tile walk fuses the pooling (checked before any launch)
    if (inf || pot_out || v_out || !nhwc || !in_nhwc || conv_path_override() != 1)
      return set_error(SNN_EINVAL, "snn_conv_fire: SNN_CONV_POOL2 needs a finite threshold, channels-last input and "
                                   "output, v_out = pot_out = NULL and the default path");
    const int rc = conv_walk_launch(lat_in, B, C, H, W, pad, w, F, KH, KW, T, theta, lat_out, v_out, ws, ws_bytes, s,
                                    nhwc, in_nhwc, 1);
    return rc == 1 ? set_error(SNN_ESHAPE, "snn_conv_fire: SNN_CONV_POOL2: the row-tile walk does not apply") : rc;
  }
  if (inf && !pot_out)  // Eq. 5: dense contraction of S[T-1] on the tensor cores
    return conv_tc_launch(lat_in, B, C, H, W, pad, w, F, KH, KW, T, lat_out, v_out, ws, ws_bytes, s, nullptr, nhwc,
                          in_nhwc);
  const int path = conv_path_override();
  if (in_nhwc && (pot_out || path != 1))
    return set_error(SNN_EINVAL, "snn_conv_fire: channels-last input needs the default path without pot_out");
  if (!inf && !pot_out && path == 0) {  // tensor cores, time step by time step (conv_tct.cu)
    int rc = conv_tct_launch(lat_in, B, C, H, W, pad, w, F, KH, KW, T, theta, lat_out, v_out, ws, ws_bytes, s, nhwc);
    if (rc != 1) return rc;
  }
  if (!inf && !pot_out && path <= 1) {  // SIMT delta walk (conv_walk.cu); the kernel below validates
    int rc = conv_walk_launch(lat_in, B, C, H, W, pad, w, F, KH, KW, T, theta, lat_out, v_out, ws, ws_bytes, s, nhwc,
                              in_nhwc);
    if (rc != 1) return rc;
    if (in_nhwc) return set_error(SNN_ESHAPE, "snn_conv_fire: channels-last input: receptive field too large for the walk");
  }
  if (pl.dense && !inf)  // the walk did not apply and the validation kernel's weight slice does not fit
    return set_error(SNN_ESHAPE, "snn_conv_fire: receptive field R=%d too large for a finite threshold%s", a.R,
                     pot_out ? " with pot_out" : "");
  {
    int64_t total = int64_t(pl.n_groups) * (a.R + 1) * pl.FGS;
    int blocks = int(ceil_div(total, 256));
    if (blocks > 2048) blocks = 2048;
    weight_prep_kernel<<<blocks, 256, 0, s>>>(w, F, a.R, pl.FGS, pl.n_groups, a.wq, 0, 1, error_word_ptr(s));
    note_launch();
  }
  if (pl.dense) {
    int64_t items = npos * pl.n_groups;
    int64_t blocks = ceil_div(items, 8);
    if (blocks > int64_t(num_sms()) * 8) blocks = int64_t(num_sms()) * 8;
    conv_dense_kernel<<<int(blocks), 256, 0, s>>>(a);
    note_launch();
    return check_launch("snn_conv_fire(dense)");
  }
  int occ = 1;
  switch (pl.fpl) {
    case 1: cudaFuncSetAttribute(conv_fire_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, conv_fire_kernel<1>, pl.nwarps * 32, pl.smem); break;
    case 2: cudaFuncSetAttribute(conv_fire_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, conv_fire_kernel<2>, pl.nwarps * 32, pl.smem); break;
    default: cudaFuncSetAttribute(conv_fire_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, conv_fire_kernel<4>, pl.nwarps * 32, pl.smem); break;
  }
  if (occ < 1) occ = 1;
  int64_t per_group = ceil_div(npos, pl.nwarps);
  int64_t want = ceil_div(int64_t(num_sms()) * occ, pl.n_groups);
  int gx = int(per_group < want ? per_group : want);
  if (gx < 1) gx = 1;
  dim3 grid(gx, pl.n_groups);
  switch (pl.fpl) {
    case 1:
      conv_fire_kernel<1><<<grid, pl.nwarps * 32, pl.smem, s>>>(a);
      note_launch();
      break;
    case 2:
      conv_fire_kernel<2><<<grid, pl.nwarps * 32, pl.smem, s>>>(a);
      note_launch();
      break;
    default:
      conv_fire_kernel<4><<<grid, pl.nwarps * 32, pl.smem, s>>>(a);
      note_launch();
      break;
  }
  return check_launch("snn_conv_fire");
}

}  // namespace snn
