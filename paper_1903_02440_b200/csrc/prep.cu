// prep.cu -- f2 GPU front end: the preprocessing that turns raw images into the
// intensities snn_encode ranks -- a filter bank (P:133 utils.Filter with DoG/Gabor kernels, P:223,
// P:232), local normalization and intensity lateral inhibition.  Readings R33-R35 of
// DESIGN.md fix the arithmetic order; every kernel below performs exactly that order with explicitly
// rounded operations (__dmul_rn/__dadd_rn/__fmul_rn, never contracted to FMA), so results are
// bit-identical to the definitions.
//
// All three are light stencils: one CTA per output tile of one (image, channel) plane (32 x 32 for the
// filter bank, 4 outputs per thread; 8 x 32 for the others, one per thread), the input tile plus halo
// staged once in shared memory (zero padded), filter taps in shared memory (warp broadcasts).
#include "common.cuh"

namespace snn {
namespace {

constexpr int kTH = 8, kTW = 32, kThreads = kTH * kTW;

// R33: out[b, k] = sum over (dy, dx) in row-major order of img[y + dy - pad, x + dx - pad] * ker[k, dy, dx]
// in fp64 (zero outside the image), then mode 0 -> r < threshold ? 0 : r; mode 1 -> channel 2k =
// max(r, 0), channel 2k+1 = max(-r, 0); mode 2 -> max(r, 0); cast to fp32 (round to nearest).
// One CTA per 32 x 32 output tile; each thread computes 4 horizontally adjacent outputs, so a row of
// S + 3 image values in registers serves 4 outputs per tap and each tap weight (a shared-memory
// broadcast) is read once per 4 outputs.  Every output keeps its own (dy, dx) summation order.
constexpr int kFB = 32, kFBX = 4;
__global__ void __launch_bounds__(kThreads) filter_bank_kernel(const double* __restrict__ img, int H, int W,
                                                               const double* __restrict__ ker, int K, int S,
                                                               int pad, double thr, int mode, float* __restrict__ out,
                                                               int Ho, int Wo, int tiles_x, int tiles) {
  pdl_begin();
  extern __shared__ double fsm[];
  const int SW = kFB + S - 1, SH = kFB + S - 1;
  double* tile = fsm;
  double* kk = fsm + SH * SW;
  const int64_t b = blockIdx.x / tiles;
  const int t = blockIdx.x % tiles;
  const int ty0 = (t / tiles_x) * kFB, tx0 = (t % tiles_x) * kFB;
  const double* im = img + b * H * W;
  for (int i = threadIdx.x; i < SH * SW; i += kThreads) {
    const int yy = ty0 + i / SW - pad, xx = tx0 + i % SW - pad;
    tile[i] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(im + int64_t(yy) * W + xx) : 0.0;
  }
  for (int i = threadIdx.x; i < K * S * S; i += kThreads) kk[i] = __ldg(ker + i);
  __syncthreads();
  const int ly = threadIdx.x / (kFB / kFBX), lx = (threadIdx.x % (kFB / kFBX)) * kFBX;
  const int y = ty0 + ly, x = tx0 + lx;
  if (y >= Ho || x >= Wo) return;
  const int Kout = mode == 1 ? 2 * K : K;
  const int64_t HWo = int64_t(Ho) * Wo;
  float* o = out + b * Kout * HWo + int64_t(y) * Wo + x;
  const int nx = Wo - x < kFBX ? Wo - x : kFBX;
  for (int k = 0; k < K; ++k) {
    const double* kw = kk + k * S * S;
    double r[kFBX] = {0.0, 0.0, 0.0, 0.0};
    for (int dy = 0; dy < S; ++dy) {
      const double* row = tile + (ly + dy) * SW + lx;
      double win[kFBX];
#pragma unroll
      for (int i = 0; i < kFBX - 1; ++i) win[i + 1] = row[i];
      for (int dx = 0; dx < S; ++dx) {
#pragma unroll
        for (int i = 0; i < kFBX - 1; ++i) win[i] = win[i + 1];
        win[kFBX - 1] = row[dx + kFBX - 1];
        const double wt = kw[dy * S + dx];
#pragma unroll
        for (int i = 0; i < kFBX; ++i) r[i] = __dadd_rn(r[i], __dmul_rn(win[i], wt));
      }
    }
#pragma unroll
    for (int i = 0; i < kFBX; ++i) {
      if (i >= nx) break;
      if (mode == 0) {
        o[k * HWo + i] = __double2float_rn(r[i] < thr ? 0.0 : r[i]);
      } else if (mode == 1) {
        o[(2 * k) * HWo + i] = __double2float_rn(r[i] > 0.0 ? r[i] : 0.0);
        o[(2 * k + 1) * HWo + i] = __double2float_rn(-r[i] > 0.0 ? -r[i] : 0.0);
      } else {
        o[k * HWo + i] = __double2float_rn(r[i] > 0.0 ? r[i] : 0.0);
      }
    }
  }
}

// R34: out = x / max(mean of the window [y-R, y+R] x [x-R, x+R] truncated at the borders, eps); the
// window sum in fp64 in row-major order, mean = sum / count, the division in fp64, cast to fp32.
__global__ void __launch_bounds__(kThreads) local_norm_kernel(const float* __restrict__ x, int H, int W, int R,
                                                              double eps, float* __restrict__ out, int tiles_x,
                                                              int tiles) {
  pdl_begin();
  extern __shared__ float lsm[];
  const int SW = kTW + 2 * R, SH = kTH + 2 * R;
  const int64_t bc = blockIdx.x / tiles;
  const int t = blockIdx.x % tiles;
  const int ty0 = (t / tiles_x) * kTH, tx0 = (t % tiles_x) * kTW;
  const float* xc = x + bc * H * W;
  for (int i = threadIdx.x; i < SH * SW; i += kThreads) {
    const int yy = ty0 + i / SW - R, xx = tx0 + i % SW - R;
    lsm[i] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(xc + int64_t(yy) * W + xx) : 0.f;
  }
  __syncthreads();
  const int ly = threadIdx.x / kTW, lx = threadIdx.x % kTW;
  const int y = ty0 + ly, xo = tx0 + lx;
  if (y >= H || xo >= W) return;
  const int y0 = max(y - R, 0), y1 = min(y + R, H - 1), x0 = max(xo - R, 0), x1 = min(xo + R, W - 1);
  double s = 0.0;
  for (int yy = y0; yy <= y1; ++yy) {
    const float* row = lsm + (yy - ty0 + R) * SW - tx0 + R;
    for (int xx = x0; xx <= x1; ++xx) s = __dadd_rn(s, double(row[xx]));
  }
  double m = __ddiv_rn(s, double((y1 - y0 + 1) * (x1 - x0 + 1)));
  if (m < eps) m = eps;
  out[bc * H * W + int64_t(y) * W + xo] = __double2float_rn(__ddiv_rn(double(lsm[(ly + R) * SW + lx + R]), m));
}

// R35: the sweep visits locations in (value descending, flat index ascending) order; a visited
// location p multiplies every strictly weaker location q with Chebyshev distance d <= n by
// factors[d - 1] (fp32).  Seen from q, the factors it receives are those of its strictly stronger
// neighbours, applied in that same visiting order -- so each thread walks its own window n_s + 1
// times, each pass selecting the next stronger neighbour in visiting order (no sort storage).
__global__ void __launch_bounds__(kThreads) lateral_inhibition_kernel(const float* __restrict__ x, int H, int W,
                                                                      const float* __restrict__ factors, int n,
                                                                      float* __restrict__ out, int tiles_x,
                                                                      int tiles) {
  pdl_begin();
  extern __shared__ float isms[];
  const int SW = kTW + 2 * n, SH = kTH + 2 * n;
  float* fac = isms + SH * SW;
  const int64_t bc = blockIdx.x / tiles;
  const int t = blockIdx.x % tiles;
  const int ty0 = (t / tiles_x) * kTH, tx0 = (t % tiles_x) * kTW;
  const float* xc = x + bc * H * W;
  for (int i = threadIdx.x; i < SH * SW; i += kThreads) {
    const int yy = ty0 + i / SW - n, xx = tx0 + i % SW - n;
    isms[i] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(xc + int64_t(yy) * W + xx) : 0.f;
  }
  for (int i = threadIdx.x; i < n; i += kThreads) fac[i] = __ldg(factors + i);
  __syncthreads();
  const int ly = threadIdx.x / kTW, lx = threadIdx.x % kTW;
  const int y = ty0 + ly, xo = tx0 + lx;
  if (y >= H || xo >= W) return;
  const float vq = isms[(ly + n) * SW + lx + n];
  const int y0 = max(y - n, 0), y1 = min(y + n, H - 1), x0 = max(xo - n, 0), x1 = min(xo + n, W - 1);
  float acc = vq;
  bool have = false;
  float lv = 0.f;
  int li = 0;
  for (;;) {
    bool found = false;
    float bv = 0.f;
    int bi = 0, bd = 0;
    for (int yy = y0; yy <= y1; ++yy) {
      const float* row = isms + (yy - ty0 + n) * SW - tx0 + n;
      for (int xx = x0; xx <= x1; ++xx) {
        const float vp = row[xx];
        if (!(vq < vp)) continue;  // only strictly stronger neighbours inhibit q (q itself excluded)
        const int ip = yy * W + xx;
        if (have && !(vp < lv || (vp == lv && ip > li))) continue;  // already applied
        if (!found || vp > bv || (vp == bv && ip < bi)) {
          found = true;
          bv = vp;
          bi = ip;
          bd = max(abs(yy - y), abs(xx - xo));
        }
      }
    }
    if (!found) break;
    acc = __fmul_rn(acc, fac[bd - 1]);
    have = true;
    lv = bv;
    li = bi;
  }
  out[bc * H * W + int64_t(y) * W + xo] = acc;
}

template <class Kern, class... Args>
int launch_tiles(Kern kern, const char* what, int64_t planes, int Ho, int Wo, size_t smem, cudaStream_t s,
                 Args... args) {
  const int tiles_x = int(ceil_div(Wo, kTW)), tiles = tiles_x * int(ceil_div(Ho, kTH));
  const int64_t grid = planes * tiles;
  if (grid > 0x7fffffff) return set_error(SNN_ESHAPE, "%s: %lld tiles exceed the grid limit", what, (long long)grid);
  if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return set_error(SNN_ECUDA, "%s: cannot opt in to %zu B of shared memory", what, smem);
  launch_k(kern, dim3(unsigned(grid)), dim3(kThreads), smem, s, args..., tiles_x, tiles);
  note_launch();
  return check_launch(what);
}

}  // namespace

size_t filter_bank_smem(int K, int S) { return sizeof(double) * (size_t(kFB + S - 1) * (kFB + S - 1) + size_t(K) * S * S); }
size_t stencil_smem(int r, int extra) { return sizeof(float) * (size_t(kTH + 2 * r) * (kTW + 2 * r) + extra); }

int filter_bank_launch(const double* img, int B, int H, int W, const double* ker, int K, int S, int pad, double thr,
                       int mode, float* out, cudaStream_t s) {
  const int Ho = H + 2 * pad - S + 1, Wo = W + 2 * pad - S + 1;
  const int tiles_x = int(ceil_div(Wo, kFB)), tiles = tiles_x * int(ceil_div(Ho, kFB));
  const int64_t grid = int64_t(B) * tiles;
  const size_t smem = filter_bank_smem(K, S);
  if (grid > 0x7fffffff) return set_error(SNN_ESHAPE, "filter_bank: %lld tiles exceed the grid limit", (long long)grid);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(filter_bank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return set_error(SNN_ECUDA, "filter_bank: cannot opt in to %zu B of shared memory", smem);
  launch_k(filter_bank_kernel, dim3(unsigned(grid)), dim3(kThreads), smem, s, img, H, W, ker, K, S, pad, thr, mode, out, Ho, Wo, tiles_x,
                                                             tiles);
  note_launch();
  return check_launch("filter_bank");
}

int local_norm_launch(const float* x, int B, int C, int H, int W, int R, double eps, float* out, cudaStream_t s) {
  return launch_tiles(local_norm_kernel, "local_norm", int64_t(B) * C, H, W, stencil_smem(R, 0), s, x, H, W, R, eps,
                      out);
}

int lateral_inhibition_launch(const float* x, int B, int C, int H, int W, const float* factors, int n, float* out,
                              cudaStream_t s) {
  return launch_tiles(lateral_inhibition_kernel, "lateral_inhibition", int64_t(B) * C, H, W, stencil_smem(n, n), s, x,
                      H, W, factors, n, out);
}

}  // namespace snn
