// api.cu -- the C ABI of libsnn (include/snn.h): host-side argument checks, workspace queries,
// error reporting, then one asynchronous launch sequence per call on the caller's stream.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>

#include "common.cuh"

namespace snn {

size_t encode_workspace(int B, int C, int H, int W, int T);
int encode_launch(const float* x, int B, int C, int H, int W, int T, int bins, uint8_t* lat, void* ws, size_t ws_bytes,
                  cudaStream_t s);
int expand_launch(const uint8_t* lat, int B, int n, int T, float* wave, cudaStream_t s);
int validate_launch(const uint8_t* lat, size_t n, int T, int32_t* n_bad, cudaStream_t s);
size_t conv_fire_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta);
int conv_fire_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta, int* path,
                   int* launches, int* chunks);
int conv_fire_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, uint8_t* lat_out, float* v_out, float* pot_out, void* ws,
                     size_t ws_bytes, cudaStream_t s, int nhwc, int in_nhwc, int pool2 = 0);
int pool_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, int PH, int PW, int SH, int SW,
                int DH, int DW, int flags, uint8_t* lat_out, float* v_out, cudaStream_t s);
int inhibit_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, uint8_t* lat_out, float* v_out,
                   int16_t* winner_f, cudaStream_t s);
size_t k_winners_workspace(int B, int F, int H, int W);
size_t seq_train_workspace(int C, int H, int W, int pad, int F, int KH, int KW, int T, int k, int N);
int seq_train_launch(const uint8_t* lat_all, int N, int C, int H, int W, int pad, float* w, int F, int KH, int KW,
                     int T, float theta, int k, int r, float a_plus, float a_minus, float lb, float ub,
                     int stabilizer, int32_t* winners, int32_t* count, float* snaps, int snap_every, void* ws,
                     size_t ws_bytes, cudaStream_t st);
int k_winners_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, int k, int r, int32_t* winners,
                     int32_t* count, void* ws, size_t ws_bytes, cudaStream_t s);
int stdp_launch(float* w, int F, int C, int KH, int KW, const uint8_t* lat_in, int H, int W, int pad,
                const uint8_t* lat_out, int Ho, int Wo, const int32_t* winners, const int32_t* count, int k,
                float a_plus, float a_minus, float lb, float ub, int stabilizer, const float* reward, int f0,
                int sharded, cudaStream_t s);
int position_keys_launch(const uint8_t* lat, const float* v, int B, int F, int H, int W, int f0, int64_t* keys,
                         cudaStream_t s);
size_t k_winners_keys_workspace(int B, int H, int W);
int k_winners_keys_launch(const int64_t* keys, int B, int H, int W, int k, int r, int32_t* winners, int32_t* count,
                          void* ws, size_t ws_bytes, cudaStream_t s);
int count_events_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                        const uint8_t* lat_out, unsigned long long* out, cudaStream_t s);
size_t filter_bank_smem(int K, int S);
size_t stencil_smem(int r, int extra);
int filter_bank_launch(const double* img, int B, int H, int W, const double* ker, int K, int S, int pad, double thr,
                       int mode, float* out, cudaStream_t s);
int local_norm_launch(const float* x, int B, int C, int H, int W, int R, double eps, float* out, cudaStream_t s);
int lateral_inhibition_launch(const float* x, int B, int C, int H, int W, const float* factors, int n, float* out,
                              cudaStream_t s);
size_t conv_inf_prepare_bytes(int B, int C, int H, int W, int pad, int F, int KH, int KW);
int conv_inf_prepare_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                            void* prep, size_t prep_bytes, cudaStream_t s);
size_t rstdp_inf_workspace(int C, int H, int W, int pad, int F, int KH, int KW);
int rstdp_inf_sequence_launch(const void* prep, int b0, int N, int C, int H, int W, int pad, const uint8_t* lat_in,
                              float* w, int F, int KH, int KW, int T, const int32_t* labels, int n_classes,
                              float a_plus, float a_minus, float lb, float ub, int stabilizer, int32_t* winners,
                              int32_t* count, int32_t* decision, float* reward, void* ws, size_t ws_bytes,
                              cudaStream_t s);
int conv_fire_prepared_launch(const void* prep, int b, int C, int H, int W, int pad, const float* w, int F, int KH,
                              int KW, int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                              cudaStream_t s);
int decide_launch(const int32_t* winners, const int32_t* count, int B, int k, int F, int n_classes,
                  const int32_t* labels, int32_t* decision, float* reward, cudaStream_t s);

static thread_local char t_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void note_launch(int n) { g_launches.fetch_add(uint64_t(n), std::memory_order_relaxed); }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return SNN_OK;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SNN_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

int num_sms() {
  static std::atomic<int> cache[64];  // per device ordinal (0 = not looked up yet)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

}  // namespace snn

using namespace snn;

#define REQUIRE(cond, code, ...)                 \
  do {                                           \
    if (!(cond)) return set_error(code, __VA_ARGS__); \
  } while (0)

static inline cudaStream_t S(snn_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

static int conv_checks(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta) {
  REQUIRE(T >= 1 && T <= 254, SNN_EINVAL, "snn_conv_fire: T=%d outside [1, 254]", T);
  REQUIRE(!isnan(theta), SNN_EINVAL, "snn_conv_fire: theta is NaN");
  REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && F >= 0 && KH >= 1 && KW >= 1 && pad >= 0, SNN_ESHAPE,
          "snn_conv_fire: bad dimensions");
  REQUIRE(KH <= H + 2 * pad && KW <= W + 2 * pad, SNN_ESHAPE,
          "snn_conv_fire: kernel %dx%d larger than padded input %dx%d", KH, KW, H + 2 * pad, W + 2 * pad);
  REQUIRE(int64_t(C) * KH * KW <= 65534, SNN_ESHAPE, "snn_conv_fire: receptive field C*KH*KW > 65534");
  REQUIRE(KH < 256 && KW < 256, SNN_ESHAPE, "snn_conv_fire: kernel side >= 256");
  return SNN_OK;
}

extern "C" {

int snn_version(void) { return 1; }

unsigned long long snn_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int snn_count_events(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                     const uint8_t* lat_out, unsigned long long* out, snn_stream_t s) {
  int rc = conv_checks(B, C, H, W, pad, F, KH, KW, T, 0.0f);
  if (rc) return rc;
  REQUIRE(out, SNN_EINVAL, "snn_count_events: NULL output");
  return count_events_launch(lat_in, B, C, H, W, pad, F, KH, KW, T, lat_out, out, S(s));
}

const char* snn_last_error(void) { return t_err; }

int snn_sync_status(snn_stream_t s) {
  cudaError_t e = cudaStreamSynchronize(S(s));
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_sync_status: %s", cudaGetErrorString(e));
  int word = 0;
  int rc = read_clear_error_word(S(s), &word);
  if (rc) return rc;
  if (word & kErrInternal) return set_error(SNN_ECUDA, "internal error: a kernel consistency trap fired");
  if (word & kErrWinner)
    return set_error(SNN_EINVAL, "snn_stdp_update: a winner lies outside the map or the layer's features (skipped)");
  if (word & kErrInexact)
    return set_error(SNN_EINEXACT, "a weight is outside the exact domain {w : w*2^31 integral, 0 <= w <= 1}");
  return SNN_OK;
}

size_t snn_encode_workspace(int B, int C, int H, int W, int T) {
  if (B < 0 || C < 0 || H < 0 || W < 0 || T < 1 || T > 254) return 0;
  return encode_workspace(B, C, H, W, T);
}

int snn_filter_bank(const double* img, int B, int H, int W, const double* kernels, int K, int ksize, int pad,
                    double threshold, int mode, float* out, snn_stream_t s) {
  REQUIRE(mode >= 0 && mode <= 2, SNN_EINVAL, "snn_filter_bank: mode=%d not in {0, 1, 2}", mode);
  REQUIRE(!(threshold != threshold), SNN_EINVAL, "snn_filter_bank: NaN threshold");
  REQUIRE(B >= 0 && H >= 1 && W >= 1 && K >= 1, SNN_ESHAPE, "snn_filter_bank: bad dimension");
  REQUIRE(ksize >= 1 && ksize <= 31 && pad >= 0 && pad < ksize, SNN_ESHAPE, "snn_filter_bank: S=%d pad=%d", ksize, pad);
  REQUIRE(H + 2 * pad - ksize + 1 >= 1 && W + 2 * pad - ksize + 1 >= 1, SNN_ESHAPE, "snn_filter_bank: kernel larger than input");
  REQUIRE(int64_t(H) * W < (int64_t(1) << 31), SNN_ESHAPE, "snn_filter_bank: H*W >= 2^31");
  REQUIRE(snn::filter_bank_smem(K, ksize) <= 200 * 1024, SNN_ESHAPE, "snn_filter_bank: %d taps of %dx%d exceed shared memory", K, ksize, ksize);
  if (B == 0) return SNN_OK;
  REQUIRE(img && kernels && out, SNN_EINVAL, "snn_filter_bank: NULL tensor");
  return snn::filter_bank_launch(img, B, H, W, kernels, K, ksize, pad, threshold, mode, out, S(s));
}

int snn_local_norm(const float* x, int B, int C, int H, int W, int radius, double eps, float* out, snn_stream_t s) {
  REQUIRE(radius >= 0 && radius <= 32, SNN_EINVAL, "snn_local_norm: radius=%d outside [0, 32]", radius);
  REQUIRE(eps > 0, SNN_EINVAL, "snn_local_norm: eps must be > 0");
  REQUIRE(B >= 0 && C >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_local_norm: negative dimension");
  REQUIRE(int64_t(H) * W < (int64_t(1) << 31), SNN_ESHAPE, "snn_local_norm: H*W >= 2^31");
  if (int64_t(B) * C * H * W == 0) return SNN_OK;
  REQUIRE(x && out && x != out, SNN_EINVAL, "snn_local_norm: NULL or aliased tensor");
  return snn::local_norm_launch(x, B, C, H, W, radius, eps, out, S(s));
}

int snn_lateral_inhibition(const float* x, int B, int C, int H, int W, const float* factors, int n, float* out,
                           snn_stream_t s) {
  REQUIRE(n >= 0 && n <= 32, SNN_EINVAL, "snn_lateral_inhibition: n=%d outside [0, 32]", n);
  REQUIRE(B >= 0 && C >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_lateral_inhibition: negative dimension");
  REQUIRE(int64_t(H) * W < (int64_t(1) << 31), SNN_ESHAPE, "snn_lateral_inhibition: H*W >= 2^31");
  if (int64_t(B) * C * H * W == 0) return SNN_OK;
  REQUIRE(x && out && x != out && (factors || n == 0), SNN_EINVAL, "snn_lateral_inhibition: NULL or aliased tensor");
  return snn::lateral_inhibition_launch(x, B, C, H, W, factors, n, out, S(s));
}

int snn_encode_ex(const float* x, int B, int C, int H, int W, int T, int bins, uint8_t* lat, void* ws,
                  size_t ws_bytes, snn_stream_t s) {
  REQUIRE(T >= 1 && T <= 254, SNN_EINVAL, "snn_encode: T=%d outside [1, 254]", T);
  REQUIRE((bins & 0xFF) <= SNN_BINS_FLOOR && (bins & ~(0xFF | SNN_ENCODE_OUT_NHWC)) == 0, SNN_EINVAL,
          "snn_encode: bins=0x%x unknown", bins);
  REQUIRE(B >= 0 && C >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_encode: negative dimension");
  REQUIRE(int64_t(C) * H * W < (int64_t(1) << 24), SNN_ESHAPE, "snn_encode: C*H*W >= 2^24");
  if (int64_t(B) * C * H * W == 0) return SNN_OK;
  REQUIRE(x && lat, SNN_EINVAL, "snn_encode: NULL tensor");
  REQUIRE(ws, SNN_EWORKSPACE, "snn_encode: NULL workspace");
  return encode_launch(x, B, C, H, W, T, bins, lat, ws, ws_bytes, S(s));
}

int snn_encode(const float* x, int B, int C, int H, int W, int T, uint8_t* lat, void* ws, size_t ws_bytes,
               snn_stream_t s) {
  return snn_encode_ex(x, B, C, H, W, T, SNN_BINS_R1, lat, ws, ws_bytes, s);
}

int snn_expand(const uint8_t* lat, int B, int n, int T, float* wave, snn_stream_t s) {
  REQUIRE(T >= 1 && T <= 254, SNN_EINVAL, "snn_expand: T=%d outside [1, 254]", T);
  REQUIRE(B >= 0 && n >= 0, SNN_ESHAPE, "snn_expand: negative dimension");
  if (int64_t(B) * n == 0) return SNN_OK;
  REQUIRE(lat && wave, SNN_EINVAL, "snn_expand: NULL tensor");
  return expand_launch(lat, B, n, T, wave, S(s));
}

int snn_validate_lat(const uint8_t* lat, size_t n, int T, int32_t* n_bad, snn_stream_t s) {
  REQUIRE(T >= 1 && T <= 254, SNN_EINVAL, "snn_validate_lat: T=%d outside [1, 254]", T);
  REQUIRE(n_bad && (lat || n == 0), SNN_EINVAL, "snn_validate_lat: NULL tensor");
  return validate_launch(lat, n, T, n_bad, S(s));
}


size_t snn_conv_fire_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta) {
  if (conv_checks(B, C, H, W, pad, F, KH, KW, T, theta)) return 0;
  return conv_fire_workspace(B, C, H, W, pad, F, KH, KW, T, theta);
}

size_t snn_conv_inf_prepare_bytes(int B, int C, int H, int W, int pad, int F, int KH, int KW) {
  if (conv_checks(B, C, H, W, pad, F, KH, KW, 1, INFINITY)) return 0;
  return conv_inf_prepare_bytes(B, C, H, W, pad, F, KH, KW);
}

int snn_conv_inf_prepare(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                         void* prep, size_t prep_bytes, snn_stream_t s) {
  int rc = conv_checks(B, C, H, W, pad, F, KH, KW, T, INFINITY);
  if (rc) return rc;
  if (B == 0 || F == 0) return SNN_OK;
  REQUIRE(lat_in && prep, SNN_EINVAL, "snn_conv_inf_prepare: NULL tensor");
  return conv_inf_prepare_launch(lat_in, B, C, H, W, pad, F, KH, KW, T, prep, prep_bytes, S(s));
}

size_t snn_rstdp_inf_workspace(int C, int H, int W, int pad, int F, int KH, int KW) {
  if (C < 1 || H < 1 || W < 1 || pad < 0 || F < 1 || KH < 1 || KW < 1 || KH > H + 2 * pad || KW > W + 2 * pad) return 0;
  return rstdp_inf_workspace(C, H, W, pad, F, KH, KW);
}

int snn_rstdp_inf_sequence(const void* prep, int b0, int N, int C, int H, int W, int pad, const uint8_t* lat_in,
                           float* w, int F, int KH, int KW, int T, const int32_t* labels, int n_classes, float a_plus,
                           float a_minus, float lb, float ub, int stabilizer, int32_t* winners, int32_t* count,
                           int32_t* decision, float* reward, void* ws, size_t ws_bytes, snn_stream_t s) {
  int rc = conv_checks(1, C, H, W, pad, F, KH, KW, T, INFINITY);
  if (rc) return rc;
  REQUIRE(b0 >= 0 && N >= 0, SNN_EINVAL, "snn_rstdp_inf_sequence: b0 or N negative");
  REQUIRE(n_classes >= 1 && F / n_classes >= 1, SNN_EINVAL, "snn_rstdp_inf_sequence: n_classes=%d", n_classes);
  REQUIRE(stabilizer >= 0 && stabilizer <= 2, SNN_EINVAL, "snn_rstdp_inf_sequence: stabilizer=%d", stabilizer);
  REQUIRE(lb < ub, SNN_EINVAL, "snn_rstdp_inf_sequence: LB >= UB");
  REQUIRE(!isnan(a_plus) && !isnan(a_minus), SNN_EINVAL, "snn_rstdp_inf_sequence: NaN rate");
  REQUIRE(int64_t(F) * (H + 2 * pad - KH + 1) * (W + 2 * pad - KW + 1) <= (int64_t(1) << 24), SNN_ESHAPE,
          "snn_rstdp_inf_sequence: F*Ho*Wo > 2^24");
  if (N == 0) return SNN_OK;
  REQUIRE(prep && lat_in && w && winners && count, SNN_EINVAL, "snn_rstdp_inf_sequence: NULL tensor");
  REQUIRE(ws, SNN_EWORKSPACE, "snn_rstdp_inf_sequence: NULL workspace");
  return rstdp_inf_sequence_launch(prep, b0, N, C, H, W, pad, lat_in, w, F, KH, KW, T, labels, n_classes, a_plus,
                                   a_minus, lb, ub, stabilizer, winners, count, decision, reward, ws, ws_bytes, S(s));
}

int snn_conv_fire_prepared(const void* prep, int b, int C, int H, int W, int pad, const float* w, int F, int KH,
                           int KW, int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes, snn_stream_t s) {
  int rc = conv_checks(1, C, H, W, pad, F, KH, KW, T, INFINITY);
  if (rc) return rc;
  REQUIRE(b >= 0, SNN_EINVAL, "snn_conv_fire_prepared: b < 0");
  if (F == 0) return SNN_OK;
  REQUIRE(prep && w && lat_out && v_out, SNN_EINVAL, "snn_conv_fire_prepared: NULL tensor");
  REQUIRE(ws, SNN_EWORKSPACE, "snn_conv_fire_prepared: NULL workspace");
  return conv_fire_prepared_launch(prep, b, C, H, W, pad, w, F, KH, KW, T, lat_out, v_out, ws, ws_bytes, S(s));
}

size_t snn_stdp_sequence_workspace(int N, int C, int H, int W, int pad, int F, int KH, int KW, int T, int k) {
  if (N < 0 || C < 1 || H < 1 || W < 1 || pad < 0 || F < 1 || KH < 1 || KW < 1 || T < 1 || T > 254 || k < 1) return 0;
  return seq_train_workspace(C, H, W, pad, F, KH, KW, T, k, N);
}

int snn_stdp_sequence(const uint8_t* lat_in, int N, int C, int H, int W, int pad, float* w, int F, int KH, int KW,
                      int T, float theta, int k, int r, float a_plus, float a_minus, float lb, float ub,
                      int stabilizer, int32_t* winners, int32_t* count, float* snapshots, int snap_every, void* ws,
                      size_t ws_bytes, snn_stream_t s) {
  REQUIRE(stabilizer >= 0 && stabilizer <= 2, SNN_EINVAL, "snn_stdp_sequence: stabilizer=%d not in {0, 1, 2}", stabilizer);
  int rc = conv_checks(N, C, H, W, pad, F, KH, KW, T, theta);
  if (rc) return rc;
  REQUIRE(k >= 1 && k <= 256, SNN_EINVAL, "snn_stdp_sequence: k=%d outside [1, 256]", k);
  REQUIRE(r >= 0, SNN_EINVAL, "snn_stdp_sequence: r=%d < 0", r);
  REQUIRE(lb < ub, SNN_EINVAL, "snn_stdp_sequence: lb >= ub");
  REQUIRE(!snapshots || snap_every >= 1, SNN_EINVAL, "snn_stdp_sequence: snap_every < 1");
  REQUIRE(lat_in && w && winners && count && ws, SNN_EINVAL, "snn_stdp_sequence: NULL pointer");
  if (N == 0) return SNN_OK;
  rc = seq_train_launch(lat_in, N, C, H, W, pad, w, F, KH, KW, T, theta, k, r, a_plus, a_minus, lb, ub, stabilizer,
                        winners, count, snapshots, snap_every, ws, ws_bytes, S(s));
  if (rc == 1)
    return set_error(SNN_ESHAPE, "snn_stdp_sequence: layer not supported by the persistent kernel "
                                 "(infinite threshold, or weights/scratch exceed shared memory)");
  return rc;
}

int snn_conv_fire_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta, int* path,
                       int* launches, int* chunks) {
  int rc = conv_checks(B, C, H, W, pad, F, KH, KW, T, theta);
  if (rc) return rc;
  REQUIRE(path && launches && chunks, SNN_EINVAL, "snn_conv_fire_plan: NULL output");
  return conv_fire_plan(B, C, H, W, pad, F, KH, KW, T, theta, path, launches, chunks);
}

int snn_conv_fire_ex(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH,
                     int KW, int T, float theta, int flags, uint8_t* lat_out, float* v_out, float* pot_out, void* ws,
                     size_t ws_bytes, snn_stream_t s) {
  int rc = conv_checks(B, C, H, W, pad, F, KH, KW, T, theta);
  if (rc) return rc;
  REQUIRE((flags & ~(SNN_CONV_OUT_NHWC | SNN_CONV_IN_NHWC | SNN_CONV_POOL2)) == 0, SNN_EINVAL,
          "snn_conv_fire: unknown flags 0x%x", flags);
  if (B == 0 || F == 0) return SNN_OK;
  REQUIRE(lat_in && w && lat_out, SNN_EINVAL, "snn_conv_fire: NULL tensor");
  REQUIRE(ws, SNN_EWORKSPACE, "snn_conv_fire: NULL workspace");
  return conv_fire_launch(lat_in, B, C, H, W, pad, w, F, KH, KW, T, theta, lat_out, v_out, pot_out, ws, ws_bytes,
                          S(s), (flags & SNN_CONV_OUT_NHWC) ? 1 : 0, (flags & SNN_CONV_IN_NHWC) ? 1 : 0,
                          (flags & SNN_CONV_POOL2) ? 1 : 0);
}

int snn_conv_fire(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F, int KH, int KW,
                  int T, float theta, uint8_t* lat_out, float* v_out, float* pot_out, void* ws, size_t ws_bytes,
                  snn_stream_t s) {
  return snn_conv_fire_ex(lat_in, B, C, H, W, pad, w, F, KH, KW, T, theta, 0, lat_out, v_out, pot_out, ws, ws_bytes,
                          s);
}

int snn_pool_ex(const uint8_t* lat, const float* v, int B, int F, int H, int W, int PH, int PW, int SH, int SW,
                int DH, int DW, int flags, uint8_t* lat_out, float* v_out, snn_stream_t s) {
  REQUIRE(B >= 0 && F >= 0 && H >= 1 && W >= 1, SNN_ESHAPE, "snn_pool: bad dimensions");
  REQUIRE(PH >= 1 && PW >= 1 && SH >= 1 && SW >= 1 && DH >= 0 && DW >= 0, SNN_EINVAL, "snn_pool: bad window");
  REQUIRE((flags & ~(SNN_POOL_EQ3 | SNN_POOL_VFINAL | SNN_POOL_IN_NHWC | SNN_POOL_OUT_NHWC)) == 0, SNN_EINVAL, "snn_pool: unknown flags 0x%x",
          flags);
  REQUIRE((flags & SNN_POOL_EQ3) ? (H + 2 * DH >= SH && W + 2 * DW >= SW) : (PH <= H + 2 * DH && PW <= W + 2 * DW),
          SNN_ESHAPE, "snn_pool: window larger than padded input");
  REQUIRE(DH < PH && DW < PW, SNN_EINVAL, "snn_pool: padding must be smaller than the window");
  if (int64_t(B) * F == 0) return SNN_OK;
  REQUIRE(lat && lat_out, SNN_EINVAL, "snn_pool: NULL tensor");
  REQUIRE(!v_out || v, SNN_EINVAL, "snn_pool: v_out without v");
  return pool_launch(lat, v, B, F, H, W, PH, PW, SH, SW, DH, DW, flags, lat_out, v_out, S(s));
}

int snn_pool(const uint8_t* lat, const float* v, int B, int F, int H, int W, int PH, int PW, int SH, int SW, int DH,
             int DW, uint8_t* lat_out, float* v_out, snn_stream_t s) {
  return snn_pool_ex(lat, v, B, F, H, W, PH, PW, SH, SW, DH, DW, 0, lat_out, v_out, s);
}

int snn_inhibit(const uint8_t* lat, const float* v, int B, int F, int H, int W, uint8_t* lat_out, float* v_out,
                int16_t* winner_f, snn_stream_t s) {
  REQUIRE(B >= 0 && F >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_inhibit: bad dimensions");
  REQUIRE(F <= 32767, SNN_ESHAPE, "snn_inhibit: F > 32767 (int16 winner map)");
  if (int64_t(B) * H * W == 0) return SNN_OK;
  REQUIRE(lat && v && lat_out && v_out, SNN_EINVAL, "snn_inhibit: NULL tensor");
  return inhibit_launch(lat, v, B, F, H, W, lat_out, v_out, winner_f, S(s));
}

size_t snn_k_winners_workspace(int B, int F, int H, int W) {
  if (B < 0 || F < 0 || H < 0 || W < 0) return 0;
  return k_winners_workspace(B, F, H, W);
}

int snn_k_winners(const uint8_t* lat, const float* v, int B, int F, int H, int W, int k, int r, int32_t* winners,
                  int32_t* count, void* ws, size_t ws_bytes, snn_stream_t s) {
  REQUIRE(k >= 1 && k <= 256, SNN_EINVAL, "snn_k_winners: k=%d outside [1, 256]", k);
  REQUIRE(r >= 0, SNN_EINVAL, "snn_k_winners: r < 0");
  REQUIRE(B >= 0 && F >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_k_winners: bad dimensions");
  REQUIRE(int64_t(F) * H * W <= (int64_t(1) << 24), SNN_ESHAPE, "snn_k_winners: F*H*W > 2^24");
  REQUIRE(F <= 8192, SNN_ESHAPE, "snn_k_winners: F > 8192");
  if (B == 0) return SNN_OK;
  REQUIRE(winners && count && (lat && v || int64_t(F) * H * W == 0), SNN_EINVAL, "snn_k_winners: NULL tensor");
  REQUIRE(ws, SNN_EWORKSPACE, "snn_k_winners: NULL workspace");
  return k_winners_launch(lat, v, B, F, H, W, k, r, winners, count, ws, ws_bytes, S(s));
}

static int stdp_update_impl(float* w, int F_local, int f_offset, int C, int KH, int KW, const uint8_t* lat_in, int H,
                            int W, int pad, const uint8_t* lat_out, int Ho, int Wo, const int32_t* winners,
                            const int32_t* count, int k, float a_plus, float a_minus, float lb, float ub,
                            int stabilizer, const float* reward, int sharded, snn_stream_t s) {
  const int F = F_local;
  REQUIRE(stabilizer >= 0 && stabilizer <= 2, SNN_EINVAL, "snn_stdp_update: stabilizer=%d not in {0, 1, 2}", stabilizer);
  REQUIRE(lb < ub, SNN_EINVAL, "snn_stdp_update: LB >= UB");
  REQUIRE(f_offset >= 0, SNN_EINVAL, "snn_stdp_update: f_offset < 0");
  REQUIRE(k >= 0 && F >= 1 && C >= 1 && KH >= 1 && KW >= 1 && H >= 1 && W >= 1 && pad >= 0, SNN_ESHAPE,
          "snn_stdp_update: bad dimensions");
  REQUIRE(Ho == H + 2 * pad - KH + 1 && Wo == W + 2 * pad - KW + 1, SNN_ESHAPE,
          "snn_stdp_update: lat_out %dx%d does not match Eq. 2 (%dx%d)", Ho, Wo, H + 2 * pad - KH + 1,
          W + 2 * pad - KW + 1);
  REQUIRE(!isnan(a_plus) && !isnan(a_minus), SNN_EINVAL, "snn_stdp_update: NaN rate");
  if (k == 0) return SNN_OK;
  REQUIRE(w && lat_in && lat_out && winners && count, SNN_EINVAL, "snn_stdp_update: NULL tensor");
  return stdp_launch(w, F, C, KH, KW, lat_in, H, W, pad, lat_out, Ho, Wo, winners, count, k, a_plus, a_minus, lb, ub,
                     stabilizer, reward, f_offset, sharded, S(s));
}

int snn_stdp_update_shard(float* w, int F_local, int f_offset, int C, int KH, int KW, const uint8_t* lat_in, int H,
                          int W, int pad, const uint8_t* lat_out, int Ho, int Wo, const int32_t* winners,
                          const int32_t* count, int k, float a_plus, float a_minus, float lb, float ub, int stabilizer,
                          const float* reward, snn_stream_t s) {
  return stdp_update_impl(w, F_local, f_offset, C, KH, KW, lat_in, H, W, pad, lat_out, Ho, Wo, winners, count, k,
                          a_plus, a_minus, lb, ub, stabilizer, reward, 1, s);
}

int snn_stdp_update(float* w, int F, int C, int KH, int KW, const uint8_t* lat_in, int H, int W, int pad,
                    const uint8_t* lat_out, int Ho, int Wo, const int32_t* winners, const int32_t* count, int k,
                    float a_plus, float a_minus, float lb, float ub, int stabilizer, const float* reward,
                    snn_stream_t s) {
  return stdp_update_impl(w, F, 0, C, KH, KW, lat_in, H, W, pad, lat_out, Ho, Wo, winners, count, k, a_plus,
                          a_minus, lb, ub, stabilizer, reward, 0, s);
}

int snn_position_keys(const uint8_t* lat, const float* v, int B, int F, int H, int W, int f_offset, int64_t* keys,
                      snn_stream_t s) {
  REQUIRE(B >= 0 && F >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_position_keys: negative dimension");
  REQUIRE(f_offset >= 0 && int64_t(f_offset) + F <= (int64_t(1) << 23), SNN_ESHAPE,
          "snn_position_keys: global feature index >= 2^23");
  REQUIRE(int64_t(H) * W < (int64_t(1) << 31), SNN_ESHAPE, "snn_position_keys: H*W >= 2^31");
  if (int64_t(B) * H * W == 0) return SNN_OK;
  REQUIRE(keys && (F == 0 || (lat && v)), SNN_EINVAL, "snn_position_keys: NULL tensor");
  return position_keys_launch(lat, v, B, F, H, W, f_offset, keys, S(s));
}

size_t snn_k_winners_keys_workspace(int B, int H, int W) {
  if (B < 0 || H < 0 || W < 0) return 0;
  return k_winners_keys_workspace(B, H, W);
}

int snn_k_winners_keys(const int64_t* keys, int B, int F, int H, int W, int k, int r, int32_t* winners,
                       int32_t* count, void* ws, size_t ws_bytes, snn_stream_t s) {
  REQUIRE(k >= 1 && k <= 256, SNN_EINVAL, "snn_k_winners_keys: k=%d outside [1, 256]", k);
  REQUIRE(r >= 0, SNN_EINVAL, "snn_k_winners_keys: r < 0");
  REQUIRE(B >= 0 && F >= 0 && H >= 0 && W >= 0, SNN_ESHAPE, "snn_k_winners_keys: bad dimensions");
  REQUIRE(int64_t(F) * H * W <= (int64_t(1) << 24), SNN_ESHAPE, "snn_k_winners_keys: F*H*W > 2^24");
  if (B == 0) return SNN_OK;
  REQUIRE(winners && count && (keys || int64_t(H) * W == 0), SNN_EINVAL, "snn_k_winners_keys: NULL tensor");
  return k_winners_keys_launch(keys, B, H, W, k, r, winners, count, ws, ws_bytes, S(s));
}

int snn_decide(const int32_t* winners, const int32_t* count, int B, int k, int F, int n_classes,
               const int32_t* labels, int32_t* decision, float* reward, snn_stream_t s) {
  REQUIRE(B >= 0 && k >= 1 && n_classes >= 1 && F >= n_classes && F % n_classes == 0, SNN_EINVAL,
          "snn_decide: need F divisible by n_classes");
  if (B == 0) return SNN_OK;
  REQUIRE(winners && count && (decision || reward), SNN_EINVAL, "snn_decide: NULL tensor");
  return decide_launch(winners, count, B, k, F, n_classes, labels, decision, reward, S(s));
}

}  // extern "C"
