/*
 * snn.h -- C ABI of libsnn, the B200 (sm_100a) spike-wave step of a convolutional SNN with at
 * most one spike per neuron (SpykeTorch, arxiv 1903.02440).  Citations: "P:<line>" = a line of
 * the paper's text, "R<n>" = a reading recorded in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Every tensor argument is a DEVICE pointer owned by the caller (allocated e.g. by torch).  The
 *    library never allocates, frees or caches device memory; scratch space comes from a caller
 *    buffer sized by the matching *_workspace() call.
 *  - Every call is asynchronous on the given CUDA stream (`snn_stream_t` = cudaStream_t; NULL =
 *    legacy default stream) and never synchronises.
 *  - Layouts are row-major (C order).  A latency grid is uint8 with SNN_NO_SPIKE = 255 for "no
 *    spike" (the paper's infinity); valid spike times are 0..T-1 with 1 <= T <= 254.
 *  - Return codes: SNN_OK (0) or a negative SNN_E* code.  Host-side argument checks run before any
 *    launch; on error nothing is launched and snn_last_error() returns a message (thread-local).
 *    Device-detected conditions (e.g. a weight outside the exact domain, see snn_conv_fire) set a
 *    device error word that snn_sync_status() reports.
 *  - Functions are stateless and thread-safe.  Plasticity calls on one weight tensor must be
 *    serialised by the caller (single writer).
 */
#ifndef SNN_H_
#define SNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* snn_stream_t;

#if defined(__GNUC__)
#define SNN_API __attribute__((visibility("default")))
#else
#define SNN_API
#endif

#define SNN_NO_SPIKE 255

#define SNN_OK 0
#define SNN_EINVAL (-1)     /* bad scalar argument (T range, k < 1, NaN threshold, LB >= UB, ...) */
#define SNN_ESHAPE (-2)     /* shape rule violated (kernel larger than padded input, index overflow) */
#define SNN_ECUDA (-3)      /* a CUDA launch / runtime call failed */
#define SNN_EINEXACT (-4)   /* device: a weight is outside the exact fixed-point domain (N1) */
#define SNN_EWORKSPACE (-5) /* workspace pointer NULL or smaller than *_workspace() */

/* ---------------------------------------------------------------------------------------------
 * f2. Front end: the preprocessing ahead of a1.  Each output is bit-identical
 * to the definition stated (explicitly rounded operations in the stated order, no FMA).  Outputs
 * must not alias inputs.  No workspace.
 *
 * snn_filter_bank (P:133 utils.Filter; DoG P:223, Gabor P:232; reading R33):
 *   img fp64 [B, H, W] grayscale images; kernels fp64 [K, S, S] (the DoG/Gabor taps, built by the
 *   caller); out fp32 [B, Kout, Ho, Wo], Ho = H + 2 pad - S + 1, Wo likewise.  For each kernel k,
 *   r = sum over (dy, dx) in row-major order of img[y + dy - pad, x + dx - pad] * kernels[k, dy, dx]
 *   (cross-correlation, zero outside the image) accumulated in fp64.  mode 0: out[k] = r < threshold
 *   ? 0 : r (Kout = K); mode 1 (on/off DoG): out[2k] = max(r, 0), out[2k+1] = max(-r, 0) (Kout = 2K);
 *   mode 2: out[k] = max(r, 0) (Kout = K).  Each cast to fp32 rounds to nearest.
 *   Requires 1 <= S <= 31, 0 <= pad < S, Ho, Wo >= 1, K >= 1, the taps and the 8 x 32 tile's halo
 *   within 200 KB of shared memory (SNN_ESHAPE otherwise); mode in {0, 1, 2} (SNN_EINVAL).
 * snn_local_norm ("uses regional mean for normalizing intensity values"; reading R34):
 *   x, out fp32 [B, C, H, W]; out = x / max(m, eps) with m = (fp64 sum, row-major, of the window
 *   [y - radius, y + radius] x [x - radius, x + radius] truncated at the borders) / (its size),
 *   the division in fp64.  Requires 0 <= radius <= 32, eps > 0.
 * snn_lateral_inhibition (P:126 intensity lateral inhibition; reading R35):
 *   x, out fp32 [B, C, H, W]; factors fp32 [n] (device).  Per (b, c) plane, locations are visited in
 *   (x descending, flat index y W + x ascending) order; visiting p multiplies (fp32) the running value
 *   of every location q with x[q] < x[p] and Chebyshev distance d = max(|dy|, |dx|) in [1, n] by
 *   factors[d - 1].  out starts as x.  Requires 0 <= n <= 32 (n = 0 copies).
 * ------------------------------------------------------------------------------------------- */
SNN_API int snn_filter_bank(const double* img, int B, int H, int W, const double* kernels, int K, int S, int pad,
                            double threshold, int mode, float* out, snn_stream_t s);
SNN_API int snn_local_norm(const float* x, int B, int C, int H, int W, int radius, double eps, float* out,
                           snn_stream_t s);
SNN_API int snn_lateral_inhibition(const float* x, int B, int C, int H, int W, const float* factors, int n,
                                   float* out, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * a1. Intensity -> latency encoding (P:51, P:135 utils.Intensity2Latency; readings R1, R2).
 * x   : float32 [B, C, H, W] intensities.  Per image, the N strictly positive entries (x > 0;
 *       zero, negative and NaN never spike) are ranked by (value descending, flat index c*H*W +
 *       y*W + x ascending) and split into T bins: with q = N / T and m = N % T the first m bins hold
 *       q + 1 entries and the others q.  lat = bin index of the entry's rank.
 * lat : uint8 [B, C, H, W] output; SNN_NO_SPIKE for non-positive entries.
 * Requires 1 <= T <= 254 and C*H*W < 2^24.  Workspace: snn_encode_workspace(B, C, H, W, T).
 * ------------------------------------------------------------------------------------------- */
SNN_API size_t snn_encode_workspace(int B, int C, int H, int W, int T);
SNN_API int snn_encode(const float* x, int B, int C, int H, int W, int T, uint8_t* lat,
               void* ws, size_t ws_bytes, snn_stream_t s);

/* f3 variant of a1 (the paper's "pre-defined number of spike bins", leaves the bin
 * sizes open).  bins: SNN_BINS_R1 = snn_encode; SNN_BINS_PROPORTIONAL = the entry of rank r gets
 * floor(r T / N); SNN_BINS_FLOOR = every bin holds q = N / T entries and ranks >= T q never spike
 * (N < T: nothing spikes).  Same workspace, arguments and errors as snn_encode (bins unknown:
 * SNN_EINVAL). */
#define SNN_BINS_R1 0
#define SNN_BINS_PROPORTIONAL 1
#define SNN_BINS_FLOOR 2
/* or'ed into bins: lat is written channels-last [B, H, W, C] (the ranking still uses the planar flat
 * index c*H*W + y*W + x; only the storage changes) -- the input layout of snn_conv_fire_ex
 * SNN_CONV_IN_NHWC. */
#define SNN_ENCODE_OUT_NHWC 0x100
SNN_API int snn_encode_ex(const float* x, int B, int C, int H, int W, int T, int bins, uint8_t* lat,
                          void* ws, size_t ws_bytes, snn_stream_t s);

/* Eq. 1: wave[b, t, i] = 1.0f if lat[b, i] != NO_SPIKE and t >= lat[b, i], else 0.
 * lat uint8 [B, n], wave float32 [B, T, n].  Validation / tests only (the hot path never
 * materialises waves). */
SNN_API int snn_expand(const uint8_t* lat, int B, int n, int T, float* wave, snn_stream_t s);

/* Count entries of lat[n] that are neither < T nor NO_SPIKE (an invalid latency); the count is
 * written (not accumulated) to *n_bad (int32, device). */
SNN_API int snn_validate_lat(const uint8_t* lat, size_t n, int T, int32_t* n_bad, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * a2 + a3. Spiking convolution fused with threshold firing.
 * Potentials (Eq. 2; R5, R6): for output neuron (f, y, x) of image b,
 *   P[t] = sum over c, ky, kx of w[f, c, ky, kx] * [lat_in[b, c, y+ky-pad, x+kx-pad] <= t],
 * a valid stride-1 cross-correlation of the zero-padded spike-wave (padding never spikes);
 * Ho = H + 2*pad - KH + 1, Wo = W + 2*pad - KW + 1.
 * Fire (R3): lat_out = min{t < T : P[t] > theta}, else NO_SPIKE; v_out = fp32(P[lat_out])
 * (round-to-nearest of the exact potential), 0 if no spike.  theta = +INFINITY selects Eq. 5
 * (R9): lat_out = T-1 iff P[T-1] > 0 and v_out = fp32(P[T-1]).
 * Exactness (N1): potentials are accumulated exactly as integers in units of 2^-31, so
 * every weight must satisfy w*2^31 integral and 0 <= w <= 1 (true for every w in {0} U [2^-8, 1]).
 * A weight outside that domain sets the device error word (SNN_EINEXACT at snn_sync_status()).
 *   lat_in  uint8 [B, C, H, W];   w float32 [F, C, KH, KW]
 *   lat_out uint8 [B, F, Ho, Wo]; v_out float32 [B, F, Ho, Wo] or NULL (not written)
 *   pot_out float32 [B, T, F, Ho, Wo] or NULL: if non-NULL every fp32(P[t]) is written (validation
 *           mode, no early exit).
 * Workspace: snn_conv_fire_workspace(..., theta) bytes.  theta = +inf without pot_out runs the
 * tensor-core path (tcgen05 kind::i8, exact 4-limb split of the fixed-point weights); its workspace
 * holds the binary im2col of S[T-1] (positions x C*KH*KW bytes) and the weight limbs.  A kernel larger
 * than the input map (H*W < KH*KW, e.g. 5 x 5 on a 4 x 4 map) runs as one fully connected contraction per
 * image over the H*W*C input pixels instead (same Eq. 5 values, no im2col; K9).
 * Finite theta: any receptive field R = C*KH*KW up to ~65,000 entries (a sorted list's u16 bucket
 * starts); a layer whose weight slice does not fit shared memory (R above ~1,700 for 32 features)
 * walks from the prepared slice in global memory (L2).  With pot_out (validation mode) the weight
 * slice must fit shared memory: SNN_ESHAPE otherwise.
 * ------------------------------------------------------------------------------------------- */
SNN_API size_t snn_conv_fire_workspace(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T,
                                       float theta);
SNN_API int snn_conv_fire(const uint8_t* lat_in, int B, int C, int H, int W, int pad,
                  const float* w, int F, int KH, int KW, int T, float theta,
                  uint8_t* lat_out, float* v_out, float* pot_out,
                  void* ws, size_t ws_bytes, snn_stream_t s);

/* snn_conv_fire with options (same arguments, workspace and errors; flags = 0 is snn_conv_fire).
 *   SNN_CONV_OUT_NHWC  lat_out and v_out are channels-last [B, Ho, Wo, F] (pot_out keeps its layout).
 *                      The finite-threshold walk assigns features to lanes, so a position's outputs
 *                      are contiguous in this layout and its stores coalesce (the planar layout puts
 *                      every feature in a separate plane); snn_pool_ex(SNN_POOL_IN_NHWC) reads it.
 *   SNN_CONV_IN_NHWC   lat_in is channels-last [B, H, W, C] (snn_encode_ex SNN_ENCODE_OUT_NHWC,
 *                      snn_pool_ex SNN_POOL_OUT_NHWC): a receptive field is KH x KW runs of C contiguous
 *                      bytes.  Not with pot_out or SNN_CONV_PATH=tct/ref (SNN_EINVAL).
 * v_out may be NULL in both calls: the potentials are then not written (a layer whose consumer only
 * needs spike times, e.g. latency-only pooling).  Unknown flag bits: SNN_EINVAL. */
#define SNN_CONV_OUT_NHWC 1
#define SNN_CONV_IN_NHWC 2
/*   SNN_CONV_POOL2     (with SNN_CONV_OUT_NHWC | SNN_CONV_IN_NHWC, a finite theta, v_out = pot_out = NULL):
 *                      lat_out receives the 2 x 2 / stride 2 / unpadded latency pooling of the layer's
 *                      spike times instead of the spike times themselves -- [B, Ho/2, Wo/2, F] channels-last
 *                      (floor; the pooled map of snn_pool_ex(lat, NULL, ..., 2, 2, 2, 2, 0, 0,
 *                      SNN_POOL_IN_NHWC | SNN_POOL_OUT_NHWC), Eq. 3 with A10/A11/A12), fused
 *                      into the row-tile walk (the unpooled map never reaches memory).  SNN_EINVAL for the
 *                      other options; SNN_ESHAPE (before any launch) when the row-tile walk does not apply
 *                      (latency-sized batches, F > 32, receptive fields past its shared-memory budget) --
 *                      the caller then runs snn_conv_fire_ex + snn_pool_ex. */
#define SNN_CONV_POOL2 4
SNN_API int snn_conv_fire_ex(const uint8_t* lat_in, int B, int C, int H, int W, int pad, const float* w, int F,
                             int KH, int KW, int T, float theta, int flags, uint8_t* lat_out, float* v_out,
                             float* pot_out, void* ws, size_t ws_bytes, snn_stream_t s);

/* Sequential theta = +inf layers (C4's R-STDP layer: one image at a time, new weights every image).
 * The A operand of Eq. 5 (the binary im2col of each image's S[T-1]) does not depend on the weights, so
 * snn_conv_inf_prepare builds it for all B images of lat_in [B, C, H, W] at once into `prep`
 * (snn_conv_inf_prepare_bytes(B, ...) bytes, caller-owned); snn_conv_fire_prepared then runs the
 * conv of image b of that batch with the current weights w: exactly snn_conv_fire(lat_in[b], w, pad, T,
 * +inf, ...) (bit-identical), minus the A preparation.  lat_out, v_out [1, F, Ho, Wo]; workspace
 * snn_conv_fire_workspace(1, C, H, W, pad, F, KH, KW, T, +inf).  Same argument errors as snn_conv_fire;
 * prep smaller than required: SNN_EWORKSPACE. */
SNN_API size_t snn_conv_inf_prepare_bytes(int B, int C, int H, int W, int pad, int F, int KH, int KW);
SNN_API int snn_conv_inf_prepare(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW,
                                 int T, void* prep, size_t prep_bytes, snn_stream_t s);
SNN_API int snn_conv_fire_prepared(const void* prep, int b, int C, int H, int W, int pad, const float* w, int F,
                                   int KH, int KW, int T, uint8_t* lat_out, float* v_out, void* ws, size_t ws_bytes,
                                   snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * snn_rstdp_inf_sequence -- SURVEY.md §8(f) f1 for a theta = +inf plastic layer (C4's R-STDP layer):
 * N sequential images, each: conv Eq. 5 of image b0 + i of a snn_conv_inf_prepare batch `prep` with
 * the current w -> the single winner = snn_k_winners(k = 1, r = 0) of that map (R13/R14)
 * -> decision[i] / reward[i] as snn_decide with labels[i] (R24/R25; labels NULL: reward
 * 0) -> snn_stdp_update of the winner (Eq. 4 with post = T - 1, rates negated for reward -1, skipped
 * for 0 or no winner, R17-R23), w updated in place.  Bit-identical to those calls made image
 * by image.  lat_in uint8 [N, C, H, W] (the layer input of the N images, planar, for the pre-synaptic
 * times); w fp32 [F, C, KH, KW]; winners int32 [N, 3] (f, y, x; -1 when silent); count int32 [N];
 * decision int32 [N] and reward fp32 [N] nullable.  Per image three kernels (a split-K tcgen05 GEMM,
 * the winner/decision kernel and Eq. 4 with the re-quantisation of the winner's weights only); no host
 * synchronisation.  SNN_RSTDP_PERSIST=1 runs the whole chain as one cooperative kernel instead (same
 * results; measured slower on C4's shape).  Workspace: snn_rstdp_inf_workspace (0 = unsupported shape).
 * Errors: as snn_conv_fire (theta = +inf) and snn_stdp_update; F*Ho*Wo > 2^24: SNN_ESHAPE.
 * ------------------------------------------------------------------------------------------- */
SNN_API size_t snn_rstdp_inf_workspace(int C, int H, int W, int pad, int F, int KH, int KW);
SNN_API int snn_rstdp_inf_sequence(const void* prep, int b0, int N, int C, int H, int W, int pad,
                                   const uint8_t* lat_in, float* w, int F, int KH, int KW, int T,
                                   const int32_t* labels, int n_classes, float a_plus, float a_minus, float lb,
                                   float ub, int stabilizer, int32_t* winners, int32_t* count, int32_t* decision,
                                   float* reward, void* ws, size_t ws_bytes, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * a4. Spike-wave max-pooling (Eq. 3; readings R10-R12).
 * Window PH x PW, stride SH x SW, zero padding DH x DW (padding never spikes).
 * Ho = (H + 2*DH - PH) / SH + 1, Wo = (W + 2*DW - PW) / SW + 1 (windows inside the padded input).
 * lat_out = min of lat over the window (earliest spike); v_out = max of v over the window entries
 * whose lat equals lat_out (0 if none): the per-time-step max-pool of the thresholded potentials
 * read at the pooled spike time.  v / v_out may both be NULL (latencies only).
 *   lat, v [B, F, H, W] -> lat_out, v_out [B, F, Ho, Wo]
 * ------------------------------------------------------------------------------------------- */
SNN_API int snn_pool(const uint8_t* lat, const float* v, int B, int F, int H, int W,
             int PH, int PW, int SH, int SW, int DH, int DW,
             uint8_t* lat_out, float* v_out, snn_stream_t s);

/* f3 variants of a4.  flags (bitwise or):
 *   SNN_POOL_EQ3    output size per Eq. 3 literally: Ho = (H + 2 DH) / SH,
 *                   Wo = (W + 2 DW) / SW; windows reaching past the padded input are truncated.
 *                   Requires H + 2 DH >= SH and W + 2 DW >= SW instead of the window rule.
 *   SNN_POOL_VFINAL v_out = max of v over EVERY spiking entry of the window (the pooled potentials
 *                   tensor at t = T - 1, for v = final potentials: the A13 tie-break variant).
 *   SNN_POOL_IN_NHWC / SNN_POOL_OUT_NHWC channels-last layouts (below); combine with the other two.
 * flags = 0 is snn_pool.  Unknown bits: SNN_EINVAL. */
#define SNN_POOL_EQ3 1
#define SNN_POOL_VFINAL 2
#define SNN_POOL_IN_NHWC 4  /* lat, v are channels-last [B, H, W, F] (snn_conv_fire_ex SNN_CONV_OUT_NHWC);
                               lat_out, v_out are [B, F, Ho, Wo] unless SNN_POOL_OUT_NHWC.  Requires
                               H*W*F < 2^32; planar output also B, Ho <= 65535. */
#define SNN_POOL_OUT_NHWC 8 /* with SNN_POOL_IN_NHWC only: lat_out, v_out channels-last [B, Ho, Wo, F]
                               (the input layout of snn_conv_fire_ex SNN_CONV_IN_NHWC) */
SNN_API int snn_pool_ex(const uint8_t* lat, const float* v, int B, int F, int H, int W, int PH, int PW, int SH,
                        int SW, int DH, int DW, int flags, uint8_t* lat_out, float* v_out, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * a5. Pointwise (cross-feature) inhibition (R13, R14).  At each (b, y, x) the spiking
 * feature with the smallest key (lat ascending, v descending, f ascending) keeps its (lat, v);
 * every other feature becomes (NO_SPIKE, 0).  winner_f[b, y, x] = that feature or -1 (may be
 * NULL).  lat, v, lat_out, v_out: [B, F, H, W]; winner_f int16 [B, H, W].
 * ------------------------------------------------------------------------------------------- */
SNN_API int snn_inhibit(const uint8_t* lat, const float* v, int B, int F, int H, int W,
                uint8_t* lat_out, float* v_out, int16_t* winner_f, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * a6. k winners-take-all with inhibition radius r (R13-R15).  Up to k rounds
 * per image: the winner is the non-excluded spiking neuron with the smallest key (lat ascending,
 * v descending, flat index f*H*W + y*W + x ascending); then its whole feature map and every neuron
 * at Chebyshev distance <= r from (y, x) in all maps are excluded.  Stops early when no candidate
 * is left (fewer than k winners is legal).
 *   winners int32 [B, k, 3] = (feature, row, column), rows past count[b] are -1.
 *   count   int32 [B].
 * Requires k >= 1, r >= 0, F*H*W <= 2^24.  Workspace: snn_k_winners_workspace(B, F, H, W).
 * ------------------------------------------------------------------------------------------- */
SNN_API size_t snn_k_winners_workspace(int B, int F, int H, int W);
SNN_API int snn_k_winners(const uint8_t* lat, const float* v, int B, int F, int H, int W, int k, int r,
                  int32_t* winners, int32_t* count, void* ws, size_t ws_bytes, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * a7. STDP / R-STDP weight update of ONE image, in place (Eq. 4; R17-R23).
 * For each winner (f, y, x) among winners[0 .. count[0]-1] and each synapse (c, ky, kx):
 *   pre  = lat_in[c, y+ky-pad, x+kx-pad] (NO_SPIKE outside the input), post = lat_out[f, y, x];
 *   a    = A+ if pre != NO_SPIKE and pre <= post, else A-;
 *   dW   = (a * (W - lb)) * (ub - W) if stabilizer else a;   W = clamp(W + dW, lb, ub)
 * stabilizer: 0 off, 1 on, 2 on WITHOUT the clamp (f3 variant A20, "clamp only when the stabilizer
 * is off"); other values SNN_EINVAL.  Evaluated in fp32 round-to-nearest without FMA contraction.  Winners have distinct features
 * (snn_k_winners guarantees it), so synapse updates never collide.
 * reward (device float scalar, may be NULL = +1): +1 applies (A+, A-), -1 applies (-A+, -A-)
 * (anti-STDP), 0 skips the update (silent sample).
 *   w        float32 [F, C, KH, KW] (in/out)
 *   lat_in   uint8 [C, H, W];  lat_out uint8 [F, Ho, Wo]
 *   winners  int32 [k, 3];     count int32 [1]
 * ------------------------------------------------------------------------------------------- */
SNN_API int snn_stdp_update(float* w, int F, int C, int KH, int KW,
                    const uint8_t* lat_in, int H, int W, int pad,
                    const uint8_t* lat_out, int Ho, int Wo,
                    const int32_t* winners, const int32_t* count, int k,
                    float a_plus, float a_minus, float lb, float ub, int stabilizer,
                    const float* reward, snn_stream_t s);

/* R-STDP decision on device (R24, R25): for each image b, decision[b] =
 * winners[b, 0, 0] / (F / n_classes) (the block decision_map) or -1 when count[b] == 0 (silent);
 * reward[b] = +1 if decision == labels[b], -1 if it differs, 0 when silent.  labels may be NULL
 * (reward then 0).  winners [B, k, 3], count [B], labels int32 [B], decision int32 [B],
 * reward float32 [B] (reward may be NULL). */
SNN_API int snn_decide(const int32_t* winners, const int32_t* count, int B, int k, int F, int n_classes,
               const int32_t* labels, int32_t* decision, float* reward, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * snn_stdp_sequence -- N sequential plasticity steps of one conv layer in ONE persistent kernel
 * (P:95).  For image i = 0..N-1, in order:
 *   conv + fire of lat_in[i] with the current weights (Eq. 2, theta finite, R3-R8),
 *   pointwise inhibition (R13/R14), k-WTA with radius r on the inhibited map (R15),
 *   STDP (Eq. 4, R17-R20) of the winners' weights, in place,
 * exactly as snn_conv_fire + snn_inhibit + snn_k_winners + snn_stdp_update called image by image
 * (bit-identical results).  lat_in uint8 [N, C, H, W]; w fp32 [F, C, KH, KW] (in place, every
 * weight in the exact domain of N1); winners int32 [N, k, 3] (-1 padded) and count int32 [N] are
 * written for every image; snapshots (nullable) fp32 [N / snap_every, F, C, KH, KW] receive the
 * weights after images snap_every, 2 snap_every, ...  Workspace: snn_stdp_sequence_workspace.
 * Cooperative launch (one CTA per SM, grid-wide barriers between the stages of an image).
 * Errors: as snn_conv_fire; SNN_ESHAPE if theta is infinite or the layer's weight slice / scratch
 * does not fit shared memory (use the per-call functions then); SNN_EINVAL for k outside [1, 256],
 * r < 0, lb >= ub, snap_every < 1 with snapshots.  SNN_EINEXACT (device) as snn_conv_fire.
 * ------------------------------------------------------------------------------------------- */
SNN_API size_t snn_stdp_sequence_workspace(int N, int C, int H, int W, int pad, int F, int KH, int KW, int T, int k);
SNN_API int snn_stdp_sequence(const uint8_t* lat_in, int N, int C, int H, int W, int pad, float* w, int F, int KH,
                              int KW, int T, float theta, int k, int r, float a_plus, float a_minus, float lb,
                              float ub, int stabilizer, int32_t* winners, int32_t* count, float* snapshots,
                              int snap_every, void* ws, size_t ws_bytes, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * f4. Feature sharding across GPUs.  Each rank owns the
 * contiguous features [f_offset, f_offset + F) of a layer.  Per image: snn_conv_fire on the rank's
 * weights -> snn_position_keys -> all-reduce(MIN) of the int64 keys over ranks (NCCL, by the caller)
 * -> snn_k_winners_keys (identical on every rank) -> snn_stdp_update_shard.  Bit-identical to the
 * unsharded snn_inhibit + snn_k_winners + snn_stdp_update.
 *
 * snn_position_keys: keys int64 [B, H, W] = min over the rank's features of the packed key
 *   (lat << 55) | (~order(v) << 23) | (f_offset + f)   -- ascending = (lat asc, v desc, f asc), the
 *   pointwise-inhibition order (R13/R14); SNN_KEY_NONE where none of them spikes.  Keys are
 *   non-negative, so a signed MIN reduction combines ranks.  lat, v [B, F, H, W].
 *   Requires f_offset + F <= 2^23.
 * snn_k_winners_keys: k-WTA (R15) on the inhibited map the keys describe (at most one candidate
 *   per position): winners int32 [B, k, 3] (global f, y, x; -1 padded), count int32 [B]; F = the
 *   layer's total feature count (for the F*H*W <= 2^24 index check).  Workspace
 *   snn_k_winners_keys_workspace(B, H, W) (used when H*W*8 B exceeds shared memory).
 * snn_stdp_update_shard: snn_stdp_update on the rank's weights w [F_local, C, KH, KW] and lat_out
 *   [F_local, Ho, Wo]; winners carry global features, those outside [f_offset, f_offset + F_local)
 *   are skipped (another rank owns them).
 * ------------------------------------------------------------------------------------------- */
#define SNN_KEY_NONE INT64_MAX
SNN_API int snn_position_keys(const uint8_t* lat, const float* v, int B, int F, int H, int W, int f_offset,
                              int64_t* keys, snn_stream_t s);
SNN_API size_t snn_k_winners_keys_workspace(int B, int H, int W);
SNN_API int snn_k_winners_keys(const int64_t* keys, int B, int F, int H, int W, int k, int r, int32_t* winners,
                               int32_t* count, void* ws, size_t ws_bytes, snn_stream_t s);
SNN_API int snn_stdp_update_shard(float* w, int F_local, int f_offset, int C, int KH, int KW, const uint8_t* lat_in,
                                  int H, int W, int pad, const uint8_t* lat_out, int Ho, int Wo,
                                  const int32_t* winners, const int32_t* count, int k, float a_plus, float a_minus,
                                  float lb, float ub, int stabilizer, const float* reward, snn_stream_t s);

/* ---------------------------------------------------------------------------------------------
 * Measurement helpers (off the hot path).
 * snn_count_events writes two uint64 counters to out[0..1] (device), overwriting them:
 *   out[0] = synaptic events as the paper's delta contraction defines them: F * sum over output
 *            positions of the number of spiking inputs in the receptive field;
 *   out[1] = necessary events: sum over output neurons of the number of receptive-field inputs that
 *            spiked at or before the neuron's first spike lat_out (all spiking inputs if it never
 *            fires) -- the inputs any exact first-spike computation must add.  0 if lat_out is NULL.
 *   lat_in uint8 [B, C, H, W], lat_out uint8 [B, F, Ho, Wo] or NULL.
 * snn_launch_count returns the number of kernels this process has launched through libsnn.
 * snn_conv_fire_plan (host only, no GPU needed) describes what one snn_conv_fire call with the same
 *   scalars (pot_out NULL) launches: *path = 0 fused sort+walk, 1 presorted walk (a sort and a walk
 *   kernel per list chunk, *chunks of them), 2 tensor-core Eq. 5 (theta = +inf), 3 tensor-core
 *   time-stepped (SNN_CONV_PATH=tct), 4 validation kernel, 5 presorted walk gathering its weights
 *   from global memory (receptive fields too large for shared memory); *launches = kernels per call.  Same
 *   argument errors as snn_conv_fire.
 * ------------------------------------------------------------------------------------------- */
SNN_API int snn_count_events(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int F, int KH, int KW,
                             int T, const uint8_t* lat_out, unsigned long long* out, snn_stream_t s);
SNN_API unsigned long long snn_launch_count(void);
SNN_API int snn_conv_fire_plan(int B, int C, int H, int W, int pad, int F, int KH, int KW, int T, float theta,
                               int* path, int* launches, int* chunks);

/* ---------------------------------------------------------------------------------------------
 * Status.
 * snn_sync_status synchronises the stream, then returns and clears the device error word
 * (SNN_OK, SNN_EINEXACT) or SNN_ECUDA if the stream reported a CUDA error.
 * snn_last_error returns the calling thread's last host-side error message ("" if none).
 * snn_version returns the ABI version (currently 1).
 * ------------------------------------------------------------------------------------------- */
SNN_API int snn_sync_status(snn_stream_t s);
SNN_API const char* snn_last_error(void);
SNN_API int snn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SNN_H_ */
