/*
 * snn_oracle.c -- CPU ORACLE for the SpykeTorch spike-wave step (arxiv 1903.02440).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, constant or helper with the CUDA path in paper_1903_02440_b200/.
 *
 * Plain, slow, obviously-correct loops written from PAPER.md (cited "P:<line>")
 * and the readings listed in DESIGN.md §3 ("R<n>").  Floating point: potentials are
 * accumulated in fp64, which is exact for the configs' weights (R2/N1);
 * the STDP update is evaluated in fp32, the precision of the paper's PyTorch weight
 * tensors, in the operation order of Eq. 4 (R7).
 *
 * Every function is pinned by tests/test_oracle_*.py.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_NO_SPIKE 255 /* "the infinity symbol stands for no spike" */

/* ------------------------------------------------------------------------- */
/* a1: intensity -> latency ("divides all of the spikes into a pre-defined
 * number of spike bins", P:135 utils.Intensity2Latency).  Readings R1:
 * rank jointly over C*H*W, x > 0 spikes, ties by flat index, near-equal bins
 * with the earlier bins taking the remainder.                                */
/* ------------------------------------------------------------------------- */
typedef struct { float v; int64_t idx; } orc_item;

static int orc_item_cmp(const void* a, const void* b) {
    const orc_item* p = (const orc_item*)a;
    const orc_item* q = (const orc_item*)b;
    if (p->v > q->v) return -1; /* intensity descending */
    if (p->v < q->v) return 1;
    return (p->idx < q->idx) ? -1 : (p->idx > q->idx); /* then flat index ascending */
}

/* bins selects the bin-size rule ("pre-defined number of spike bins"; the paper does not fix
 * the sizes -- DESIGN.md R1 and the f3 variants):
 *   0 (R1, default): q = N / T, m = N % T; the first m bins hold q + 1 ranks, the rest q;
 *   1 (proportional): the entry of rank r gets bin floor(r * T / N);
 *   2 (floor): every bin holds q = N / T ranks; ranks >= T q never spike.                       */
void orc_encode_bins(const float* x, int64_t B, int64_t n, int T, int bins, uint8_t* lat) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b) {
        const float* xb = x + b * n;
        uint8_t* lb = lat + b * n;
        orc_item* items = (orc_item*)malloc(sizeof(orc_item) * (size_t)(n > 0 ? n : 1));
        int64_t N = 0;
        for (int64_t i = 0; i < n; ++i) {
            lb[i] = ORC_NO_SPIKE;
            if (xb[i] > 0.0f) { items[N].v = xb[i]; items[N].idx = i; ++N; }
        }
        qsort(items, (size_t)N, sizeof(orc_item), orc_item_cmp);
        int64_t q = N / T, m = N % T, rank = 0;
        if (bins == 1) {
            for (rank = 0; rank < N; ++rank) lb[items[rank].idx] = (uint8_t)((rank * T) / N);
        } else {
            for (int t = 0; t < T; ++t) {
                int64_t size = q + ((bins == 0 && t < m) ? 1 : 0);
                for (int64_t j = 0; j < size; ++j, ++rank) lb[items[rank].idx] = (uint8_t)t;
            }
        }
        free(items);
    }
}

void orc_encode(const float* x, int64_t B, int64_t n, int T, uint8_t* lat) { orc_encode_bins(x, B, n, T, 0, lat); }

/* Eq. 1: S[t,i] = 0 if t < T_i else 1; NO_SPIKE rows all zero. */
void orc_expand(const uint8_t* lat, int64_t B, int64_t n, int T, float* wave /* [B][T][n] */) {
    for (int64_t b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
            for (int64_t i = 0; i < n; ++i) {
                uint8_t l = lat[b * n + i];
                wave[(b * T + t) * n + i] = (l != ORC_NO_SPIKE && t >= l) ? 1.0f : 0.0f;
            }
}

/* ------------------------------------------------------------------------- */
/* a2: potentials.  Eq. 2 geometry on the zero-padded input (P:182,
 * R6: padding never spikes).  Definition (north_star): P[t,f,y,x] is the sum of
 * the weights of the inputs that spiked by t.  Written as a histogram over the
 * input spike times followed by a prefix sum along t.                        */
/* ------------------------------------------------------------------------- */
static inline uint8_t orc_lat_at(const uint8_t* lat_c, int H, int W, int yy, int xx) {
    if (yy < 0 || yy >= H || xx < 0 || xx >= W) return ORC_NO_SPIKE;
    return lat_c[(int64_t)yy * W + xx];
}

/* P for one neuron (f,y,x) of one image, written to P[0..T-1]. */
static void orc_neuron_potential(const uint8_t* lat_in, int C, int H, int W, int pad,
                                 const float* w, int KH, int KW, int T,
                                 int f, int y, int x, double* hist, double* P) {
    for (int t = 0; t < T; ++t) hist[t] = 0.0;
    for (int c = 0; c < C; ++c)
        for (int ky = 0; ky < KH; ++ky)
            for (int kx = 0; kx < KW; ++kx) {
                uint8_t l = orc_lat_at(lat_in + (int64_t)c * H * W, H, W, y + ky - pad, x + kx - pad);
                if (l != ORC_NO_SPIKE && l < T)
                    hist[l] += (double)w[(((int64_t)f * C + c) * KH + ky) * KW + kx];
            }
    double s = 0.0;
    for (int t = 0; t < T; ++t) { s += hist[t]; P[t] = s; }
}

/* Full potentials tensor of one image: P[T][F][Ho][Wo] (fp64). */
void orc_potentials(const uint8_t* lat_in, int C, int H, int W, int pad,
                    const float* w, int F, int KH, int KW, int T, double* P) {
    int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
    double* hist = (double*)malloc(sizeof(double) * T);
    double* p = (double*)malloc(sizeof(double) * T);
    for (int f = 0; f < F; ++f)
        for (int y = 0; y < Ho; ++y)
            for (int x = 0; x < Wo; ++x) {
                orc_neuron_potential(lat_in, C, H, W, pad, w, KH, KW, T, f, y, x, hist, p);
                for (int t = 0; t < T; ++t) P[(((int64_t)t * F + f) * Ho + y) * Wo + x] = p[t];
            }
    free(hist); free(p);
}

/* Brute-force twin, the way P:93 computes it: materialise S[t] (Eq. 1) and run a
 * direct valid cross-correlation of every time step. */
void orc_potentials_brute(const uint8_t* lat_in, int C, int H, int W, int pad,
                          const float* w, int F, int KH, int KW, int T, double* P) {
    int Hp = H + 2 * pad, Wp = W + 2 * pad;
    int Ho = Hp - KH + 1, Wo = Wp - KW + 1;
    double* S = (double*)calloc((size_t)C * Hp * Wp, sizeof(double));
    for (int t = 0; t < T; ++t) {
        for (int c = 0; c < C; ++c)
            for (int y = 0; y < Hp; ++y)
                for (int x = 0; x < Wp; ++x) {
                    uint8_t l = orc_lat_at(lat_in + (int64_t)c * H * W, H, W, y - pad, x - pad);
                    S[((int64_t)c * Hp + y) * Wp + x] = (l != ORC_NO_SPIKE && t >= l) ? 1.0 : 0.0;
                }
        for (int f = 0; f < F; ++f)
            for (int y = 0; y < Ho; ++y)
                for (int x = 0; x < Wo; ++x) {
                    double acc = 0.0;
                    for (int c = 0; c < C; ++c)
                        for (int ky = 0; ky < KH; ++ky)
                            for (int kx = 0; kx < KW; ++kx)
                                acc += (double)w[(((int64_t)f * C + c) * KH + ky) * KW + kx] *
                                       S[((int64_t)c * Hp + y + ky) * Wp + x + kx];
                    P[(((int64_t)t * F + f) * Ho + y) * Wo + x] = acc;
                }
    }
    free(S);
}

/* ------------------------------------------------------------------------- */
/* a3: fire (R3): spike iff P > theta; first-spike time = first such t;
 * v = fp32(P[lat]) = the thresholded potential at the spike (0 if none).
 * Infinite threshold = Eq. 5: only P[T-1] survives; a spike at T-1
 * iff P[T-1] > 0, v = fp32(P[T-1]).                                          */
/* ------------------------------------------------------------------------- */
static inline void orc_fire_one(const double* P, int T, float theta, int theta_inf,
                                uint8_t* lat, float* v) {
    if (theta_inf) {
        *lat = (P[T - 1] > 0.0) ? (uint8_t)(T - 1) : ORC_NO_SPIKE;
        *v = (float)P[T - 1];
        return;
    }
    *lat = ORC_NO_SPIKE;
    *v = 0.0f;
    for (int t = 0; t < T; ++t)
        if (P[t] > (double)theta) { *lat = (uint8_t)t; *v = (float)P[t]; return; }
}

/* P laid out [T][n]. */
void orc_fire(const double* P, int T, int64_t n, float theta, int theta_inf, uint8_t* lat, float* v) {
    double* p = (double*)malloc(sizeof(double) * T);
    for (int64_t i = 0; i < n; ++i) {
        for (int t = 0; t < T; ++t) p[t] = P[(int64_t)t * n + i];
        orc_fire_one(p, T, theta, theta_inf, lat + i, v + i);
    }
    free(p);
}

/* conv + fire for a batch (potentials of each neuron, then fire), OpenMP over images. */
void orc_conv_fire(const uint8_t* lat_in, int64_t B, int C, int H, int W, int pad,
                   const float* w, int F, int KH, int KW, int T, float theta, int theta_inf,
                   uint8_t* lat_out, float* v_out) {
    int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
    int64_t n_in = (int64_t)C * H * W, n_out = (int64_t)F * Ho * Wo;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b) {
        double* hist = (double*)malloc(sizeof(double) * T);
        double* p = (double*)malloc(sizeof(double) * T);
        for (int f = 0; f < F; ++f)
            for (int y = 0; y < Ho; ++y)
                for (int x = 0; x < Wo; ++x) {
                    int64_t o = b * n_out + ((int64_t)f * Ho + y) * Wo + x;
                    orc_neuron_potential(lat_in + b * n_in, C, H, W, pad, w, KH, KW, T, f, y, x, hist, p);
                    orc_fire_one(p, T, theta, theta_inf, lat_out + o, v_out + o);
                }
        free(hist); free(p);
    }
}

/* The same for a list of sampled neurons: neuron[i] = b*F*Ho*Wo + (f*Ho+y)*Wo + x. */
void orc_conv_fire_sample(const uint8_t* lat_in, int C, int H, int W, int pad,
                          const float* w, int F, int KH, int KW, int T, float theta, int theta_inf,
                          const int64_t* neuron, int64_t n_samples, uint8_t* lat_out, float* v_out,
                          double* p_out /* nullable [n_samples][T] */) {
    int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
    int64_t n_in = (int64_t)C * H * W, n_out = (int64_t)F * Ho * Wo;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_samples; ++i) {
        double hist[256], p[256];
        int64_t b = neuron[i] / n_out, r = neuron[i] % n_out;
        int f = (int)(r / ((int64_t)Ho * Wo)), y = (int)((r / Wo) % Ho), x = (int)(r % Wo);
        orc_neuron_potential(lat_in + b * n_in, C, H, W, pad, w, KH, KW, T, f, y, x, hist, p);
        orc_fire_one(p, T, theta, theta_inf, lat_out + i, v_out + i);
        if (p_out) for (int t = 0; t < T; ++t) p_out[i * T + t] = p[t];
    }
}

/* Synaptic events: F * sum over output positions of the number of
 * spiking inputs in the receptive field. */
int64_t orc_events(const uint8_t* lat_in, int64_t B, int C, int H, int W, int pad, int F, int KH, int KW) {
    int Ho = H + 2 * pad - KH + 1, Wo = W + 2 * pad - KW + 1;
    int64_t n_in = (int64_t)C * H * W, total = 0;
#pragma omp parallel for reduction(+ : total)
    for (int64_t b = 0; b < B; ++b)
        for (int y = 0; y < Ho; ++y)
            for (int x = 0; x < Wo; ++x)
                for (int c = 0; c < C; ++c)
                    for (int ky = 0; ky < KH; ++ky)
                        for (int kx = 0; kx < KW; ++kx)
                            total += orc_lat_at(lat_in + b * n_in + (int64_t)c * H * W, H, W,
                                                y + ky - pad, x + kx - pad) != ORC_NO_SPIKE;
    return total * F;
}

/* ------------------------------------------------------------------------- */
/* a4: pooling (Eq. 3).  Per time step, 2-D max-pooling of the
 * spike-wave S[t] and of the thresholded potentials thr(P)[t].  With the compact
 * (lat, v) input (v = P at the spike, R3) the pooled wave's first spike is the
 * first t at which the pooled S is 1, and the pooled thresholded potential at
 * that t is the max over the window of thr(P_i)[t], i.e. v_i for the neurons
 * that spiked by t (none spiked earlier, since t is the first).  Padding = no
 * spike (R11).  Output size per R10.                                        */
/* ------------------------------------------------------------------------- */
/* f3 variants: eq3 = 1 takes Eq. 3's output size literally,
 * Ho = floor((H + 2 DH) / SH), the last windows truncated at the
 * edge of the padded input (outside it nothing spikes, like the padding);
 * vfinal = 1 reads the pooled thresholded potentials at t = T-1 instead of at
 * the pooled spike time: the max of v over every window entry that spiked.     */
void orc_pool_ex(const uint8_t* lat, const float* v, int64_t B, int F, int H, int W,
                 int PH, int PW, int SH, int SW, int DH, int DW, int T, int eq3, int vfinal,
                 uint8_t* lat_out, float* v_out) {
    int Ho = eq3 ? (H + 2 * DH) / SH : (H + 2 * DH - PH) / SH + 1;
    int Wo = eq3 ? (W + 2 * DW) / SW : (W + 2 * DW - PW) / SW + 1;
#pragma omp parallel for schedule(static)
    for (int64_t bf = 0; bf < B * F; ++bf) {
        const uint8_t* l = lat + bf * H * W;
        const float* vv = v ? v + bf * H * W : NULL;
        for (int oy = 0; oy < Ho; ++oy)
            for (int ox = 0; ox < Wo; ++ox) {
                uint8_t lo = ORC_NO_SPIKE;
                float vo = 0.0f;
                for (int t = 0; t < T && lo == ORC_NO_SPIKE; ++t) {
                    int s = 0;
                    for (int py = 0; py < PH; ++py)
                        for (int px = 0; px < PW; ++px) {
                            uint8_t li = orc_lat_at(l, H, W, oy * SH + py - DH, ox * SW + px - DW);
                            if (li != ORC_NO_SPIKE && t >= li) s = 1;
                        }
                    if (s) {
                        lo = (uint8_t)t;
                        const int tr = vfinal ? T - 1 : t; /* time at which the pooled potential is read */
                        for (int py = 0; py < PH; ++py)
                            for (int px = 0; px < PW; ++px) {
                                int yy = oy * SH + py - DH, xx = ox * SW + px - DW;
                                uint8_t li = orc_lat_at(l, H, W, yy, xx);
                                if (li != ORC_NO_SPIKE && tr >= li && vv) {
                                    float c = vv[(int64_t)yy * W + xx];
                                    if (c > vo) vo = c;
                                }
                            }
                    }
                }
                lat_out[(bf * Ho + oy) * Wo + ox] = lo;
                if (v_out) v_out[(bf * Ho + oy) * Wo + ox] = vo;
            }
    }
}

void orc_pool(const uint8_t* lat, const float* v, int64_t B, int F, int H, int W,
              int PH, int PW, int SH, int SW, int DH, int DW, int T,
              uint8_t* lat_out, float* v_out) {
    orc_pool_ex(lat, v, B, F, H, W, PH, PW, SH, SW, DH, DW, T, 0, 0, lat_out, v_out);
}

/* ------------------------------------------------------------------------- */
/* a5: pointwise inhibition: at each location only the most salient
 * feature may spike -- "the earliest spike with the highest potential";
 * remaining ties by lowest feature index (R14).                             */
/* ------------------------------------------------------------------------- */
void orc_inhibit(const uint8_t* lat, const float* v, int64_t B, int F, int H, int W,
                 uint8_t* lat_out, float* v_out, int16_t* winner_f) {
    int64_t HW = (int64_t)H * W;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t p = 0; p < HW; ++p) {
            int best = -1;
            for (int f = 0; f < F; ++f) {
                int64_t i = (b * F + f) * HW + p;
                if (lat[i] == ORC_NO_SPIKE) continue;
                if (best < 0) { best = f; continue; }
                int64_t j = (b * F + best) * HW + p;
                if (lat[i] < lat[j] || (lat[i] == lat[j] && v[i] > v[j])) best = f;
            }
            for (int f = 0; f < F; ++f) {
                int64_t i = (b * F + f) * HW + p;
                lat_out[i] = (f == best) ? lat[i] : ORC_NO_SPIKE;
                v_out[i] = (f == best) ? v[i] : 0.0f;
            }
            if (winner_f) winner_f[b * HW + p] = (int16_t)best;
        }
}

/* ------------------------------------------------------------------------- */
/* a6: k winners-take-all.  Up to k rounds; each round the
 * winner is the candidate with the earliest spike, then the highest potential
 * (R13: v at the spike), then the lowest flat index f*H*W + y*W + x (R14).
 * After a pick, the winner's feature map and the Chebyshev-radius-r square
 * around it in all maps are inhibited (R15).  Written naively: every round scans
 * all F*H*W neurons.                                                         */
/* ------------------------------------------------------------------------- */
int orc_k_winners(const uint8_t* lat, const float* v, int F, int H, int W, int k, int r,
                  int32_t* winners /* [k][3] */) {
    int64_t n = (int64_t)F * H * W;
    uint8_t* excluded = (uint8_t*)calloc((size_t)n, 1);
    int count = 0;
    for (int i = 0; i < k; ++i) winners[3 * i] = winners[3 * i + 1] = winners[3 * i + 2] = -1;
    for (int round = 0; round < k; ++round) {
        int64_t best = -1;
        for (int64_t i = 0; i < n; ++i) {
            if (excluded[i] || lat[i] == ORC_NO_SPIKE) continue;
            if (best < 0 || lat[i] < lat[best] || (lat[i] == lat[best] && v[i] > v[best])) best = i;
        }
        if (best < 0) break;
        int f = (int)(best / ((int64_t)H * W)), y = (int)((best / W) % H), x = (int)(best % W);
        winners[3 * count] = f; winners[3 * count + 1] = y; winners[3 * count + 2] = x;
        ++count;
        for (int ff = 0; ff < F; ++ff)
            for (int yy = 0; yy < H; ++yy)
                for (int xx = 0; xx < W; ++xx)
                    if (ff == f || (abs(yy - y) <= r && abs(xx - x) <= r))
                        excluded[((int64_t)ff * H + yy) * W + xx] = 1;
    }
    free(excluded);
    return count;
}

void orc_k_winners_batch(const uint8_t* lat, const float* v, int64_t B, int F, int H, int W, int k, int r,
                         int32_t* winners, int32_t* count) {
    int64_t n = (int64_t)F * H * W;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b)
        count[b] = orc_k_winners(lat + b * n, v + b * n, F, H, W, k, r, winners + b * 3 * k);
}

/* ------------------------------------------------------------------------- */
/* a7: STDP, Eq. 4.  For winner i (post) and each synapse j of its
 * receptive field: dW = A+ (W-LB)(UB-W) if T_j <= T_i else A- (W-LB)(UB-W);
 * NO_SPIKE / padded pre counts as T_j > T_i (R17); stabilizer off => dW = A;
 * then clamp to [LB, UB] (R20) -- except stabilizer == 2 (stabilizer on, no clamp:
 * the A20 variant "clamp only when the stabilizer is off").  fp32, Eq. 4 left-to-right, no FMA (R19).
 * R-STDP: reward = +1 applies (A+, A-), -1 applies the negated
 * rates (anti-STDP), 0 = no update (silent, R25).                            */
/* ------------------------------------------------------------------------- */
void orc_stdp(float* w, int F, int C, int KH, int KW,
              const uint8_t* lat_in, int H, int W, int pad,
              const uint8_t* lat_out, int Ho, int Wo,
              const int32_t* winners, int count,
              float a_plus, float a_minus, float lb, float ub, int stabilizer, int reward) {
    if (reward == 0) return;
    float ap = reward > 0 ? a_plus : -a_plus;
    float am = reward > 0 ? a_minus : -a_minus;
    (void)F;
    for (int i = 0; i < count; ++i) {
        int f = winners[3 * i], y = winners[3 * i + 1], x = winners[3 * i + 2];
        uint8_t post = lat_out[((int64_t)f * Ho + y) * Wo + x];
        for (int c = 0; c < C; ++c)
            for (int ky = 0; ky < KH; ++ky)
                for (int kx = 0; kx < KW; ++kx) {
                    uint8_t pre = orc_lat_at(lat_in + (int64_t)c * H * W, H, W, y + ky - pad, x + kx - pad);
                    float a = (pre != ORC_NO_SPIKE && pre <= post) ? ap : am;
                    float* wp = &w[(((int64_t)f * C + c) * KH + ky) * KW + kx];
                    float W0 = *wp;
                    float dw;
                    if (stabilizer) {
                        float t1 = a * (W0 - lb);
                        dw = t1 * (ub - W0);
                    } else {
                        dw = a;
                    }
                    float w1 = W0 + dw;
                    if (stabilizer != 2) { /* 2: stabilizer on, no clamp (A20 variant) */
                        if (w1 < lb) w1 = lb;
                        if (w1 > ub) w1 = ub;
                    }
                    *wp = w1;
                }
    }
}

/* R-STDP decision (R24/R25): decision = decision_map[f] with the
 * block map f / (F / n_classes); +1 if it equals the label, -1 otherwise,
 * 0 (and decision -1) when silent. */
int orc_decide(const int32_t* winners, int count, int F, int n_classes, int label, int* decision) {
    if (count <= 0) { *decision = -1; return 0; }
    *decision = winners[0] / (F / n_classes);
    return (*decision == label) ? 1 : -1;
}

/* ------------------------------------------------------------------------- */
/* f2: the input-transform front end of the paper's pipeline  */
/* ("utils.Filter ... DoG and Gabor kernels", "intensity_lateral_   */
/* inhibition ... local_normalization", P:232 InputTransform).  The paper gives   */
/* intent only; the readings R33-R35 follow SPEC.md's definitions.    */
/* ------------------------------------------------------------------------- */

/* R33: zero-padded cross-correlation of [B][H][W] fp64 images with [K][S][S] fp64
 * kernels, fp64 sum over (dy, dx) in row-major kernel order, one multiply
 * and one add per term (no fused multiply-add), then per mode:
 *   mode 0: out[b][k] = r, values below `threshold` set to 0 (SPEC apply_filter_bank);
 *   mode 1: DoG on/off split, out[b][2k] = max(r, 0), out[b][2k+1] = max(-r, 0);
 *   mode 2: rectified, out[b][k] = max(r, 0) (Gabor).
 * Output fp32 (round to nearest), [B][Kout][Ho][Wo], Ho = H + 2 pad - S + 1.       */
void orc_filter_bank(const double* img, int64_t B, int H, int W, const double* ker, int K, int S, int pad,
                     double threshold, int mode, float* out) {
    const int Ho = H + 2 * pad - S + 1, Wo = W + 2 * pad - S + 1;
    const int Kout = mode == 1 ? 2 * K : K;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < B; ++b) {
        const double* im = img + b * (int64_t)H * W;
        for (int k = 0; k < K; ++k) {
            const double* kk = ker + (int64_t)k * S * S;
            for (int y = 0; y < Ho; ++y) {
                for (int x = 0; x < Wo; ++x) {
                    double r = 0.0;
                    for (int dy = 0; dy < S; ++dy) {
                        for (int dx = 0; dx < S; ++dx) {
                            const int yy = y + dy - pad, xx = x + dx - pad;
                            const double p = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? im[(int64_t)yy * W + xx] : 0.0;
                            const double term = p * kk[dy * S + dx];
                            r = r + term;
                        }
                    }
                    const int64_t o = (int64_t)y * Wo + x;
                    if (mode == 0) {
                        out[((b * Kout) + k) * (int64_t)Ho * Wo + o] = (float)(r < threshold ? 0.0 : r);
                    } else if (mode == 1) {
                        out[((b * Kout) + 2 * k) * (int64_t)Ho * Wo + o] = (float)(r > 0.0 ? r : 0.0);
                        out[((b * Kout) + 2 * k + 1) * (int64_t)Ho * Wo + o] = (float)(-r > 0.0 ? -r : 0.0);
                    } else {
                        out[((b * Kout) + k) * (int64_t)Ho * Wo + o] = (float)(r > 0.0 ? r : 0.0);
                    }
                }
            }
        }
    }
}

/* R34: local normalization ("uses regional mean for normalizing intensity
 * values"): out = x / max(mean of the (2 radius + 1)^2 window around it, eps), the
 * window truncated at the borders (SPEC); fp64 window sum in row-major order, the
 * mean as sum / count, the division in fp64, output fp32.                           */
void orc_local_norm(const float* x, int64_t B, int C, int H, int W, int radius, double eps, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t bc = 0; bc < B * C; ++bc) {
        const float* xc = x + bc * (int64_t)H * W;
        float* oc = out + bc * (int64_t)H * W;
        for (int y = 0; y < H; ++y) {
            for (int xx = 0; xx < W; ++xx) {
                double s = 0.0;
                int cnt = 0;
                for (int yy = y - radius; yy <= y + radius; ++yy) {
                    if (yy < 0 || yy >= H) continue;
                    for (int x2 = xx - radius; x2 <= xx + radius; ++x2) {
                        if (x2 < 0 || x2 >= W) continue;
                        s = s + (double)xc[(int64_t)yy * W + x2];
                        ++cnt;
                    }
                }
                double m = s / (double)cnt;
                if (m < eps) m = eps;
                oc[(int64_t)y * W + xx] = (float)((double)xc[(int64_t)y * W + xx] / m);
            }
        }
    }
}

/* R35: intensity lateral inhibition ("decreases the surrounding intensities
 * ... of each salient point"), SPEC's sweep: locations are processed in descending
 * order of their ORIGINAL intensity (ties: row-major index ascending); each processed
 * location multiplies every strictly weaker location of the same channel within
 * Chebyshev distance n (1 <= d <= n) by factors[d - 1].  Done literally: sort, sweep,
 * fp32 multiplications in sweep order.                                                */
typedef struct { float v; int idx; } orc_li_item;
static int orc_li_cmp(const void* a, const void* b) {
    const orc_li_item* p = (const orc_li_item*)a;
    const orc_li_item* q = (const orc_li_item*)b;
    if (p->v > q->v) return -1;
    if (p->v < q->v) return 1;
    return (p->idx < q->idx) ? -1 : (p->idx > q->idx);
}
void orc_lateral_inhibition(const float* x, int64_t B, int C, int H, int W, const float* factors, int n,
                            float* out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t bc = 0; bc < B * C; ++bc) {
        const float* xc = x + bc * (int64_t)H * W;
        float* oc = out + bc * (int64_t)H * W;
        orc_li_item* it = (orc_li_item*)malloc(sizeof(orc_li_item) * (size_t)H * W);
        for (int i = 0; i < H * W; ++i) { it[i].v = xc[i]; it[i].idx = i; oc[i] = xc[i]; }
        qsort(it, (size_t)H * W, sizeof(orc_li_item), orc_li_cmp);
        for (int s = 0; s < H * W; ++s) {
            const int p = it[s].idx, py = p / W, px = p % W;
            const float vp = xc[p];
            for (int yy = py - n; yy <= py + n; ++yy) {
                if (yy < 0 || yy >= H) continue;
                for (int x2 = px - n; x2 <= px + n; ++x2) {
                    if (x2 < 0 || x2 >= W || (yy == py && x2 == px)) continue;
                    const int q = yy * W + x2;
                    if (!(xc[q] < vp)) continue; /* only strictly weaker neighbours */
                    const int dy = yy > py ? yy - py : py - yy, dx = x2 > px ? x2 - px : px - x2;
                    const int d = dy > dx ? dy : dx;
                    oc[q] = oc[q] * factors[d - 1];
                }
            }
        }
        free(it);
    }
}
