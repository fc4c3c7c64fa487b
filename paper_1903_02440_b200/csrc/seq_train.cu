// seq_train.cu -- SURVEY.md §8(f) f1: the per-image plasticity chain (conv + fire -> pointwise
// inhibition -> k-WTA -> STDP, image after image; each image's weights feed the next) as ONE
// persistent cooperative kernel, so the chain pays no kernel launch or host interaction per image
// (the paper's residual cost).  Same arithmetic as the separate kernels (N1,
// K2, K3, R13-R23), so results are bit-identical to snn_conv_fire + snn_inhibit + snn_k_winners +
// snn_stdp_update run image by image.
//
// Grid: one CTA per SM (cooperative launch: all CTAs resident), CTA c holds feature group
// g = c % n_groups (FGS = 32 * FPL features) as fixed-point weights in shared memory for the whole
// run.  Per image:
//   A  every CTA walks its share of the output positions for its group (fused receptive-field sort +
//      delta walk, K2/K3) and writes (lat, v) of its features to a one-image scratch map;
//   -- grid barrier --
//   B  CTA 0: pointwise inhibition (best key per position over all features, R13/R14: the minimum of
//      the per-group bests phase A left) and the k-WTA rounds on the inhibited map (one candidate per
//      position, R15): winners, their post times;
//   -- grid barrier --
//   C  every CTA applies Eq. 4 to the winners of its group in its shared-memory copy (old weights
//      recovered exactly from the fixed point); the group's leader CTA also writes the fp32 weights
//      (and the snapshots).  The next image's phase A uses the updated shared-memory copy.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "walk_dev.cuh"

namespace snn {

struct SeqArgs {
  WalkArgs wa;              // geometry of one image (B = 1), smem layout, threshold
  const uint8_t* lat_all;   // [N][C][H][W] layer input of every image
  int N;
  float* w;                 // [F][R] fp32, updated in place
  int k, r;
  float a_plus, a_minus, lb, ub;
  int stabilizer;
  float* snaps;             // nullable [N / snap_every][F][R]
  int snap_every;
  uint8_t* lat_map;         // [F][Ho][Wo] one-image scratch
  float* v_map;
  int32_t* winners;         // [N][k][3]
  int32_t* count;           // [N]
  int32_t* post;            // [N][k] post-synaptic spike time of each winner
  uint64_t* gbest;          // [n_groups][HoWo] best inhibition key of each group at each position
  uint64_t* stamps;         // [N][6] CTA-0 phase timestamps (globaltimer ns), timing diagnostics
  unsigned* bar;            // grid barrier words [2] (zeroed before the launch)
  int n_groups, FGS;
  int off_keys;             // CTA 0 scratch: per-position candidate keys [HoWo] u64
  int dbg;                  // timing experiments only (SNN_SEQ_DBG): 1 = skip conv, 2 = skip inhibit/kWTA, 4 = skip STDP
  const unsigned char* lists;  // [N][HoWo] presorted receptive-field records (rf_sort_lists_launch)
  int rec, hdr, npre, buf_bytes;
};

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).  gen = barriers passed so far.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = gen;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(&bar[1], g + 1);
    } else {
      const uint64_t t0 = globaltimer_ns();
      for (;;) {
        unsigned cur;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
        if (cur != g) break;
        __nanosleep(64);
        watchdog(t0);
      }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

template <int FPL>
__global__ void __launch_bounds__(FPL == 4 ? 768 : 1024, 1) seq_train_kernel(const SeqArgs s) {
  constexpr int FGS = 32 * FPL;
  extern __shared__ __align__(16) unsigned char smem[];
  const WalkArgs& a = s.wa;
  const int R = a.R, F = a.F, HoWo = a.Ho * a.Wo;
  uint32_t* Wsh = reinterpret_cast<uint32_t*>(smem);  // [R+1][FGS] fixed point
  int32_t* eoff = reinterpret_cast<int32_t*>(smem + a.off_eoff);
  uint16_t* ekk = reinterpret_cast<uint16_t*>(smem + a.off_ekk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  unsigned char* pb = smem + a.off_warps + warp * a.warp_bytes;  // [2 mbarriers][2 record buffers]
  uint64_t* pmb = reinterpret_cast<uint64_t*>(pb);
  unsigned char* pbuf = pb + 16;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem + s.off_keys);  // [HoWo] candidate keys
  uint16_t* fpos = reinterpret_cast<uint16_t*>(keys + HoWo);           // [HoWo] candidate features
  uint16_t* ypos = fpos + HoWo;                                         // [HoWo] row, column of each position
  uint16_t* xpos = ypos + HoWo;
  __shared__ int s_count;
  const int g = int(blockIdx.x) % s.n_groups;
  const int cg = int(blockIdx.x) / s.n_groups, ncg = int(gridDim.x) / s.n_groups;
  const bool leader = cg == 0;
  const int fbase = g * FGS + lane * FPL;
  unsigned valid = 0;
#pragma unroll
  for (int j = 0; j < FPL; ++j) valid |= (fbase + j < F) ? (1u << j) : 0u;
  const unsigned char* wl = smem + lane * FPL * 4;
  const int64_t CHW = int64_t(a.C) * a.H * a.W;

  // the group's weights -> fixed point (exact domain checked), row R = 0
  for (int i = tid; i < (R + 1) * FGS; i += blockDim.x) {
    const int e = i / FGS, f = g * FGS + (i - e * FGS);
    uint32_t u = 0;
    if (f < F && e < R) {
      const float x = s.w[int64_t(f) * R + e];
      const float sx = x * 2147483648.0f;
      if (!(x >= 0.0f && x <= 1.0f) || sx != truncf(sx)) flag_error(a.err, kErrInexact);
      else u = uint32_t(sx);
    }
    Wsh[i] = u;
  }
  (void)eoff; (void)ekk;
  for (int pos = tid; pos < HoWo; pos += blockDim.x) {  // (row, col) of every position, for phase B
    ypos[pos] = uint16_t(pos / a.Wo);
    xpos[pos] = uint16_t(pos - (pos / a.Wo) * a.Wo);
  }
  // this warp's positions: pos0 + j * pstride (the same every image); records prefetched one item ahead
  const int pstride = ncg * nwarps, pos0 = cg + ncg * warp;
  auto rec_of = [&](int im, int pos) { return s.lists + (int64_t(im) * HoWo + pos) * s.rec; };
  if (lane == 0) {
    mbar_init(smem_u32(&pmb[0]), 1);
    mbar_init(smem_u32(&pmb[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (pos0 < HoWo && s.N > 0) {
      mbar_expect_tx(smem_u32(&pmb[0]), uint32_t(s.buf_bytes));
      bulk_g2s(smem_u32(pbuf), rec_of(0, pos0), uint32_t(s.buf_bytes), smem_u32(&pmb[0]));
    }
  }
  __syncthreads();
  unsigned gen = 0;
  int item = 0;  // walks done by this warp (buffer / phase bookkeeping)

  for (int img = 0; img < s.N; ++img) {
    const uint8_t* lat_img = s.lat_all + int64_t(img) * CHW;
    if (blockIdx.x == 0 && tid == 0) s.stamps[img * 6 + 0] = globaltimer_ns();
    if (img == 100 && tid == 0) s.stamps[int64_t(s.N) * 6 + blockIdx.x * 2] = globaltimer_ns();
    // ---------------- A: conv + fire of this CTA's positions, this group's features ----------------
    // positions round-robin over the group's CTAs first, so a small map spreads over all SMs
    for (int pos = pos0; pos < ((s.dbg & 1) ? 0 : HoWo); pos += pstride, ++item) {
      const int bi = item & 1;
      if (lane == 0) {  // prefetch this warp's next (image, position) record into the other buffer
        int nim = img, npos = pos + pstride;
        if (npos >= HoWo) { ++nim; npos = pos0; }
        if (nim < s.N) {
          mbar_expect_tx(smem_u32(&pmb[bi ^ 1]), uint32_t(s.buf_bytes));
          bulk_g2s(smem_u32(pbuf + (bi ^ 1) * s.buf_bytes), rec_of(nim, npos), uint32_t(s.buf_bytes),
                   smem_u32(&pmb[bi ^ 1]));
        }
      }
      mbar_wait(smem_u32(&pmb[bi]), (item >> 1) & 1);
      const uint16_t* start = reinterpret_cast<const uint16_t*>(pbuf + bi * s.buf_bytes);
      uint32_t lo;
      float vo[FPL];
      walk_list<FPL, 1, true>(a, wl, start, pbuf + bi * s.buf_bytes + s.hdr, rec_of(img, pos) + s.hdr, nullptr,
                              true, valid, 0xffffffffu, lo, vo);
      uint64_t best = ~uint64_t(0);  // this group's inhibition candidate at pos (R13/R14: key over f)
#pragma unroll
      for (int j = 0; j < FPL; ++j)
        if (valid >> j & 1) {
          const uint8_t l = uint8_t(lo >> (8 * j));
          s.lat_map[int64_t(fbase + j) * HoWo + pos] = l;
          s.v_map[int64_t(fbase + j) * HoWo + pos] = vo[j];
          if (l != kNoSpike) {
            const uint64_t kk = wta_key(l, vo[j], uint32_t(fbase + j));
            best = kk < best ? kk : best;
          }
        }
      best = warp_min_u64(best);
      if (lane == 0) s.gbest[int64_t(g) * HoWo + pos] = best;
      __syncwarp();
    }
    if (blockIdx.x == 0) { __syncthreads(); if (tid == 0) s.stamps[img * 6 + 1] = globaltimer_ns(); }
    if (img == 100) { __syncthreads(); if (tid == 0) s.stamps[int64_t(s.N) * 6 + blockIdx.x * 2 + 1] = globaltimer_ns(); }
    grid_barrier(s.bar, gen);
    if (blockIdx.x == 0 && tid == 0) s.stamps[img * 6 + 2] = globaltimer_ns();
    // ---------------- B (CTA 0): pointwise inhibition, then k-WTA on the inhibited map ----------------
    if (blockIdx.x == 0 && !(s.dbg & 2)) {
      for (int pos = tid; pos < HoWo; pos += blockDim.x) {  // best (lat, v, f) per position over the groups
        uint64_t best = ~uint64_t(0);
        for (int gg = 0; gg < s.n_groups; ++gg) {
          const uint64_t kk = s.gbest[int64_t(gg) * HoWo + pos];
          best = kk < best ? kk : best;
        }
        uint64_t cand = ~uint64_t(0);  // the survivor's k-WTA key: flat index f * HoWo + pos (R14)
        if (best != ~uint64_t(0)) cand = (best & ~uint64_t(0xFFFFFFu)) | uint64_t(uint32_t(best & 0xFFFFFFu) * HoWo + pos);
        keys[pos] = cand;
        fpos[pos] = best != ~uint64_t(0) ? uint16_t(best & 0xFFFFFFu) : uint16_t(0xFFFF);
      }
      __syncthreads();
      if (img == 100 && tid == 0) s.stamps[int64_t(s.N) * 6 + 400] = globaltimer_ns();
      if (warp == 0) {  // k-WTA rounds by one warp (no block barriers)
        // inhibited map: one candidate key per position; a round's winner kills the positions of its
        // feature and those within Chebyshev distance r (R15), so each round is a plain warp min
        int nwin = 0;
        auto emit = [&](uint64_t best, int f, int yy, int xx) {
          if (lane == 0) {
            int32_t* wrec = s.winners + (int64_t(img) * s.k + nwin) * 3;
            wrec[0] = f; wrec[1] = yy; wrec[2] = xx;
            s.post[int64_t(img) * s.k + nwin] = int(best >> 56);  // the winner's spike time (key bits 56..63)
          }
        };
        if (HoWo <= 32 * 8 && a.Ho <= 256 && a.Wo <= 256) {
          // small maps: every lane keeps its <= 8 positions' keys and (f, y, x) in registers
          uint64_t kr[8];
          uint32_t fxy[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = lane + 32 * j;
            kr[j] = pos < HoWo ? keys[pos] : ~uint64_t(0);
            fxy[j] = pos < HoWo ? (uint32_t(fpos[pos]) << 16 | uint32_t(ypos[pos]) << 8 | uint32_t(xpos[pos])) : 0u;
          }
          for (int round = 0; round < s.k; ++round) {
            uint64_t mine = ~uint64_t(0);
#pragma unroll
            for (int j = 0; j < 8; ++j) mine = kr[j] < mine ? kr[j] : mine;
            const uint32_t hi = __reduce_min_sync(0xffffffffu, uint32_t(mine >> 32));
            const uint32_t lo = __reduce_min_sync(0xffffffffu, uint32_t(mine >> 32) == hi ? uint32_t(mine) : ~0u);
            const uint64_t best = uint64_t(hi) << 32 | lo;
            if (best == ~uint64_t(0)) break;  // no candidate left
            uint32_t w = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) w = kr[j] == best ? fxy[j] : w;
            const int src = __ffs(__ballot_sync(0xffffffffu, mine == best)) - 1;
            w = __shfl_sync(0xffffffffu, w, src);
            const int f = int(w >> 16), yy = int(w >> 8 & 0xFFu), xx = int(w & 0xFFu);
            emit(best, f, yy, xx);
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // branchless: one select per slot
              const int fj = int(fxy[j] >> 16), yj = int(fxy[j] >> 8 & 0xFFu), xj = int(fxy[j] & 0xFFu);
              const bool kill = (fj == f) | ((abs(yj - yy) <= s.r) & (abs(xj - xx) <= s.r));
              kr[j] = kill ? ~uint64_t(0) : kr[j];
            }
            ++nwin;
          }
        } else {
          for (int round = 0; round < s.k; ++round) {
            uint64_t best = ~uint64_t(0);
            for (int pos = lane; pos < HoWo; pos += 32) {
              const uint64_t kk = keys[pos];
              best = kk < best ? kk : best;
            }
            best = warp_min_u64(best);
            if (best == ~uint64_t(0)) break;  // no candidate left
            const int idx = int(best & 0xFFFFFFu);
            const int f = idx / HoWo, p = idx - f * HoWo;
            const int yy = p / a.Wo, xx = p - yy * a.Wo;
            emit(best, f, yy, xx);
            for (int pos = lane; pos < HoWo; pos += 32)
              if (int(fpos[pos]) == f || (abs(int(ypos[pos]) - yy) <= s.r && abs(int(xpos[pos]) - xx) <= s.r))
                keys[pos] = ~uint64_t(0);
            __syncwarp();
            ++nwin;
          }
        }
        if (lane == 0) s_count = nwin;
      }
      __syncthreads();
      if (img == 100 && tid == 0) s.stamps[int64_t(s.N) * 6 + 401] = globaltimer_ns();
      for (int i = s_count + tid; i < s.k; i += blockDim.x) {  // unused winner slots: -1
        int32_t* wrec = s.winners + (int64_t(img) * s.k + i) * 3;
        wrec[0] = -1; wrec[1] = -1; wrec[2] = -1;
      }
      if (tid == 0) s.count[img] = s_count;
      __syncthreads();
      if (tid == 0) s.stamps[img * 6 + 3] = globaltimer_ns();
    }
    grid_barrier(s.bar, gen);
    if (blockIdx.x == 0 && tid == 0) s.stamps[img * 6 + 4] = globaltimer_ns();
    // ---------------- C: Eq. 4 on this group's winners (shared-memory copy; leader writes fp32) ----------------
    {
      const int nwin = (s.dbg & 4) ? 0 : s.count[img];
      const int KK = a.KH * a.KW;
      for (int i = 0; i < nwin; ++i) {
        const int32_t* wrec = s.winners + (int64_t(img) * s.k + i) * 3;
        const int f = wrec[0], y = wrec[1], x = wrec[2];
        if (f < g * FGS || f >= g * FGS + FGS) continue;
        const int fl = f - g * FGS;
        const int post = s.post[int64_t(img) * s.k + i];
        for (int e = tid; e < R; e += blockDim.x) {
          const int c = e / KK, rr = e - c * KK, ky = rr / a.KW, kx = rr - ky * a.KW;
          const int yy = y + ky - a.pad, xx = x + kx - a.pad;
          int pre = kNoSpike;
          if (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W) pre = lat_img[(int64_t(c) * a.H + yy) * a.W + xx];
          const float am = (pre != kNoSpike && pre <= post) ? s.a_plus : s.a_minus;  // T_j <= T_i -> LTP
          const float w0 = __uint2float_rn(Wsh[e * FGS + fl]) * 4.656612873077392578125e-10f;  // exact
          const float dw = s.stabilizer ? __fmul_rn(__fmul_rn(am, __fsub_rn(w0, s.lb)), __fsub_rn(s.ub, w0)) : am;
          float w1 = __fadd_rn(w0, dw);
          if (s.stabilizer != 2) {  // 2 = stabilized without the clamp (A20 variant)
            w1 = w1 < s.lb ? s.lb : w1;
            w1 = w1 > s.ub ? s.ub : w1;
          }
          const float sx = w1 * 2147483648.0f;
          if (!(w1 >= 0.0f && w1 <= 1.0f) || sx != truncf(sx)) flag_error(a.err, kErrInexact);
          Wsh[e * FGS + fl] = uint32_t(sx);
          if (leader) s.w[int64_t(f) * R + e] = w1;
        }
      }
      if (leader && s.snaps && (img + 1) % s.snap_every == 0) {
        __syncthreads();
        float* snap = s.snaps + int64_t((img + 1) / s.snap_every - 1) * F * R;
        const int f0 = g * FGS, f1 = f0 + FGS < F ? f0 + FGS : F;
        for (int64_t i = int64_t(f0) * R + tid; i < int64_t(f1) * R; i += blockDim.x) snap[i] = s.w[i];
      }
      __syncthreads();
      if (blockIdx.x == 0 && tid == 0) s.stamps[img * 6 + 5] = globaltimer_ns();
    }
  }
}

// ------------------------------------------------------------------------------------- host
struct SeqPlan {
  int fpl, n_groups, FGS, nwarps, smem, grid;
  WalkArgs a;
  int off_keys;
  int rec, hdr, npre, buf_bytes;  // presorted records and the per-warp prefetch buffers
};

static int al16h(int x) { return (x + 15) & ~15; }

static bool seq_plan(int C, int H, int W, int pad, int F, int KH, int KW, int T, SeqPlan* pl) {
  WalkArgs& a = pl->a;
  a = WalkArgs{};
  a.B = 1; a.C = C; a.H = H; a.W = W; a.pad = pad; a.F = F; a.KH = KH; a.KW = KW; a.T = T;
  a.Ho = H + 2 * pad - KH + 1; a.Wo = W + 2 * pad - KW + 1; a.R = C * KH * KW;
  const int R = a.R;
  if (a.Ho < 1 || a.Wo < 1 || list_cap(R, T) >= 65536 || F > 8192) return false;
  a.pad_unit = 4;  // bucket-by-bucket walk (walk_list default)
  const int HoWo = a.Ho * a.Wo;
  if (int64_t(F) * HoWo >= (int64_t(1) << 24)) return false;
  // Latency-bound (one image at a time): when one walk per (position, 32-feature group) fits in a wave
  // of warps, the narrowest groups give the shortest critical walk (measured C3: FPL 4 43.1k, 2 49.7k,
  // 1 50.1k img/s); larger maps take the widest groups that fit.
  const bool one_wave = int64_t(HoWo) * ceil_div(F, 32) <= int64_t(num_sms()) * 32;
  const int fpls[3] = {one_wave ? 1 : 4, 2, one_wave ? 4 : 1};
  for (int i = 0; i < 3; ++i) {
    const int fpl = fpls[i], fgs = 32 * fpl;
    if (fpl > 1 && F <= fgs / 2) continue;  // lanes would idle
    if (const char* e = getenv("SNN_SEQ_FPL"))  // tuning experiments: force the features per lane
      if (atoi(e) != fpl) continue;
    const int nwarps = fpl == 4 ? 24 : 32;
    a.row_bytes = fgs * 4;
    const int wsb = al16h((R + 1) * fgs * 4);
    pl->hdr = al16h((T + 1) * 2);
    pl->rec = pl->hdr + int((list_cap(R, T) + kIt - 1) / kIt) * kIt * 4;
    // per warp: 2 mbarriers + 2 record buffers [header | up to 256 prefetched entries]
    const long left = (220L * 1024 - wsb - al16h(HoWo * 8) - al16h(HoWo * 6)) / nwarps - 16;
    int npre = int(((left / 2 - pl->hdr) / 4) / kIt) * kIt;
    const int full = pl->rec - pl->hdr;
    if (npre > full / 4) npre = full / 4;
    if (npre > 256) npre = 256;
    if (npre < kIt) continue;
    pl->npre = npre;
    pl->buf_bytes = pl->hdr + npre * 4;
    a.off_eoff = wsb; a.off_ekk = wsb;
    a.off_warps = wsb;
    a.warp_bytes = 16 + 2 * pl->buf_bytes;
    const int off_keys = a.off_warps + nwarps * a.warp_bytes;
    const int smem = off_keys + al16h(HoWo * 8) + al16h(HoWo * 6);
    if (smem > 220 * 1024) continue;
    pl->fpl = fpl; pl->FGS = fgs; pl->nwarps = nwarps; pl->smem = smem; pl->off_keys = off_keys;
    pl->n_groups = (F + fgs - 1) / fgs;
    pl->grid = (num_sms() / pl->n_groups) * pl->n_groups;
    if (pl->grid < pl->n_groups) return false;
    a.np = HoWo;
    return true;
  }
  return false;
}

static size_t r256(size_t x) { return (x + 255) & ~size_t(255); }
// workspace: [barrier words 256 B][lat_map F*HoWo][v_map F*HoWo*4][post N*k*4][gbest n_groups*HoWo*8]
//            [stamps N*48][presorted records N*HoWo*rec][slack]
size_t seq_train_workspace(int C, int H, int W, int pad, int F, int KH, int KW, int T, int k, int N) {
  SeqPlan pl;
  if (!seq_plan(C, H, W, pad, F, KH, KW, T, &pl)) return 0;
  const size_t HoWo = size_t(pl.a.Ho) * pl.a.Wo;
  return 256 + r256(size_t(F) * HoWo) + r256(size_t(F) * HoWo * 4) + r256(size_t(N) * k * 4) +
         r256(size_t(pl.n_groups) * HoWo * 8) + r256(size_t(N) * 48 + 16384) + r256(size_t(N) * HoWo * pl.rec) + 4096;
}

int rf_sort_lists_launch(const uint8_t* lat_in, int B, int C, int H, int W, int pad, int KH, int KW, int T,
                         int row_bytes, unsigned char* lists, int rec, int hdr, cudaStream_t s);

template <int FPL>
static int seq_go(const SeqPlan& pl, SeqArgs& s, cudaStream_t st) {
  auto kern = seq_train_kernel<FPL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_stdp_sequence: %s", cudaGetErrorString(e));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, pl.nwarps * 32, pl.smem);
  if (occ < 1) return set_error(SNN_ESHAPE, "snn_stdp_sequence: kernel does not fit an SM");
  void* args[] = {&s};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(pl.grid), dim3(pl.nwarps * 32), args,
                                  size_t(pl.smem), st);
  if (e != cudaSuccess) return set_error(SNN_ECUDA, "snn_stdp_sequence: %s", cudaGetErrorString(e));
  note_launch();
  return SNN_OK;
}

// Returns 1 if the persistent path does not apply (caller uses the per-call kernels), else an SNN code.
int seq_train_launch(const uint8_t* lat_all, int N, int C, int H, int W, int pad, float* w, int F, int KH, int KW,
                     int T, float theta, int k, int r, float a_plus, float a_minus, float lb, float ub,
                     int stabilizer, int32_t* winners, int32_t* count, float* snaps, int snap_every, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  SeqPlan pl;
  if (!(isfinite(theta)) || k > 256 || !seq_plan(C, H, W, pad, F, KH, KW, T, &pl)) return 1;
  const size_t need = seq_train_workspace(C, H, W, pad, F, KH, KW, T, k, N);
  if (ws_bytes < need) return set_error(SNN_EWORKSPACE, "snn_stdp_sequence: workspace %zu < %zu", ws_bytes, need);
  SeqArgs s;
  s.wa = pl.a;
  s.wa.lat_in = lat_all;
  s.wa.err = error_word_ptr(st);
  const double tt = floor(double(theta) * 2147483648.0);
  s.wa.thr = tt >= 9.0e18 ? INT64_MAX : (tt < -1.0 ? -1 : int64_t(tt));
  s.lat_all = lat_all; s.N = N; s.w = w; s.k = k; s.r = r;
  s.a_plus = a_plus; s.a_minus = a_minus; s.lb = lb; s.ub = ub; s.stabilizer = stabilizer;
  s.snaps = snaps; s.snap_every = snap_every > 0 ? snap_every : 1;
  if (!snaps) s.snap_every = 1;
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  s.bar = reinterpret_cast<unsigned*>(p);
  const size_t HoWo = size_t(pl.a.Ho) * pl.a.Wo;
  s.lat_map = p + 256;
  s.v_map = reinterpret_cast<float*>(p + 256 + r256(size_t(F) * HoWo));
  s.post = reinterpret_cast<int32_t*>(p + 256 + r256(size_t(F) * HoWo) + r256(size_t(F) * HoWo * 4));
  s.gbest = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s.post) + r256(size_t(N) * k * 4));
  s.stamps = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(s.gbest) + r256(size_t(pl.n_groups) * HoWo * 8));
  unsigned char* lists = reinterpret_cast<unsigned char*>(s.stamps) + r256(size_t(N) * 48 + 16384);
  s.lists = lists; s.rec = pl.rec; s.hdr = pl.hdr; s.npre = pl.npre; s.buf_bytes = pl.buf_bytes;
  s.wa.npre = pl.npre;
  // every image's receptive fields sorted up front (they do not depend on the weights)
  int rc = rf_sort_lists_launch(lat_all, N, C, H, W, pad, KH, KW, T, pl.a.row_bytes, lists, pl.rec, pl.hdr, st);
  if (rc) return rc;
  s.winners = winners; s.count = count;
  s.n_groups = pl.n_groups; s.FGS = pl.FGS; s.off_keys = pl.off_keys;
  s.dbg = getenv("SNN_SEQ_DBG") ? atoi(getenv("SNN_SEQ_DBG")) : 0;
  if (cudaMemsetAsync(s.bar, 0, 2 * sizeof(unsigned), st) != cudaSuccess) return check_launch("snn_stdp_sequence");
  switch (pl.fpl) {
    case 4: return seq_go<4>(pl, s, st);
    case 2: return seq_go<2>(pl, s, st);
    default: return seq_go<1>(pl, s, st);
  }
}

}  // namespace snn
