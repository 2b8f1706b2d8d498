// K5+K6 with SSIM, vertical-first variant (frames + float32 original,
// W % 4 == 0, no PCA) — the hot kernel of the benchmark.
//
// A CTA covers one frame t of one cube, two bands and 128 adjacent input
// columns x0..x0+127 (x0 = 118*g): warp w owns band w/4 and columns
// 32*(w%4)..+31, lane l one column. The CTA scores the 118 output columns
// x0+5..x0+122 (valid region: an output needs its whole 11x11 window inside
// the frame, so no out-of-image data is ever read; neighbouring CTAs overlap
// by 10 input columns; W = 128 is one CTA).
//
// Per input row y every thread
//   1. converts its own element (warp-private 8-stage cp.async ring, no
//      barrier): float64 dequantisation (shared-memory table for <= 10 bits),
//      SSE, recon write, and the two SSIM inputs s = x'+y', d = x-y;
//   2. runs the VERTICAL 11-tap filter of s, d, s^2, d^2 for its own column
//      as a transposed-form FIR (ten float4 partial sums in registers, updated
//      in place: 11 FFMA per map and row, no rotation), completing
//      column-filtered row e = y-10 (output row y-5), which the warp stores
//      (float4) into slot e % 8 of a shared row ring and announces on the
//      slot's `full` mbarrier (the slot's previous row must have been
//      filtered: `empty` mbarrier);
//   3. one warp per row (warp e % 4 of the band, one input row later) runs
//      the HORIZONTAL 11-tap filter of row e: lane q computes output columns
//      4q+5 .. 4q+8 from the 14 entries 4q .. 4q+13 (14 LDS.128 + 176 FFMA
//      for 4 outputs), then the SSIM of each output.
// Producers never wait on consumers except through the 8-deep ring, so the
// warps of a band drift freely (no barrier stalls); the horizontal work is
// spread evenly (each warp filters every fourth row). All Gaussian weights are
// compile-time immediates.
#pragma once
#include "ssim4_kernel.cuh"

namespace cvb {

#ifndef CVB_SSIM6_MINB
#define CVB_SSIM6_MINB 2
#endif

constexpr int k6Cols = 128;  // input columns per CTA (4 warps x 32 lanes)
constexpr int k6Out = k6Cols - 2 * kSsimRadius;  // 118 output columns per CTA
constexpr int k6Tasks = k6Out / 2;               // 59 two-column tasks per row
constexpr int k6Chans = 2;
constexpr int k6LutMax = 1024;  // bit depth <= 10
constexpr int k6Stages = 8;     // input ring (rows), power of two
constexpr int k6Depth = 6;      // input rows in flight per warp (< k6Stages)
constexpr int k6Ring = 8;       // mbarrier-pipelined row ring

// PCA: the frames hold E <= k6PcaMax principal-component planes (12/16-bit);
// every band's recon is mean_c + sum_j pc_j W[j][c] (transform.py:202-210).
constexpr int k6PcaMax = 12;

template <bool PCA>
struct Ssim6SharedT {
  // column-filtered rows: [band][row slot e % 8][column % 4][column / 4]; a
  // sub-array pitch of 34 (= 2 mod 8) float4 makes both the producer stores
  // (lane = column) and the consumer loads (lane q reads column 4q+k) hit 32
  // distinct banks per quarter warp
  float4 vb[k6Chans][k6Ring][4][34];
  unsigned long long full[k6Chans][k6Ring];   // 4 warp arrivals: row stored
  unsigned long long empty[k6Chans][k6Ring];  // 1 arrival: row filtered
  float raw_o[2 * 4][k6Stages][32];
  // frame words of the warp's 32 columns: u16 -> 16 words per plane; u8 -> <= 9
  // (rows may start 2 samples into a word); PCA: E planes of 16 words
  uint32_t raw_f[2 * 4][k6Stages][PCA ? 16 * k6PcaMax : 16];
  double lut[k6Chans][PCA ? 1 : k6LutMax];
  // PCA: recon_c = base_c + sum_j q_j coef[c][j] with coef = (span_j / L) W[j][c]
  // and base_c = mean_c + sum_j min_j W[j][c] (the dequantisation folded into
  // the inverse projection; float64 throughout)
  double coef[PCA ? k6Chans : 1][PCA ? k6PcaMax : 1];
  int64_t poff[PCA ? k6PcaMax : 1];  // PCA: element offset of plane j from plane 0
  double base[k6Chans];
};
using Ssim6Shared = Ssim6SharedT<false>;

// Transposed-form 11-tap FIR along the rows of one column: z[k] holds the
// partial sum of the output row completed k rows from now. One step consumes
// input row y and returns the column-filtered value of row y-5.
struct Fir4 {
  float4 z[10];
};

__device__ __forceinline__ float4 fir4_step(Fir4 &f, float s, float d) {
  const float ss = s * s, dd = d * d;
  float4 out;
  {
    const float wt = gtap(5);  // tap 0 of the window (row y-10 .. y: weight g[|k-5|])
    out = make_float4(fmaf(wt, s, f.z[0].x), fmaf(wt, d, f.z[0].y), fmaf(wt, ss, f.z[0].z),
                      fmaf(wt, dd, f.z[0].w));
  }
#pragma unroll
  for (int k = 1; k < 10; ++k) {
    const float wt = gtap(k - 5 < 0 ? 5 - k : k - 5);
    float4 &v = f.z[k - 1];
    const float4 n = f.z[k];
    v = make_float4(fmaf(wt, s, n.x), fmaf(wt, d, n.y), fmaf(wt, ss, n.z), fmaf(wt, dd, n.w));
  }
  {
    const float wt = gtap(5);
    f.z[9] = make_float4(wt * s, wt * d, wt * ss, wt * dd);
  }
  return out;
}

__device__ __forceinline__ void mbar_init(unsigned long long *b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__host__ __device__ inline int ssim6_groups(int64_t W) { return (int)((W - 2 * kSsimRadius + k6Out - 1) / k6Out); }

// EP: 0 without PCA, else the component-plane count the loops are unrolled
// for (E itself for the common 6 and 9, k6PcaMax with runtime guards otherwise)
template <int RS, bool LUT, int EP>
__global__ void __launch_bounds__(256, CVB_SSIM6_MINB)
k_eval_ssim6(const EvalArgs args, const PcaParams inv) {
  constexpr bool PCA = EP > 0;
  using R = typename RawT<RS>::type;
  constexpr int FPW = (RS == RS_FRAMES_U8) ? 4 : 2;  // frame samples per 32-bit word
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ssim6SharedT<PCA> &sh = *reinterpret_cast<Ssim6SharedT<PCA> *>(smem_raw);
  static_assert(!PCA || (RS == RS_FRAMES_U16 && !LUT), "PCA path: u16 component planes");
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int j = w & 3, cl = w >> 2;
  const int C = args.C;
  const int ncg = (C + k6Chans - 1) / k6Chans;
  const int grp = blockIdx.x / ncg;
  const int cgrp = blockIdx.x % ncg;
  const int c = cgrp * k6Chans + cl;
  const int64_t T = args.T, H = args.H, W = args.W;
  const int64_t HW = H * W, inner = HW * C, rowlen = W * C;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int64_t x0 = (int64_t)grp * k6Out;
  const bool last_grp = grp == (int)gridDim.x / ncg - 1;
  const double L = args.L, rL = args.rL;

  const int E = args.E;
  if constexpr (PCA) {
    if (threadIdx.x < E) {
      const int jp = threadIdx.x;
      sh.poff[jp] = ((int64_t)(jp / 3) * 3 * args.T + jp % 3) * args.H * args.W;
    }
    const int cc = cgrp * k6Chans + (int)threadIdx.x / k6PcaMax, jj = (int)threadIdx.x % k6PcaMax;
    if (threadIdx.x < k6Chans * k6PcaMax && cc < C && jj < E) {
      const double m = args.qmins[a * E + jj];
      const double sp = __dsub_rn(args.qmaxs[a * E + jj], m);
      sh.coef[threadIdx.x / k6PcaMax][jj] = (sp / L) * inv.W[jj * kMaxC + cc];
    }
    if (threadIdx.x < k6Chans && cgrp * k6Chans + (int)threadIdx.x < C) {
      const int cb = cgrp * k6Chans + threadIdx.x;
      double b = inv.mean[cb];
      for (int j2 = 0; j2 < E; ++j2) b = __fma_rn(args.qmins[a * E + j2], inv.W[j2 * kMaxC + cb], b);
      sh.base[threadIdx.x] = b;
    }
  }
  double my_m = 0.0, my_span = 0.0;
  if (!PCA && c < C) {
    my_m = args.qmins[a * C + c];
    my_span = __dsub_rn(args.qmaxs[a * C + c], my_m);
  }
  if constexpr (LUT) {
    const int nch = min(k6Chans, C - cgrp * k6Chans);
    for (int i = threadIdx.x; i < k6Chans * k6LutMax; i += blockDim.x) {
      const int ch = i / k6LutMax, q = i % k6LutMax;
      if (ch < nch && q <= (int)args.Li) {
        const double m = args.qmins[a * C + cgrp * k6Chans + ch];
        const double sp = __dsub_rn(args.qmaxs[a * C + cgrp * k6Chans + ch], m);
        sh.lut[ch][q] = dequantize_fast((uint32_t)q, m, sp, L, rL);
      }
    }
  }
  if (threadIdx.x < k6Chans * k6Ring) {
    mbar_init(&sh.full[0][0] + threadIdx.x, 4);
    mbar_init(&sh.empty[0][0] + threadIdx.x, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  // every ring slot starts out free: complete phase 0 of its `empty` barrier
  if (threadIdx.x < k6Chans * k6Ring) mbar_arrive(&sh.empty[0][0] + threadIdx.x);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (c >= C) return;  // absent band: its four warps leave together

  const double peak = args.peaks[a * C + c];
  const float c0 = (float)peak;
  const float C1 = fmaxf((float)((0.01 * peak) * (0.01 * peak)), 1e-30f);
  const float C2 = fmaxf((float)((0.03 * peak) * (0.03 * peak)), 1e-30f);

  // ---- this thread's input column (32-bit: W < 2^31, checked by the host)
  const int lc = 32 * j + lane;  // local column 0..127
  const int W32 = (int)W;
  const int xv = (int)x0 + lc;
  const bool vimg = xv < W32;
  // every element is counted (SSE, recon write) by exactly one CTA
  const bool own = vimg && (lc < k6Out || last_grp);
  const int xc = vimg ? xv : W32 - 1;  // clamped column: loads stay in bounds

  const float *obase = reinterpret_cast<const float *>(args.orig) + (a * T + t) * inner + c;
  // non-PCA: the band's own plane; PCA: component plane 0 (+ poff[j] per copy)
  const int fpl = PCA ? 0 : c;
  const int Eg = (EP == k6PcaMax) ? E : EP;  // compile-time for the exact-E instances
  const R *fbase = reinterpret_cast<const R *>(args.frames) + (((a * args.G + fpl / 3) * T + t) * 3 + fpl % 3) * HW;
  // frame words: the warp's 32 samples start `foff` samples into the 4-byte word at xa
  const int xw = (int)x0 + 32 * j;
  const int xa = xw & ~(FPW - 1);
  const int foff = xw - xa;
  const int fx = xa + (PCA ? (lane & 15) : lane) * FPW;
  // words past the row end copy the row's last word instead (valid samples for
  // lanes outside the frame, whose results are never counted)
  const bool fok = PCA ? true : lane < (foff + 32 + FPW - 1) / FPW;
  const int fxc = min(fx, W32 - FPW);  // W % 4 == 0: words never straddle the row end
  // PCA: copy k of a row moves plane 2k + (lane >> 4), word lane & 15
  const char *ip_o = reinterpret_cast<const char *>(obase + (int64_t)xc * C);
  const char *ip_f = reinterpret_cast<const char *>(fbase + (fok ? fxc : 0));
  const int64_t ostride = rowlen * (int64_t)sizeof(float), fstride = W * (int64_t)sizeof(R);
  const uint32_t sa_o = smem_u32(&sh.raw_o[w][0][lane]);
  const uint32_t sa_f = smem_u32(&sh.raw_f[w][0][PCA ? 16 * (lane >> 4) + (lane & 15) : lane]);
  constexpr uint32_t kPO = 32 * sizeof(float), kPF = (PCA ? 16 * k6PcaMax : 16) * sizeof(uint32_t);
  auto copy_frames = [&](uint32_t soff) {
    if constexpr (PCA) {
#pragma unroll
      for (int k = 0; k < (EP + 1) / 2; ++k) {
        const int jj = 2 * k + (lane >> 4);
        if (jj < Eg)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_f + soff + k * 32 * 4),
                       "l"(ip_f + sh.poff[jj] * (int64_t)sizeof(R))
                       : "memory");
      }
    } else {
      if (fok) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_f + soff), "l"(ip_f) : "memory");
    }
  };
  const int H32 = (int)H;
  // copy row yi into stage yi % k6Stages (rows past the frame: empty group)
  auto issue_s = [&](auto scst) {  // steady state: the row exists, stage S static
    constexpr uint32_t S = decltype(scst)::value;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_o + S * kPO), "l"(ip_o) : "memory");
    copy_frames(S * kPF);
    ip_o += ostride;
    ip_f += fstride;
    cp_async_commit();
  };
  auto issue = [&](int yi) {
    if (yi < H32) {
      const uint32_t s = (uint32_t)yi & (k6Stages - 1);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_o + s * kPO), "l"(ip_o) : "memory");
      copy_frames(s * kPF);
    }
    ip_o += ostride;
    ip_f += fstride;
    cp_async_commit();
  };
  const int fi = foff + lane;
  const int fw = fi / FPW, fsh = (fi % FPW) * (32 / FPW);
  uint32_t qmax = 0;

  float *wq = args.recon_out ? args.recon_out + (a * T + t) * inner + (int64_t)xc * C + c : nullptr;
  const bool wr = wq != nullptr && own;

  double sse = 0.0, ssum_d = 0.0;
  float ssum = 0.f;

  // convert row y (stage y % k6Stages) into (s, d); SSE + recon write
  auto convert = [&](int st, float &sv, float &dv) {
    const float om = sh.raw_o[w][st][lane];
    double rm;
    uint32_t q;
    if constexpr (PCA) {
      // recon = mean_c + sum_j pc_j W[j][c] with pc_j = min_j + q_j span_j / L,
      // reassociated (base + sum q_j coef_j): agrees with the reference's
      // float64 evaluation to ~1e-16 relative
      double acc = sh.base[cl];
      q = 0;
#pragma unroll
      for (int jj = 0; jj < EP; ++jj) {
        if (jj < Eg) {
          const uint32_t qj = (sh.raw_f[w][st][16 * jj + fw] >> fsh) & 0xffffu;
          q = max(q, qj);
          acc = __fma_rn((double)qj, sh.coef[cl][jj], acc);
        }
      }
      rm = acc;
    } else {
      q = (sh.raw_f[w][st][fw] >> fsh) & ((1u << (32 / FPW)) - 1u);
      if constexpr (LUT) rm = sh.lut[cl][min(q, (uint32_t)(k6LutMax - 1))];
      else rm = dequantize_fast(q, my_m, my_span, L, rL);
    }
    // lanes outside the frame (or owned by the next CTA) compute on valid
    // neighbour samples: their maps only reach masked outputs and their SSE
    // is dropped at the end
    const double diff = __dsub_rn((double)om, rm);
    const float df = (float)diff;
    qmax = max(qmax, q);
    sv = fmaf(2.f, om - c0, -df);
    dv = df;
    sse = __fma_rn(diff, diff, sse);
    if (wr) *wq = (float)rm;
    wq += rowlen;
  };

  Fir4 fir;
#pragma unroll
  for (int i = 0; i < 10; ++i) fir.z[i] = make_float4(0.f, 0.f, 0.f, 0.f);

  // prologue: rows 0 .. k6Depth-1 in flight, row 0 converted
#pragma unroll
  for (int r = 0; r < k6Depth; ++r) issue(r);
  float sv_n, dv_n;
  cp_async_wait<k6Depth - 1>();
  __syncwarp();
  convert(0, sv_n, dv_n);  // stage 0

  // mbarrier pipeline: every warp stores column-filtered row e into ring slot
  // e % 8 (after the slot's previous row was filtered: empty barrier) and
  // arrives on full; warp e % 4 of the band filters row e one input row later
  // (lane q: output columns 4q+5 .. 4q+8 from columns 4q .. 4q+13, 14 LDS.128
  // + 44 FFMA per output) and arrives on empty.
  float4 *vbw = &sh.vb[cl][0][lc & 3][lc >> 2];
  constexpr int kVbRow = 4 * 34;
  const int hq = lane;
  bool hvalid[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) hvalid[i] = 4 * hq + i < k6Out && xv - lc + 4 * hq + i + 5 < W32 - kSsimRadius;
  auto consume = [&](int e) {
    const int slot = e & (k6Ring - 1);
    mbar_wait(&sh.full[cl][slot], (uint32_t)(e >> 3) & 1u);
    __syncwarp();
    const float4 *hv = &sh.vb[cl][slot][0][hq];
    float4 acc[4];
#pragma unroll
    for (int k = 0; k < 14; ++k) {
      const float4 v = hv[(k & 3) * 34 + (k >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int tp = k - i;  // tap of output i
        if (tp < 0 || tp > 10) continue;
        const float wt = gtap(tp < 5 ? 5 - tp : tp - 5);
        if (tp == 0) acc[i] = make_float4(wt * v.x, wt * v.y, wt * v.z, wt * v.w);
        else acc[i] = make_float4(fmaf(wt, v.x, acc[i].x), fmaf(wt, v.y, acc[i].y),
                                  fmaf(wt, v.z, acc[i].z), fmaf(wt, v.w, acc[i].w));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[cl][slot]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float s0 = ssim_px(acc[i].x, acc[i].y, acc[i].z, acc[i].w, c0, C1, C2);
      ssum += hvalid[i] ? s0 : 0.f;
    }
  };
  // input row y (generic: runtime bounds and indices): issue row y + k6Depth,
  // convert row y + 1, FIR step of row y; from row 10 on store column-filtered
  // row e = y - 10 and filter row e-1 (warp (e-1) % 4)
  auto do_row = [&](int y) {
    const float sv = sv_n, dv = dv_n;
    issue(y + k6Depth);
    if (y + 1 < H32) {
      cp_async_wait<k6Depth - 1>();
      __syncwarp();
      convert((y + 1) & (k6Stages - 1), sv_n, dv_n);
    }
    const float4 o = fir4_step(fir, sv, dv);
    if (y >= 2 * kSsimRadius) {
      const int e = y - 2 * kSsimRadius;
      const int slot = e & (k6Ring - 1);
      mbar_wait(&sh.empty[cl][slot], (uint32_t)(e >> 3) & 1u);
      vbw[slot * kVbRow] = o;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.full[cl][slot]);
      if (e >= 1 && j == ((e - 1) & 3)) consume(e - 1);
    }
  };
  // steady state (P = y % 8 static; rows y+1 and y+k6Depth exist, y >= 16):
  // stage, ring slot and consumer warp are compile-time, no bounds checks
  auto do_row_s = [&](int y, auto pcst) {
    constexpr int P = decltype(pcst)::value;
    constexpr int SL = (P + 8 - 2 * kSsimRadius % 8) % 8;  // ring slot of e = y - 10
    const float sv = sv_n, dv = dv_n;
    issue_s(std::integral_constant<uint32_t, (P + k6Depth) % k6Stages>{});
    cp_async_wait<k6Depth - 1>();
    __syncwarp();
    convert((P + 1) % k6Stages, sv_n, dv_n);
    const float4 o = fir4_step(fir, sv, dv);
    const int e = y - 2 * kSsimRadius;
    mbar_wait(&sh.empty[cl][SL], (uint32_t)(e >> 3) & 1u);
    vbw[SL * kVbRow] = o;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.full[cl][SL]);
  };
  // in a steady half-block of rows y..y+3 warp j filters the one row the
  // per-row schedule gives it (position (j+3)%4: row y + (j+3)%4 - 11), once,
  // after the four rows: the filter body exists twice in the loop, not 8x
  const int pj = (j + 3) & 3;

  static_assert(k6Stages == 8 && k6Ring == 8, "steady-state loop is unrolled by 8");
  for (int y = 0; y < H32; y += 8) {
    if (y >= 16 && y + 7 + k6Depth < H32) {
      do_row_s(y, std::integral_constant<int, 0>{});
      do_row_s(y + 1, std::integral_constant<int, 1>{});
      do_row_s(y + 2, std::integral_constant<int, 2>{});
      do_row_s(y + 3, std::integral_constant<int, 3>{});
      consume(y + pj - 2 * kSsimRadius - 1);
      do_row_s(y + 4, std::integral_constant<int, 4>{});
      do_row_s(y + 5, std::integral_constant<int, 5>{});
      do_row_s(y + 6, std::integral_constant<int, 6>{});
      do_row_s(y + 7, std::integral_constant<int, 7>{});
      consume(y + 4 + pj - 2 * kSsimRadius - 1);
    } else {
      for (int k = 0; k < 8 && y + k < H32; ++k) do_row(y + k);
    }
    ssum_d += (double)ssum;
    ssum = 0.f;
  }
  {  // the last column-filtered row (H-11) is filtered after the loop
    const int e = H32 - 1 - 2 * kSsimRadius;
    if (j == (e & 3)) consume(e);
    ssum_d += (double)ssum;
  }
  if (!own) sse = 0.0;
  flag_warp(args.err, qmax > args.Li, CV_FLAG_INT_RANGE);

#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    ssum_d += __shfl_xor_sync(0xffffffffu, ssum_d, o);
  }
  if (lane == 0) {
    // partials layout [n][T][nstrips][2C], nstrips = 4 * groups: one slot per warp
    double *p = args.part + (((a * T + t) * args.nstrips) + grp * 4 + j) * 2 * C;
    p[c] = sse;
    p[C + c] = ssum_d;
  }
}

}  // namespace cvb
