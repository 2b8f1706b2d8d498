// K5+K6 with SSIM for the common case (frames + float32 original, W % 4 == 0):
// a CTA covers one frame t of one cube, 128 columns (4 strips of 32) and two
// bands; warp w owns strip w % 4 of band w / 4, lane l one column.
//
// Compared with k_eval_ssim (one warp = one isolated 32-column strip) the four
// strips of a band share one shared-memory row buffer, so interior halos are
// read from the neighbouring warp instead of being converted twice; only the
// CTA's outer halos (none when the CTA spans the whole width, e.g. W = 128)
// are converted. The four warps of a band meet at a named barrier once per
// row. For 8/10-bit frames the float64 dequantisation is a shared-memory table
// lookup (exact: the table holds the same float64 values). Raw inputs stream
// through warp-private cp.async rings as before; rows are software pipelined
// (convert row y while row y-1 is filtered).
#pragma once
#include "ssim_kernel.cuh"

namespace cvb {

constexpr int kS4Strips = 4;
constexpr int kS4Chans = 2;
constexpr int kS4Row = kS4Strips * kSsimStrip + 2 * kSsimRadius;  // 138
constexpr int kS4LutMax = 1024;                                    // bit depth <= 10

// Row-buffer entry: (s, d) with the squares formed by the filter (halves the
// shared-memory bytes the 11-tap horizontal filter reads; the smem pipe is
// the co-bottleneck of this kernel), or (s, d, s^2, d^2) with CVB_SROW_F4.
#ifdef CVB_SROW_F4
using SRow = float4;
__device__ __forceinline__ SRow make_srow(float s, float d) { return make_float4(s, d, s * s, d * d); }
#else
using SRow = float2;
__device__ __forceinline__ SRow make_srow(float s, float d) { return make_float2(s, d); }
#endif

struct Ssim4Shared {
  SRow srow[kS4Chans][2][kS4Row];
  float raw_o[kS4Strips * kS4Chans][kStages][40];       // 32 main + 5 halo (+pad)
  uint32_t raw_f[kS4Strips * kS4Chans][kStages][24];    // 48 samples (u16 pairs / u8 quads)
  double lut[kS4Chans][kS4LutMax];
};

// barrier ids must be immediates, or ptxas reserves all 16 per CTA
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  if (id == 1) asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
  else asm volatile("bar.sync 2, %0;\n" ::"r"(nthreads) : "memory");
}

template <int RS, bool LUT>
__global__ void __launch_bounds__(256, 2)
k_eval_ssim4(const EvalArgs args) {
  using R = typename RawT<RS>::type;
  constexpr int HALO = kSsimRadius;
  constexpr int FPW = (RS == RS_FRAMES_U8) ? 4 : 2;  // samples per 32-bit word
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ssim4Shared &sh = *reinterpret_cast<Ssim4Shared *>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int j = w % kS4Strips, cl = w / kS4Strips;
  const int C = args.C;
  const int ncg = (C + kS4Chans - 1) / kS4Chans;
  const int grp = blockIdx.x / ncg;
  const int cgrp = blockIdx.x % ncg;
  const int c = cgrp * kS4Chans + cl;
  const int64_t T = args.T, H = args.H, W = args.W;
  const int64_t HW = H * W, inner = HW * C, rowlen = W * C;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int64_t x0c = (int64_t)grp * (kS4Strips * kSsimStrip);
  const int nvalid = (int)min((int64_t)kS4Strips, (W - x0c + kSsimStrip - 1) / kSsimStrip);
  const bool chan_ok = c < C;
  const double L = args.L, rL = args.rL;

  // band constants (warp-uniform); the dequantisation table of each band
  double my_m = 0.0, my_span = 0.0;
  if (chan_ok) {
    my_m = args.qmins[a * C + c];
    my_span = __dsub_rn(args.qmaxs[a * C + c], my_m);
  }
  if constexpr (LUT) {
    const int nch = min(kS4Chans, C - cgrp * kS4Chans);
    for (int i = threadIdx.x; i < kS4Chans * kS4LutMax; i += blockDim.x) {
      const int ch = i / kS4LutMax, q = i % kS4LutMax;
      if (ch < nch && q <= args.Li) {
        const double m = args.qmins[a * C + cgrp * kS4Chans + ch];
        const double sp = __dsub_rn(args.qmaxs[a * C + cgrp * kS4Chans + ch], m);
        sh.lut[ch][q] = dequantize_fast((uint32_t)q, m, sp, L, rL);
      }
    }
  }
  // out-of-image row entries stay zero for every row: write them once
  for (int i = threadIdx.x; i < kS4Chans * 2 * kS4Row; i += blockDim.x) {
    const int e = i % kS4Row;
    const int64_t x = x0c - HALO + e;
    if (x < 0 || x >= W) (&sh.srow[0][0][0])[i] = make_srow(0.f, 0.f);
  }
  __syncthreads();
  if (!chan_ok || j >= nvalid) return;  // absent strip / band: no barrier use below
  const int bar_id = 1 + cl, bar_n = 32 * nvalid;

  const double peak = args.peaks[a * C + c];
  const float c0 = (float)peak;
  const float C1 = fmaxf((float)((0.01 * peak) * (0.01 * peak)), 1e-30f);
  const float C2 = fmaxf((float)((0.03 * peak) * (0.03 * peak)), 1e-30f);

  // lane geometry
  const int64_t x0w = x0c + (int64_t)j * kSsimStrip;
  const int64_t xm = x0w + lane;
  const bool mimg = xm < W;
  const bool col_valid = xm >= HALO && xm < W - HALO;
  // outer halo duty: left halo by strip 0, right halo by the last strip (lanes 0..4)
  const bool hleft = (j == 0) && lane < HALO;
  const bool hright = (j == nvalid - 1) && lane < HALO;
  const int64_t xh = hleft ? x0c - HALO + lane : x0c + (int64_t)kSsimStrip * nvalid + lane;
  const bool himg = (hleft || hright) && xh >= 0 && xh < W;
  const int sidx_m = HALO + j * kSsimStrip + lane;
  const int sidx_h = (int)(xh - (x0c - HALO));

  const float *obase = reinterpret_cast<const float *>(args.orig) + (a * T + t) * inner + c;
  const R *fbase = reinterpret_cast<const R *>(args.frames) + (((a * args.G + c / 3) * T + t) * 3 + c % 3) * HW;
  const int64_t xf0 = x0w - 8;
  const int fwords = kRawF / FPW;
  const int64_t fx = xf0 + (int64_t)lane * FPW;
  const bool fok = lane < fwords && fx >= 0 && fx + FPW <= W;
  const char *ip_m = reinterpret_cast<const char *>(obase + (mimg ? xm : 0) * C);
  const char *ip_h = reinterpret_cast<const char *>(obase + (himg ? xh : 0) * C);
  const char *ip_f = reinterpret_cast<const char *>(fbase + (fok ? fx : 0));
  const int64_t ostride = rowlen * (int64_t)sizeof(float), fstride = W * (int64_t)sizeof(R);
  const uint32_t sa_m = smem_u32(&sh.raw_o[w][0][lane]);
  const uint32_t sa_h = smem_u32(&sh.raw_o[w][0][32 + lane]);
  const uint32_t sa_f = smem_u32(&sh.raw_f[w][0][lane]);
  constexpr uint32_t kPO = 40 * sizeof(float), kPF = 24 * sizeof(uint32_t);
  auto issue = [&](int y) {
    const uint32_t s = (uint32_t)y & (kStages - 1);
    if (mimg)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_m + s * kPO), "l"(ip_m) : "memory");
    if (himg)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_h + s * kPO), "l"(ip_h) : "memory");
    if (fok)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_f + s * kPF), "l"(ip_f) : "memory");
    ip_m += ostride;
    ip_h += ostride;
    ip_f += fstride;
  };
  const int fi_m = min(max((int)(xm - xf0), 0), kRawF - 1);
  const int fi_h = min(max((int)(xh - xf0), 0), kRawF - 1);
  auto frame_at = [&](int s, int i) -> uint32_t {
    const uint32_t word = sh.raw_f[w][s][i / FPW];
    if constexpr (FPW == 2) return (word >> (16 * (i & 1))) & 0xffffu;
    else return (word >> (8 * (i & 3))) & 0xffu;
  };
  uint32_t qmax = 0;
  auto recon = [&](uint32_t q) -> double {
    qmax = max(qmax, q);
    if constexpr (LUT) return sh.lut[cl][min(q, (uint32_t)(kS4LutMax - 1))];
    else return dequantize_fast(q, my_m, my_span, L, rL);
  };

  const bool wr = args.recon_out != nullptr && mimg;
  float *wq = (args.recon_out ? args.recon_out : reinterpret_cast<float *>(0)) + (a * T + t) * inner +
              (mimg ? xm : 0) * C + c;
  SRow(*srow)[kS4Row] = sh.srow[cl];
  double sse = 0.0, ssum_d = 0.0;
  float ssum = 0.f;
  Ring ring;
#pragma unroll
  for (int i = 0; i < 11; ++i) ring.s[i] = ring.d[i] = ring.ss[i] = ring.dd[i] = 0.f;

  const int H32 = (int)H;
#pragma unroll
  for (int r = 0; r < kStages - 1; ++r) {
    if (r < H32) issue(r);
    cp_async_commit();
  }

  auto filter_row = [&](int b, int y, auto ucst) {
    constexpr int U = decltype(ucst)::value;
    const SRow *sr = &srow[b][j * kSsimStrip + lane];
    float hs = 0.f, hd = 0.f, hss = 0.f, hdd = 0.f;
#pragma unroll
    for (int k = 0; k < kSsimTaps; ++k) {
      const SRow v = sr[k];
      const float wt = gtap(k < kSsimRadius ? kSsimRadius - k : k - kSsimRadius);
      hs = fmaf(wt, v.x, hs);
      hd = fmaf(wt, v.y, hd);
#ifdef CVB_SROW_F4
      hss = fmaf(wt, v.z, hss);
      hdd = fmaf(wt, v.w, hdd);
#else
      hss = fmaf(wt * v.x, v.x, hss);
      hdd = fmaf(wt * v.y, v.y, hdd);
#endif
    }
    float os, odv, oss, odd;
    ring_step<U>(ring, hs, hd, hss, hdd, os, odv, oss, odd);
    if (y >= 2 * kSsimRadius && col_valid) ssum += ssim_px(os, odv, oss, odd, c0, C1, C2);
  };

  auto do_row = [&](int y, auto ucst) {
    constexpr int U = decltype(ucst)::value;
    const int b = y & 1;
    if (y + kStages - 1 < H32) issue(y + kStages - 1);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncwarp();
    const int s = y & (kStages - 1);
    if (mimg) {
      const float om = sh.raw_o[w][s][lane];
      const double rm = recon(frame_at(s, fi_m));
      const double diff = __dsub_rn((double)om, rm);
      sse = __fma_rn(diff, diff, sse);
      if (wr) *wq = (float)rm;
      const float d = (float)diff;
      const float sv = fmaf(2.f, om - c0, -d);
      srow[b][sidx_m] = make_srow(sv, d);
    }
    wq += rowlen;
    if (himg) {
      const float oh = sh.raw_o[w][s][32 + lane];
      const double rh = recon(frame_at(s, fi_h));
      const float d = (float)__dsub_rn((double)oh, rh);
      const float sv = fmaf(2.f, oh - c0, -d);
      srow[b][sidx_h] = make_srow(sv, d);
    }
    if (y >= 1) filter_row(b ^ 1, y - 1, std::integral_constant<int, (U + 10) % 11>{});
    named_bar(bar_id, bar_n);  // row y complete for all strips of the band
  };

  for (int jb = 0; jb < H32; jb += 11) {
#define CV_ROW(U)                                                   \
  if (jb + U < H32) do_row(jb + U, std::integral_constant<int, U>{});
    CV_ROW(0) CV_ROW(1) CV_ROW(2) CV_ROW(3) CV_ROW(4) CV_ROW(5)
    CV_ROW(6) CV_ROW(7) CV_ROW(8) CV_ROW(9) CV_ROW(10)
#undef CV_ROW
    ssum_d += (double)ssum;
    ssum = 0.f;
  }
  {
    const int yl = H32 - 1;
    switch (yl % 11) {
#define CV_LAST(U) \
  case U: filter_row(yl & 1, yl, std::integral_constant<int, U>{}); break;
      CV_LAST(0) CV_LAST(1) CV_LAST(2) CV_LAST(3) CV_LAST(4) CV_LAST(5)
      CV_LAST(6) CV_LAST(7) CV_LAST(8) CV_LAST(9) CV_LAST(10)
#undef CV_LAST
    }
    ssum_d += (double)ssum;
  }
  cp_async_wait<0>();
  flag_warp(args.err, qmax > args.Li, CV_FLAG_INT_RANGE);

#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    ssum_d += __shfl_xor_sync(0xffffffffu, ssum_d, o);
  }
  if (lane == 0) {
    // partials layout [n][T][nstrips][2C]: strip index of this warp
    const int strip = (int)(x0w / kSsimStrip);
    double *p = args.part + (((a * T + t) * args.nstrips) + strip) * 2 * C;
    p[c] = sse;
    p[C + c] = ssum_d;
  }
}

}  // namespace cvb
