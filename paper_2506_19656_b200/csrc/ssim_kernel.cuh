// K5+K6 with SSIM, warp-per-channel variant (the hot kernel of the benchmark).
//
// A CTA covers one frame t of one cube and a strip of 32 output columns
// x0..x0+31 for up to 8 bands; warp w owns band c = cg*8 + w and lane l owns
// column x0+l. The warp walks the H rows of its strip alone:
//  * its raw inputs (original float + decoded frame samples of the strip row
//    and the 5-pixel halos) stream through a warp-private 4-stage cp.async
//    (LDGSTS) ring in shared memory, 3 rows ahead of the row being scored;
//  * every row it converts its 32 elements plus the 10 halo elements (lanes
//    0..9) into the four SSIM maps in its own float4 row buffer, __syncwarp,
//    runs the 11-tap horizontal Gaussian (shared loads at immediate offsets)
//    and scatters the result into an 11-slot register ring that accumulates
//    the vertical filter.
// No CTA-wide barrier sits in the row loop, so the warps of a CTA drift freely
// and hide each other's latencies; band constants are warp-uniform.
#pragma once
#include "eval_kernel.cuh"

namespace cvb {

constexpr int kSsimWarpsPerCta = 8;
constexpr int kSsimStrip = 32;
constexpr int kSsimRow = kSsimStrip + 2 * kSsimRadius;  // 42 row entries per warp
constexpr int kStages = 4;                              // cp.async ring depth (rows)
constexpr int kRawO = 44;                               // original floats per stage row
constexpr int kRawF = 48;                               // frame samples per stage row

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct SsimShared {
  float4 srow[kSsimWarpsPerCta][2][kSsimRow];
  float raw_o[kSsimWarpsPerCta][kStages][kRawO];
  uint32_t raw_f[kSsimWarpsPerCta][kStages][kRawF / 2];  // u16 pairs / u8 quads
};

// ASYNC: f32 original + non-PCA u8/u16 frames with W a multiple of 4 (frame
// rows then start 4-byte aligned): raw rows stream through the cp.async ring.
// Otherwise: one-row register prefetch (PCA, f64/u16 originals, recon_in).
#ifndef CVB_SSIM_MINB
#define CVB_SSIM_MINB 2
#endif

template <typename TO, int RS, bool PCA, bool ASYNC>
__global__ void __launch_bounds__(256, CVB_SSIM_MINB)
k_eval_ssim(const EvalArgs args, const PcaParams inv) {
  using R = typename RawT<RS>::type;
  constexpr bool FRAMES = (RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16);
  constexpr int HALO = kSsimRadius;
  __shared__ __align__(16) SsimShared sh;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int C = args.C, E = args.E;
  const int ncg = (C + kSsimWarpsPerCta - 1) / kSsimWarpsPerCta;
  const int strip = blockIdx.x / ncg;
  const int c = (blockIdx.x % ncg) * kSsimWarpsPerCta + w;
  if (c >= C) return;  // whole warp; no CTA barrier follows
  const int64_t T = args.T, H = args.H, W = args.W;
  const int64_t HW = H * W, inner = HW * C, rowlen = W * C;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int64_t x0 = (int64_t)strip * kSsimStrip;
  float4(*srow)[kSsimRow] = sh.srow[w];

  double my_m = 0.0, my_span = 0.0;
  if constexpr (FRAMES && !PCA) {
    my_m = args.qmins[a * E + c];
    my_span = __dsub_rn(args.qmaxs[a * E + c], my_m);
  }
  const double peak = args.peaks[a * C + c];
  const float c0 = (float)peak;
  const float C1 = fmaxf((float)((0.01 * peak) * (0.01 * peak)), 1e-30f);
  const float C2 = fmaxf((float)((0.03 * peak) * (0.03 * peak)), 1e-30f);

  // lane geometry: main column x0+lane, halo column (lanes 0..9)
  const int64_t xm = x0 + lane;
  const bool mimg = xm < W;
  const bool col_valid = xm >= HALO && xm < W - HALO;
  const bool hact = lane < 2 * HALO;
  const int pin_h = lane < HALO ? lane : kSsimStrip + lane;
  const int64_t xh = x0 - HALO + pin_h;
  const bool himg = hact && xh >= 0 && xh < W;
  const float mmask = mimg ? 1.f : 0.f, hmask = himg ? 1.f : 0.f;
  const int64_t xmc = mimg ? xm : 0, xhc = himg ? xh : 0;

  const TO *obase = reinterpret_cast<const TO *>(args.orig) + (a * T + t) * inner + c;
  const R *fbase = nullptr;
  if constexpr (FRAMES && !PCA)
    fbase = reinterpret_cast<const R *>(args.frames) + (((a * args.G + c / 3) * T + t) * 3 + c % 3) * HW;
  const R *pcbase = nullptr;
  if constexpr (PCA) pcbase = reinterpret_cast<const R *>(args.frames) + (a * args.G * T + t) * 3 * HW;

  // ---- raw input streams
  // ASYNC ring: raw_o[s][5+l] = original of main lane l, raw_o[s][pin_h] = halo;
  // raw_f[s] = frame samples of pixels [xf0, xf0 + 48), xf0 = x0 - 8 (16-B aligned words).
  constexpr int FPW = (RS == RS_FRAMES_U8) ? 4 : 2;  // samples per 32-bit word
  const int64_t xf0 = x0 - 8;
  const int fwords = kRawF / FPW;                     // words per stage row
  const bool fcopy = lane < fwords;
  const int64_t fx = xf0 + (int64_t)lane * FPW;       // first pixel of this lane's word
  const bool fok = fcopy && fx >= 0 && fx + FPW <= W;
  // running source pointers of the next row to copy (rows are issued in order)
  const char *ip_m = reinterpret_cast<const char *>(obase + xmc * C);
  const char *ip_h = reinterpret_cast<const char *>(obase + xhc * C);
  const char *ip_f = fbase ? reinterpret_cast<const char *>(fbase + (fok ? fx : 0)) : nullptr;
  const int64_t ostride = rowlen * (int64_t)sizeof(TO), fstride = W * (int64_t)sizeof(R);
  // shared-memory byte addresses of this lane's slots in stage 0 (stage pitch below)
  const uint32_t sa_m = smem_u32(&sh.raw_o[w][0][HALO + lane]);
  const uint32_t sa_h = smem_u32(&sh.raw_o[w][0][pin_h]);
  const uint32_t sa_f = smem_u32(&sh.raw_f[w][0][lane]);
  constexpr uint32_t kPitchO = kRawO * sizeof(float), kPitchF = (kRawF / 2) * sizeof(uint32_t);
  auto issue = [&](int y) {
    if constexpr (ASYNC) {
      const uint32_t s = (uint32_t)y & (kStages - 1);
      if (mimg)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_m + s * kPitchO), "l"(ip_m) : "memory");
      if (himg)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_h + s * kPitchO), "l"(ip_h) : "memory");
      if (fok)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa_f + s * kPitchF), "l"(ip_f) : "memory");
      ip_m += ostride;
      ip_h += ostride;
      ip_f += fstride;
    }
  };
  // frame sample of pixel x in stage s; masked lanes read any valid slot
  const int fi_m = min(max((int)(xm - xf0), 0), kRawF - 1);
  const int fi_h = min(max((int)(xh - xf0), 0), kRawF - 1);
  auto frame_at = [&](int s, int i) -> uint32_t {
    const uint32_t word = sh.raw_f[w][s][i / FPW];
    if constexpr (FPW == 2) return (word >> (16 * (i & 1))) & 0xffffu;
    else return (word >> (8 * (i & 3))) & 0xffu;
  };

  // register prefetch (non-ASYNC)
  const TO *op_m = obase + xmc * C, *op_h = obase + xhc * C;
  const R *rp_m = nullptr, *rp_h = nullptr;
  int64_t rrow = rowlen;
  if constexpr (FRAMES && !PCA) {
    rp_m = fbase + xmc;
    rp_h = fbase + xhc;
    rrow = W;
  } else if constexpr (!FRAMES) {
    const R *rb = reinterpret_cast<const R *>(args.recon_in) + (a * T + t) * inner + c;
    rp_m = rb + xmc * C;
    rp_h = rb + xhc * C;
  }
  TO o_m = TO(0), o_h = TO(0), o_mn = TO(0), o_hn = TO(0);
  R r_m = R(0), r_h = R(0), r_mn = R(0), r_hn = R(0);
  auto load_next = [&]() {
    o_mn = ldg(op_m);
    op_m += rowlen;
    if constexpr (!PCA) {
      r_mn = ldg(rp_m);
      rp_m += rrow;
    }
    if (hact) {
      o_hn = ldg(op_h);
      op_h += rowlen;
      if constexpr (!PCA) {
        r_hn = ldg(rp_h);
        rp_h += rrow;
      }
    }
  };

  uint32_t qmax = 0;
  auto recon_pca = [&](int64_t y, int64_t x) -> double {
    double acc = 0.0;
    for (int j = 0; j < E; ++j) {
      const uint32_t q = (uint32_t)ldg(pcbase + ((int64_t)(j / 3) * T * 3 + (j % 3)) * HW + y * W + x);
      qmax = max(qmax, q);
      const double m = args.qmins[a * E + j];
      const double pc = dequantize_fast(q, m, __dsub_rn(args.qmaxs[a * E + j], m), args.L, args.rL);
      acc = __fma_rn(pc, inv.W[j * kMaxC + c], acc);
    }
    return __dadd_rn(acc, inv.mean[c]);
  };
  auto recon_raw = [&](uint32_t q, bool ok) -> double {
    if (ok) qmax = max(qmax, q);
    return dequantize_fast(q, my_m, my_span, args.L, args.rL);
  };

  double sse = 0.0, ssum_d = 0.0;
  float ssum = 0.f;
  Ring ring;
#pragma unroll
  for (int i = 0; i < 11; ++i) ring.s[i] = ring.d[i] = ring.ss[i] = ring.dd[i] = 0.f;

  if constexpr (ASYNC) {
#pragma unroll
    for (int r = 0; r < kStages - 1; ++r) {
      if (r < (int)H) issue(r);
      cp_async_commit();
    }
  } else {
    load_next();
    o_m = o_mn;
    o_h = o_hn;
    r_m = r_mn;
    r_h = r_hn;
  }

  const int H32 = (int)H;
  const bool wr = args.recon_out != nullptr && mimg;
  float *wq = (args.recon_out ? args.recon_out : reinterpret_cast<float *>(0)) + (a * T + t) * inner + xmc * C + c;

  // horizontal 11-tap filter of a converted row + vertical ring step + SSIM of row y-5
  auto filter_row = [&](int b, int y, auto ucst) {
    constexpr int U = decltype(ucst)::value;
    float hs = 0.f, hd = 0.f, hss = 0.f, hdd = 0.f;
#pragma unroll
    for (int k = 0; k < kSsimTaps; ++k) {
      const float4 v = srow[b][lane + k];
      const float wt = gtap(k < kSsimRadius ? kSsimRadius - k : k - kSsimRadius);
      hs = fmaf(wt, v.x, hs);
      hd = fmaf(wt, v.y, hd);
      hss = fmaf(wt, v.z, hss);
      hdd = fmaf(wt, v.w, hdd);
    }
    float os, odv, oss, odd;
    ring_step<U>(ring, hs, hd, hss, hdd, os, odv, oss, odd);
    if (y >= 2 * kSsimRadius && col_valid) ssum += ssim_px(os, odv, oss, odd, c0, C1, C2);
  };

  auto do_row = [&](int y, auto ucst) {
    constexpr int U = decltype(ucst)::value;
    const int B = y & 1;  // row buffer: row y converts into B while row y-1 is filtered from B^1
    float om, oh = 0.f;
    double rm, rh = 0.0;
    if constexpr (ASYNC) {
      if (y + kStages - 1 < H32) issue(y + kStages - 1);
      cp_async_commit();
      cp_async_wait<kStages - 1>();
      __syncwarp();
      const int s = y & (kStages - 1);
      const float vm = sh.raw_o[w][s][HALO + lane];
      om = mimg ? vm : 0.f;  // never-copied slots may hold NaN bits
      rm = recon_raw(frame_at(s, fi_m), mimg);
      if (hact) {
        const float vh = sh.raw_o[w][s][pin_h];
        oh = himg ? vh : 0.f;
        rh = recon_raw(frame_at(s, fi_h), himg);
      }
    } else {
      if (y + 1 < H32) load_next();
      om = (float)o_m;
      if constexpr (PCA) rm = recon_pca(y, xmc);
      else if constexpr (FRAMES) rm = recon_raw((uint32_t)r_m, true);
      else rm = (double)r_m;
      if (hact) {
        oh = (float)o_h;
        if constexpr (PCA) rh = recon_pca(y, xhc);
        else if constexpr (FRAMES) rh = recon_raw((uint32_t)r_h, true);
        else rh = (double)r_h;
      }
    }
    {
      const double od = (sizeof(TO) == 8 && !ASYNC) ? (double)o_m : (double)om;
      const double diff = __dsub_rn(od, rm);
      if (mimg) sse = __fma_rn(diff, diff, sse);
      if (wr) *wq = (float)rm;
      wq += rowlen;
      const float d = mimg ? (float)diff : 0.f;
      const float sv = mimg ? fmaf(2.f, om - c0, -d) : 0.f;
      srow[B][lane + HALO] = make_float4(sv, d, sv * sv, d * d);
    }
    if (hact) {
      const double od = (sizeof(TO) == 8 && !ASYNC) ? (double)o_h : (double)oh;
      const float d = himg ? (float)__dsub_rn(od, rh) : 0.f;
      const float sv = himg ? fmaf(2.f, oh - c0, -d) : 0.f;
      srow[B][pin_h] = make_float4(sv, d, sv * sv, d * d);
    }
    // software pipeline: filter row y-1 (converted last iteration) while the
    // conversion of row y above is still in flight
    if (y >= 1) {
      constexpr int UP = (U + 10) % 11;  // (y-1) mod 11
      filter_row(B ^ 1, y - 1, std::integral_constant<int, UP>{});
    }
    __syncwarp();
    if constexpr (!ASYNC) {
      o_m = o_mn;
      o_h = o_hn;
      r_m = r_mn;
      r_h = r_hn;
    }
  };

  // 11-row blocks keep the ring slots static (U = y mod 11).
  for (int jb = 0; jb < H32; jb += 11) {
#define CV_ROW(U)                                                   \
  if (jb + U < H32) do_row(jb + U, std::integral_constant<int, U>{});
    CV_ROW(0) CV_ROW(1) CV_ROW(2) CV_ROW(3) CV_ROW(4) CV_ROW(5)
    CV_ROW(6) CV_ROW(7) CV_ROW(8) CV_ROW(9) CV_ROW(10)
#undef CV_ROW
    ssum_d += (double)ssum;  // float partials over at most 11 rows
    ssum = 0.f;
  }
  {  // drain: filter the last row
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
  if constexpr (ASYNC) cp_async_wait<0>();
  if constexpr (FRAMES) flag_warp(args.err, qmax > args.Li, CV_FLAG_INT_RANGE);

  // warp reduction of the band partials (fixed shuffle tree: deterministic)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    ssum_d += __shfl_xor_sync(0xffffffffu, ssum_d, o);
  }
  if (lane == 0) {
    double *p = args.part + (((a * T + t) * args.nstrips) + strip) * 2 * C;
    p[c] = sse;
    p[C + c] = ssum_d;
  }
}

}  // namespace cvb
