// K5+K6 device code: fused decode + PSNR/SSIM (see eval.cu for the host side).
//
// One CTA per (cube, frame t, column strip of TX pixels) walks the H rows of
// its strip top to bottom; thread (px, c) owns output column x0+px, band c.
// Per row each thread converts its own input element (dequantise in float64,
// SSE, recon write) and threads tid < 10*C also convert one of the 5-pixel
// halo elements; the four SSIM maps (s, d, s^2, d^2) of the strip row go to
// shared memory as float4; each thread then runs the horizontal 11-tap
// Gaussian and scatters into an 11-slot register ring (vertical filter).
// Gaussian weights are compile-time immediates (full-rate FFMA: 120
// FMA/clk/SM measured on B200 vs 77 for the register form); the row loop is
// unrolled by 11 so ring slots are static registers. Row y+1 is prefetched
// into registers while row y is processed.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "pca_params.cuh"

namespace cvb {

struct EvalArgs {
  const void *frames;
  int E, G;
  const double *qmins, *qmaxs;
  int bit_depth;
  double L, rL;  // 2^B-1 and RN(1/L)
  uint32_t Li;
  const void *recon_in;
  const void *orig;
  int64_t T, H, W;
  int C;
  const double *peaks;
  float *recon_out;
  double *part;  // [n][T][nstrips][2C]
  uint32_t *err;
  int TX, nstrips;
  int ssim7;  // launch k_eval_ssim7 (nstrips = ssim7_strips(W))
  int psnr_vec;  // launch k_eval_psnr (nstrips = pixel chunks per frame)
};

enum { RS_FRAMES_U8 = 0, RS_FRAMES_U16 = 1, RS_RECON_F32 = 2, RS_RECON_F64 = 3 };

__host__ __device__ inline int eval_tx(int C, bool ssim) {
  if (!ssim) return C <= 8 ? 64 : 32;
  return 32;  // k_eval_ssim: one lane per output column
}

// Gaussian taps g[|k|], k = -5..5, sigma = 1.5, normalised (float32 of the
// float64 weights of the oracle).
#define CV_G0 0.26601171493530273f
#define CV_G1 0.21300554275512695f
#define CV_G2 0.10936068743467331f
#define CV_G3 0.036000773310661316f
#define CV_G4 0.0075987582094967365f
#define CV_G5 0.001028380123898387f

__device__ __forceinline__ constexpr float gtap(int k) {
  return k == 0 ? CV_G0 : k == 1 ? CV_G1 : k == 2 ? CV_G2 : k == 3 ? CV_G3 : k == 4 ? CV_G4 : CV_G5;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// SSIM from the filtered maps of s = x'+y' and d = x-y (x' = x-c0, y' = y-c0):
//   mu_x = (ms+md)/2 + c0, mu_y = (ms-md)/2 + c0,
//   sigma_x^2+sigma_y^2 = (vs+vd)/2, 2 sigma_xy = (vs-vd)/2,
// written as l = 1 - md^2/den_l, cs = 1 - vd/den_c so the float32 rounding
// only touches the small difference terms. C1, C2 > 0 keep den_l, den_c > 0.
// mu_x^2 + mu_y^2 = (u^2 + md^2)/2 with u = ms + 2 c0 (13 instructions).
__device__ __forceinline__ float ssim_px(float ms, float md, float ess, float edd, float c0,
                                         float C1, float C2) {
  const float u = fmaf(2.f, c0, ms);
  const float md2 = md * md;
  const float vd = fmaf(-md, md, edd);
  const float vs = fmaf(-ms, ms, ess);
  const float den_l = fmaf(0.5f, fmaf(u, u, md2), C1);
  const float den_c = fmaf(0.5f, vs + vd, C2);
  const float l = fmaf(-md2, rcp_approx(den_l), 1.f);
  const float cs = fmaf(-vd, rcp_approx(den_c), 1.f);
  return l * cs;
}

// One ring step of the vertical 11-tap filter for input row y, U = y mod 11.
// Slot (U+5)%11 starts output row y+5 (first contribution: a plain multiply,
// no zeroing); slot (U+6)%11 completes output row y-5.
struct Ring {
  float s[11], d[11], ss[11], dd[11];
};

template <int U>
__device__ __forceinline__ void ring_step(Ring &r, float hs, float hd, float hss, float hdd,
                                          float &os, float &od, float &oss, float &odd) {
#pragma unroll
  for (int i = -kSsimRadius; i <= kSsimRadius; ++i) {
    const int slot = (U + i + 11) % 11;
    const float w = gtap(i < 0 ? -i : i);
    if (i == kSsimRadius) {
      r.s[slot] = w * hs;
      r.d[slot] = w * hd;
      r.ss[slot] = w * hss;
      r.dd[slot] = w * hdd;
    } else {
      r.s[slot] = fmaf(w, hs, r.s[slot]);
      r.d[slot] = fmaf(w, hd, r.d[slot]);
      r.ss[slot] = fmaf(w, hss, r.ss[slot]);
      r.dd[slot] = fmaf(w, hdd, r.dd[slot]);
    }
  }
  constexpr int fs = (U + 6) % 11;
  os = r.s[fs];
  od = r.d[fs];
  oss = r.ss[fs];
  odd = r.dd[fs];
}

template <int RS> struct RawT { using type = double; };
template <> struct RawT<RS_FRAMES_U8> { using type = uint8_t; };
template <> struct RawT<RS_FRAMES_U16> { using type = uint16_t; };
template <> struct RawT<RS_RECON_F32> { using type = float; };

#ifndef CVB_EVAL_MAXT
#define CVB_EVAL_MAXT 512
#define CVB_EVAL_MINB 1
#endif

template <typename TO, int RS, bool PCA, bool SSIM>
__global__ void __launch_bounds__(CVB_EVAL_MAXT, CVB_EVAL_MINB)
k_eval(const EvalArgs args, const PcaParams inv) {
  using R = typename RawT<RS>::type;
  constexpr bool FRAMES = (RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16);
  constexpr int HALO = SSIM ? kSsimRadius : 0;
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = blockDim.x, tid = threadIdx.x;
  const int C = args.C, E = args.E, TX = args.TX;
  const int NX = TX + 2 * HALO;
  const int NXC = NX * C;
  const int64_t T = args.T, H = args.H, W = args.W;
  const int64_t HW = H * W, inner = HW * C, rowlen = W * C;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int64_t x0 = (int64_t)blockIdx.x * TX;
  const int c = tid % C;
  const int px = tid / C;

  // shared memory: srow [2][NXC] float4 | rec [NXC] double | qm, qs [E]
  float4 *srow = reinterpret_cast<float4 *>(smem);
  size_t off = SSIM ? 2 * (size_t)NXC * sizeof(float4) : 0;
  double *rec = reinterpret_cast<double *>(smem + off);
  off += PCA ? (size_t)NXC * sizeof(double) : 0;
  double *qm = reinterpret_cast<double *>(smem + off);
  double *qs = qm + (PCA ? E : 0);
  if constexpr (PCA) {
    for (int j = tid; j < E; j += NT) {
      qm[j] = args.qmins[a * E + j];
      qs[j] = __dsub_rn(args.qmaxs[a * E + j], qm[j]);
    }
    __syncthreads();
  }
  double my_m = 0.0, my_span = 0.0;
  if constexpr (!PCA && FRAMES) {
    my_m = args.qmins[a * E + c];
    my_span = __dsub_rn(args.qmaxs[a * E + c], my_m);
  }
  const double peak = args.peaks ? args.peaks[a * C + c] : 1.0;
  const float c0 = (float)peak;
  // a zero peak makes C1 = C2 = 0; the floor keeps constant windows at SSIM 1
  const float C1 = fmaxf((float)((0.01 * peak) * (0.01 * peak)), 1e-30f);
  const float C2 = fmaxf((float)((0.03 * peak) * (0.03 * peak)), 1e-30f);
  const bool col_valid = SSIM && (x0 + px >= HALO) && (x0 + px < W - HALO);

  // ---- element slots: main = (x0+px, c); halo (tid < 10C) = one of the 10 halo columns
  const int64_t xm = x0 + px;
  const bool mimg = xm < W;
  const int hp = tid / C;  // 0..9 for halo threads
  const bool hact = SSIM && tid < 2 * HALO * C;
  const int pin_h = hp < HALO ? hp : TX + hp;
  const int64_t xh = x0 - HALO + pin_h;
  const bool himg = hact && xh >= 0 && xh < W;
  const float mmask = mimg ? 1.f : 0.f, hmask = himg ? 1.f : 0.f;

  const TO *obase = reinterpret_cast<const TO *>(args.orig) + (a * T + t) * inner;
  const TO *op_m = obase + (mimg ? xm : 0) * C + c;
  const TO *op_h = obase + (himg ? xh : 0) * C + c;
  const R *rp_m = nullptr, *rp_h = nullptr;
  int64_t rrow = rowlen;
  if constexpr (FRAMES && !PCA) {
    const R *fb = reinterpret_cast<const R *>(args.frames) + (((a * args.G + c / 3) * T + t) * 3 + c % 3) * HW;
    rp_m = fb + (mimg ? xm : 0);
    rp_h = fb + (himg ? xh : 0);
    rrow = W;
  } else if constexpr (!FRAMES) {
    const R *rb = reinterpret_cast<const R *>(args.recon_in) + (a * T + t) * inner;
    rp_m = rb + (mimg ? xm : 0) * C + c;
    rp_h = rb + (himg ? xh : 0) * C + c;
  }
  float *wp = (args.recon_out && mimg) ? args.recon_out + (a * T + t) * inner + xm * C + c : nullptr;
  const int sidx_m = (px + HALO) * C + c;
  const int sidx_h = pin_h * C + c;

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

  double sse = 0.0, ssum_d = 0.0;
  float ssum = 0.f;
  uint32_t qmax = 0;
  Ring ring;
#pragma unroll
  for (int i = 0; i < 11; ++i) ring.s[i] = ring.d[i] = ring.ss[i] = ring.dd[i] = 0.f;
  int buf = 0;

  // recon of one element from its raw value (float64, reference rounding)
  auto recon_of = [&](R raw, int sidx) -> double {
    if constexpr (PCA) {
      return rec[sidx];
    } else if constexpr (FRAMES) {
      const uint32_t q = (uint32_t)raw;
      qmax = max(qmax, q);
      return dequantize_fast(q, my_m, my_span, args.L, args.rL);
    } else {
      return (double)raw;
    }
  };

  load_next();
  o_m = o_mn;
  o_h = o_hn;
  r_m = r_mn;
  r_h = r_hn;

  auto do_row = [&](int64_t y, auto ucst) {
    constexpr int U = decltype(ucst)::value;
    if (y + 1 < H) load_next();
    // ---- PCA: dequantise the strip row's components and invert (1 thread / pixel)
    if constexpr (PCA) {
      for (int p = tid; p < NX; p += NT) {
        const int64_t x = x0 - HALO + p;
        if (x < 0 || x >= W) continue;
        double pc[kMaxC];
#pragma unroll
        for (int j = 0; j < kMaxC; ++j) {
          if (j < E) {
            const int64_t fi = (((a * args.G + j / 3) * T + t) * 3 + j % 3) * HW + y * W + x;
            const uint32_t q = (uint32_t)ldg(reinterpret_cast<const R *>(args.frames) + fi);
            qmax = max(qmax, q);
            pc[j] = dequantize_fast(q, qm[j], qs[j], args.L, args.rL);
          }
        }
        for (int cc = 0; cc < C; ++cc) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < kMaxC; ++j)
            if (j < E) acc = __fma_rn(pc[j], inv.W[j * kMaxC + cc], acc);
          rec[p * C + cc] = __dadd_rn(acc, inv.mean[cc]);
        }
      }
      __syncthreads();
    }
    // ---- main element: recon, SSE, recon write, SSIM maps
    {
      const double r = recon_of(r_m, sidx_m);
      const float of = (float)o_m;
      const double diff = __dsub_rn((double)o_m, r);
      if (mimg) {
        sse = __fma_rn(diff, diff, sse);
        if (wp) {
          *wp = (float)r;
          wp += rowlen;
        }
      }
      if constexpr (SSIM) {
        const float d = (float)diff * mmask;
        const float sv = fmaf(2.f, of - c0, -d) * mmask;
        srow[(size_t)buf * NXC + sidx_m] = make_float4(sv, d, sv * sv, d * d);
      }
    }
    if constexpr (SSIM) {
      if (hact) {
        const double r = recon_of(r_h, sidx_h);
        const float of = (float)o_h;
        const float d = (float)__dsub_rn((double)o_h, r) * hmask;
        const float sv = fmaf(2.f, of - c0, -d) * hmask;
        srow[(size_t)buf * NXC + sidx_h] = make_float4(sv, d, sv * sv, d * d);
      }
      __syncthreads();
      const float4 *sr = srow + (size_t)buf * NXC + px * C + c;
      float hs = 0.f, hd = 0.f, hss = 0.f, hdd = 0.f;
#pragma unroll
      for (int k = 0; k < kSsimTaps; ++k) {
        const float4 v = sr[k * C];
        const float w = gtap(k < kSsimRadius ? kSsimRadius - k : k - kSsimRadius);
        hs = fmaf(w, v.x, hs);
        hd = fmaf(w, v.y, hd);
        hss = fmaf(w, v.z, hss);
        hdd = fmaf(w, v.w, hdd);
      }
      float os, odv, oss, odd;
      ring_step<U>(ring, hs, hd, hss, hdd, os, odv, oss, odd);
      if (y >= 2 * kSsimRadius && col_valid) ssum += ssim_px(os, odv, oss, odd, c0, C1, C2);
      buf ^= 1;
    } else if constexpr (PCA) {
      __syncthreads();  // rec is rewritten for the next row
    }
    o_m = o_mn;
    o_h = o_hn;
    r_m = r_mn;
    r_h = r_hn;
  };

  for (int64_t jb = 0; jb < H; jb += 11) {
#define CV_ROW(U)                                                   \
  if (jb + U < H) do_row(jb + U, std::integral_constant<int, U>{});
    CV_ROW(0) CV_ROW(1) CV_ROW(2) CV_ROW(3) CV_ROW(4) CV_ROW(5)
    CV_ROW(6) CV_ROW(7) CV_ROW(8) CV_ROW(9) CV_ROW(10)
#undef CV_ROW
    ssum_d += (double)ssum;  // float partials over at most 11 rows
    ssum = 0.f;
  }
  if constexpr (FRAMES) flag_warp(args.err, qmax > args.Li, CV_FLAG_INT_RANGE);

  // per-band partials: threads c, c+C, ... share band c (NT multiple of C)
  __syncthreads();
  double *red = reinterpret_cast<double *>(smem);
  red[tid] = sse;
  red[NT + tid] = ssum_d;
  __syncthreads();
  if (tid < C) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = tid; i < NT; i += C) {
      s1 += red[i];
      s2 += red[NT + i];
    }
    double *p = args.part + (((a * T + t) * args.nstrips) + blockIdx.x) * 2 * C;
    p[tid] = s1;
    p[C + tid] = s2;
  }
}

}  // namespace cvb
