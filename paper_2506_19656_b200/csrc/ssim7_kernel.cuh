// K5+K6 with SSIM — the decode + PSNR + SSIM kernel of the benchmark
// (frames + float32 original; every bit depth, with or without band PCA).
//
// Replaces, for the array path: _planar_bytes_to_frames (bridge.py:163-174),
// dropping padded planes (plan.py:106), dequantize (transform.py:108-126),
// pca_inverse (transform.py:202-210) and the absent metrics module's psnr /
// ssim (11x11 Gaussian window, sigma 1.5, valid region).
//
// CTA = one frame t of one cube, 128 adjacent input columns x0 .. x0+127
// (x0 = 118 s; the 118 output columns x0+5 .. x0+122 need their whole window
// inside the strip) and a group of up to four bands g*4 .. g*4+3. Warps:
//   * 16 "vertical" warps; lane = (column 8w + lane/4, band lane%4), so the
//     four bands of a pixel sit in adjacent lanes: conflict-free reads of the
//     channel-last original and contiguous recon runs;
//   * a loader warp (in its own warpgroup, which gives its registers to the
//     vertical warps with setmaxnreg) feeds a 4-stage input ring of row
//     pairs: one mbarrier-tracked bulk copy (cp.async.bulk, the TMA path) per
//     original row segment (all C bands of 128 pixels, contiguous) and per
//     frame-plane row segment;
// The recon is stored straight from the vertical lanes: a warp store covers
// 8 pixels x 4 bands, i.e. eight 16-byte runs of the channel-last cube.
// Per row every vertical lane decodes its element (float2 lookup table
// (hi, lo) of the exact float64 dequantisation for <= 10 bits; exact float64
// for 12/16-bit without PCA; float32 inverse PCA with the dequantisation
// folded into the coefficients), adds its float32 squared error (flushed to
// float64 every 8 rows), and runs the VERTICAL 11-tap filter of (s, d) and
// (s^2, d^2) as a transposed-form FIR with packed FFMA2 (s = x'+y', d = x-y,
// x' = x - peak): 22 FFMA2 per element. The column-filtered rows go to a
// 4-slot ring of row pairs; for every pair and band one vertical warp runs
// the HORIZONTAL filter (lane q: outputs 4q .. 4q+3 from 14 LDS.128, 22 FFMA2
// per output) and the SSIM of each output. Gaussian weights are compile-time
// immediates.
#pragma once
#include "eval_kernel.cuh"
#include "ssim_kernel.cuh"

namespace cvb {

constexpr int k7Cols = 128;
constexpr int k7Out = k7Cols - 2 * kSsimRadius;  // 118
constexpr int k7GB = 4;                          // bands per CTA
constexpr int k7VW = 16;                         // vertical warps (warpgroups 0-3)
constexpr int k7HW = 15;                         // horizontal warps (17 .. 31)
constexpr int k7LoadWarp = k7VW;                 // warp 16 feeds the input ring
constexpr int k7Threads = 1024;
constexpr int k7RegsV = 80;                      // setmaxnreg: vertical warpgroups
constexpr int k7RegsH = 48;                      // setmaxnreg: loader + horizontal warpgroups
constexpr int k7NS = 4;                          // input ring stages (row pairs)
constexpr int k7Ring = 6;                        // filtered-row ring slots (row pairs)
constexpr int k7Tasks = 2 * 4;                   // horizontal tasks per filtered pair (rows x bands)
constexpr int k7PcaMax = 12;
constexpr int k7LutMax = 1024;
constexpr int k7VbBand = 144;                    // float4 per band row (136 used + skew)
constexpr int k7VbRow = k7GB * k7VbBand;         // float4 per filtered row (4 bands)
constexpr int k7Bars = 256;                      // bytes reserved for mbarriers
enum { K7_LUT = 0, K7_F64 = 1, K7_PCA = 2 };

__host__ __device__ inline int ssim7_strips(int64_t W) { return (int)((W - 2 * kSsimRadius + k7Out - 1) / k7Out); }

struct Ssim7Geom {
  int ob, fb, np, stage, off_in, off_vb, off_lut, total;
};

// shared-memory geometry: np frame planes per row (PCA: E; else the group's bands)
__host__ __device__ inline Ssim7Geom ssim7_geom(int C, int np, int fsz, bool lut) {
  Ssim7Geom g;
  g.ob = ((k7Cols * C * 4 + 15) & ~15) + 32;  // 16-byte aligned copy of 128 pixels + slack
  g.fb = ((k7Cols * fsz + 15) & ~15) + 32;
  g.np = np;
  g.stage = 2 * g.ob + 2 * np * g.fb;
  g.off_in = k7Bars;
  g.off_vb = g.off_in + k7NS * g.stage;
  g.off_lut = g.off_vb + k7Ring * 2 * k7VbRow * 16;
  g.total = g.off_lut + (lut ? k7GB * k7LutMax * 8 : 0);
  return g;
}

// mbarriers and shared-memory accesses on 32-bit shared addresses. Ring data
// is read through volatile asm so that no load is hoisted above the barrier
// wait that publishes it.
__device__ __forceinline__ void mbar_init7(uint32_t b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive7(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx7(uint32_t b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(tx) : "memory");
}
__device__ __forceinline__ bool mbar_test7(uint32_t b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(b), "r"(parity)
      : "memory");
  return ok != 0;
}
// the waiting warp sleeps in try_wait (suspend-time hint) instead of spinning
// on issue slots the working warps need
__device__ __forceinline__ void mbar_wait7(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW7_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra W7_%=;\n}\n" ::"r"(b),
      "r"(parity), "n"(0x989680)
      : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on `bar` in bytes
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds_f32x2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32x4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// a value the compiler must keep (it cannot rematerialise it from thread
// indices inside the hot loop)
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;\n" : "=r"(r) : "r"(x));
  return r;
}
template <int FSZ>
__device__ __forceinline__ uint32_t lds_code(uint32_t a) {
  uint32_t v;
  if constexpr (FSZ == 2) asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(v) : "r"(a));
  else asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}

// a - b on packed pairs (one rounding: b * -1 + a)
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }

// transposed-form 11-tap FIR on packed pairs: zsd = (s, d), zq = (s^2, d^2);
// z[k] holds the partial sums of the output row completed k rows from now.
struct Fir2 {
  float2 zsd[10], zq[10];
};

__device__ __forceinline__ float4 fir2_step(Fir2 &f, float2 p) {
  const float2 q = __fmul2_rn(p, p);
  const float w0 = gtap(5);
  const float2 osd = __ffma2_rn(p, make_float2(w0, w0), f.zsd[0]);
  const float2 oq = __ffma2_rn(q, make_float2(w0, w0), f.zq[0]);
#pragma unroll
  for (int k = 1; k < 10; ++k) {
    const float wt = gtap(k - 5 < 0 ? 5 - k : k - 5);
    f.zsd[k - 1] = __ffma2_rn(p, make_float2(wt, wt), f.zsd[k]);
    f.zq[k - 1] = __ffma2_rn(q, make_float2(wt, wt), f.zq[k]);
  }
  f.zsd[9] = __fmul2_rn(p, make_float2(w0, w0));
  f.zq[9] = __fmul2_rn(q, make_float2(w0, w0));
  return make_float4(osd.x, osd.y, oq.x, oq.y);
}

__device__ __forceinline__ int vb_skew(int b) { return b * k7VbBand + ((b & 1) | ((b & 2) << 1)); }  // {0,1,4,5} mod 8
__device__ __forceinline__ int vb_idx(int col) { return (col & 3) * 34 + (col >> 2); }

// Raw inputs of one row pair for one lane, loaded one pair ahead of the math.
template <int EPL>
struct Raw7 {
  float om[2];
  uint32_t q[2][EPL];
  float2 lv[2];
};

// EP: PCA planes the loops are unrolled for (E for 6 and 9, k7PcaMax with
// runtime guards otherwise); 0 without PCA.
template <int RS, int MODE, int EP>
__global__ void __launch_bounds__(k7Threads, 1)
k_eval_ssim7(const EvalArgs args, const PcaParams inv) {
  using R = typename RawT<RS>::type;
  constexpr int FSZ = (int)sizeof(R);
  constexpr bool PCA = MODE == K7_PCA;
  constexpr int EPL = PCA ? EP : 1;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int C = args.C, E = args.E;
  const int ngrp = (C + k7GB - 1) / k7GB;
  const int strip = blockIdx.x / ngrp, g = blockIdx.x % ngrp;
  const int nb = min(k7GB, C - g * k7GB);
  const int64_t T = args.T, H = args.H, W = args.W, HW = H * W;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int64_t x0 = (int64_t)strip * k7Out;
  const int nstr = gridDim.x / ngrp;
  const bool last_strip = strip == nstr - 1;
  const int H32 = (int)H, W32 = (int)W;
  const int npairs = (H32 + 1) >> 1;
  const int np = PCA ? E : nb;
  const Ssim7Geom geo = ssim7_geom(C, PCA ? E : k7GB, FSZ, MODE == K7_LUT);

  const uint32_t s0 = smem_u32(smem);
  const uint32_t full_in = s0, empty_in = s0 + 8 * k7NS;                   // + 8 * stage
  const uint32_t vb_full = s0 + 16 * k7NS, vb_empty = vb_full + 8 * k7Ring;  // + 8 * slot
  const uint32_t in_ring = s0 + geo.off_in;
  const uint32_t vb = s0 + geo.off_vb;
  float2 *lut = reinterpret_cast<float2 *>(smem + geo.off_lut);
  const bool want_recon = args.recon_out != nullptr;
  const double L = args.L;

  if (threadIdx.x < k7NS) {
    mbar_init7(full_in + 8 * threadIdx.x, 1);  // the loader's expect_tx arrival + bytes
    mbar_init7(empty_in + 8 * threadIdx.x, k7VW);
  } else if (threadIdx.x < k7NS + k7Ring) {
    mbar_init7(vb_full + 8 * (threadIdx.x - k7NS), k7VW);
    mbar_init7(vb_empty + 8 * (threadIdx.x - k7NS), k7Tasks);
  }
  if constexpr (MODE == K7_LUT) {
    // (hi, lo) float pair of the exact float64 dequantisation of every code
    for (int i = threadIdx.x; i < k7GB * k7LutMax; i += blockDim.x) {
      const int b = i / k7LutMax, q = i % k7LutMax;
      if (b < nb && q <= (int)args.Li) {
        const double m = args.qmins[a * C + g * k7GB + b];
        const double sp = __dsub_rn(args.qmaxs[a * C + g * k7GB + b], m);
        const double v = dequantize_fast((uint32_t)q, m, sp, L, args.rL);
        const float hi = (float)v;
        lut[i] = make_float2(hi, (float)(v - (double)hi));
      }
    }
  }
  // the input ring starts zeroed: bytes no copy ever writes (columns past the
  // frame edge) read as 0, so the decode needs no per-element masking
  for (int i = threadIdx.x; i < k7NS * geo.stage / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(smem + geo.off_in)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // zeros before the first bulk copies
  __syncthreads();
  double2 *red = reinterpret_cast<double2 *>(smem + geo.off_vb);  // end-of-kernel partials

  if (w >= k7VW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(k7RegsH));
    if (w == k7LoadWarp) {
      // ---------------------------------------------------------------- loader warp
      const int64_t rowb = W * C * 4;
      const char *obase = reinterpret_cast<const char *>(args.orig) + (a * T + t) * H * rowb;
      const int64_t xe = min(x0 + k7Cols, W);
      const int64_t oa0 = (x0 * C * 4) & ~15ll, oa1 = (xe * C * 4 + 15) & ~15ll;
      const uint32_t obytes = (uint32_t)(oa1 - oa0);
      const int64_t fa0 = (x0 * FSZ) & ~15ll, fa1 = (xe * FSZ + 15) & ~15ll;
      const uint32_t fbytes = (uint32_t)(fa1 - fa0);
      const int ncp = 1 + np;  // copies per row
      // this lane's copy (k = lane): row k / ncp of the pair, piece k % ncp
      const int row_k = lane / ncp, piece = lane % ncp;
      const char *src = nullptr;
      uint32_t dst = 0, bytes = 0;
      int64_t stride = 0;
      if (lane < 2 * ncp) {
        if (piece == 0) {
          src = obase + oa0;
          dst = in_ring + row_k * geo.ob;
          bytes = obytes;
          stride = rowb;
        } else {
          const int j = PCA ? piece - 1 : g * k7GB + piece - 1;  // frame plane
          src = reinterpret_cast<const char *>(args.frames) +
                ((((a * args.G + j / 3) * T + t) * 3 + j % 3) * HW) * FSZ + fa0;
          dst = in_ring + 2 * geo.ob + ((piece - 1) * 2 + row_k) * geo.fb;
          bytes = fbytes;
          stride = W * FSZ;
        }
      }
      src += (int64_t)row_k * stride;
      const uint32_t tx = obytes + (uint32_t)np * fbytes;
      for (int p = 0; p < npairs; ++p) {
        const int st = p & (k7NS - 1);
        if (p >= k7NS) mbar_wait7(empty_in + 8 * st, (uint32_t)((p / k7NS) - 1) & 1u);
        const int rows = min(2, H32 - 2 * p);
        if (lane == 0) mbar_arrive_tx7(full_in + 8 * st, (uint32_t)rows * tx);
        __syncwarp();
        if (lane < rows * ncp) bulk_g2s(dst + (uint32_t)st * geo.stage, src, bytes, full_in + 8 * st);
        src += 2 * stride;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(k7Threads) : "memory");
      asm volatile("bar.sync 1, %0;\n" ::"n"(k7Threads) : "memory");
      return;
    }
    // ------------------------------------------------------------------ horizontal warps
    // task k = (filtered pair k / 8, row (k / 4) % 2, band k % 4); warp h takes
    // tasks h, h + 15, ...: lane q filters columns 4q .. 4q+13 of the row into
    // outputs 4q .. 4q+3 (14 LDS.128, 22 FFMA2 per output) and scores them
    const int hw = w - k7LoadWarp - 1;
    const int hq = lane;
    const int hlim = min(k7Out, W32 - kSsimTaps - (int)x0 + 1);  // valid output columns of the strip
    const bool hv_any = 4 * hq < hlim;
    float c0h[k7GB], C1h[k7GB], C2h[k7GB];
#pragma unroll
    for (int bq = 0; bq < k7GB; ++bq) {
      const double pk = bq < nb ? args.peaks[a * C + g * k7GB + bq] : 1.0;
      c0h[bq] = (float)pk;
      C1h[bq] = fmaxf((float)((0.01 * pk) * (0.01 * pk)), 1e-30f);
      C2h[bq] = fmaxf((float)((0.03 * pk) * (0.03 * pk)), 1e-30f);
    }
    double hsum[k7GB] = {0.0, 0.0, 0.0, 0.0};
    constexpr uint32_t kVbPair = 2u * k7VbRow * 16u;
    const int ntask = (npairs - 5) * k7Tasks;
#pragma unroll 1
    for (int k = hw; k < ntask; k += k7HW) {
      const int e = k >> 3, sub = (k >> 2) & 1, bb = k & 3;
      const int slot = e % k7Ring;
      mbar_wait7(vb_full + 8 * slot, (uint32_t)(e / k7Ring) & 1u);
      if (bb < nb && hv_any && 2 * e + sub <= H32 - kSsimTaps) {
        const uint32_t hv = vb + 16u * (uint32_t)(vb_skew(bb) + hq) + (uint32_t)slot * kVbPair +
                            (uint32_t)sub * (k7VbRow * 16u);
        float2 asd[4], aq[4];
        float4 nx = lds_f32x4(hv);
#pragma unroll
        for (int kk = 0; kk < 14; ++kk) {
          const float4 v = nx;
          if (kk + 1 < 14) nx = lds_f32x4(hv + 16u * (uint32_t)(((kk + 1) & 3) * 34 + ((kk + 1) >> 2)));
          const float2 vsd = make_float2(v.x, v.y), vq = make_float2(v.z, v.w);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int tp = kk - i;
            if (tp < 0 || tp > 10) continue;
            const float wt = gtap(tp < 5 ? 5 - tp : tp - 5);
            if (tp == 0) {
              asd[i] = __fmul2_rn(vsd, make_float2(wt, wt));
              aq[i] = __fmul2_rn(vq, make_float2(wt, wt));
            } else {
              asd[i] = __ffma2_rn(vsd, make_float2(wt, wt), asd[i]);
              aq[i] = __ffma2_rn(vq, make_float2(wt, wt), aq[i]);
            }
          }
        }
        float cc0 = c0h[0], cc1 = C1h[0], cc2 = C2h[0];
#pragma unroll
        for (int bq = 1; bq < k7GB; ++bq)
          if (bb == bq) {
            cc0 = c0h[bq];
            cc1 = C1h[bq];
            cc2 = C2h[bq];
          }
        float ts = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float s1 = ssim_px(asd[i].x, asd[i].y, aq[i].x, aq[i].y, cc0, cc1, cc2);
          ts += 4 * hq + i < hlim ? s1 : 0.f;
        }
#pragma unroll
        for (int bq = 0; bq < k7GB; ++bq)
          if (bb == bq) hsum[bq] += (double)ts;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive7(vb_empty + 8 * slot);
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(k7Threads) : "memory");
    // H partials: [hw][lane][band] after the V area (16 x 32 double2)
    double *hred = reinterpret_cast<double *>(red + k7VW * 32);
#pragma unroll
    for (int bq = 0; bq < k7GB; ++bq) hred[(hw * 32 + lane) * k7GB + bq] = hsum[bq];
    asm volatile("bar.sync 1, %0;\n" ::"n"(k7Threads) : "memory");
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(k7RegsV));

  // ------------------------------------------------------------------ vertical warps
  const int b = lane & 3, cl = lane >> 2;
  const int lc = 8 * w + cl;  // local input column
  const int c = g * k7GB + b;
  const bool bact = b < nb;
  const int xv = (int)x0 + lc;
  const bool vimg = xv < W32;
  const bool rd_lane = bact && vimg;
  const bool own = rd_lane && (lc < k7Out || last_strip);
  const double peak = bact ? args.peaks[a * C + c] : 1.0;
  const float c0 = (float)peak;

  // decode constants
  double dq_m = 0.0, dq_span = 0.0;
  float coef[EPL];
  float base = 0.f;
  coef[0] = 0.f;
  if constexpr (MODE == K7_F64) {
    if (bact) {
      dq_m = args.qmins[a * C + c];
      dq_span = __dsub_rn(args.qmaxs[a * C + c], dq_m);
    }
  }
  if constexpr (PCA) {
    // recon_c = mean_c + sum_j (min_j + q_j span_j / L) W[j][c]
    //         = base_c + sum_j q_j coef_cj   (float32; |error| << one code step)
    double bd = inv.mean[bact ? c : 0];
#pragma unroll
    for (int j = 0; j < EP; ++j) {
      coef[j] = 0.f;
      if (j < E && bact) {
        const double m = args.qmins[a * E + j];
        const double sp = __dsub_rn(args.qmaxs[a * E + j], m);
        coef[j] = (float)((sp / L) * inv.W[j * kMaxC + c]);
        bd = __fma_rn(m, inv.W[j * kMaxC + c], bd);
      }
    }
    base = (float)bd;
  }

  // per-lane shared-memory byte offsets inside a stage (lanes without data
  // read offset 0 of the stage, a valid address, and discard the value)
  // Lanes of an absent band (b >= nb) read the neighbouring band's finite
  // values, lanes past the frame edge read zeros: neither reaches a counted
  // output, so only the squared error and the recon store are masked.
  const uint32_t o_off = opaque((uint32_t)((x0 * C * 4) & 15) + (uint32_t)(lc * C + min(c, C - 1)) * 4u);
  const uint32_t f_off = opaque(2u * geo.ob + (uint32_t)((PCA ? 0 : 2 * min(b, nb - 1)) * geo.fb) +
                                (uint32_t)((x0 * FSZ) & 15) + (uint32_t)(lc * FSZ));
  const uint32_t code_hi = ~args.Li;  // a code with these bits set is out of range
  const uint32_t ob = geo.ob, fb = geo.fb;
  const uint32_t lut_b = opaque(s0 + geo.off_lut + (uint32_t)(b * k7LutMax * 8));
  uint32_t qor = 0;
  float sse_f = 0.f;
  double sse = 0.0;
  float *wq = want_recon ? args.recon_out + (a * T + t) * HW * C + (int64_t)xv * C + c : nullptr;
  const bool wr = want_recon && own;
  const int64_t rstride = W * C;  // recon row stride (floats)
  float *wq1 = wq + rstride;

  // raw loads of pair p (stage st): original values, codes (+ LUT entries)
  auto load_raw = [&](uint32_t st, Raw7<EPL> &rw) {
#pragma unroll
    for (int sub = 0; sub < 2; ++sub) {
      rw.om[sub] = lds_f32(st + (uint32_t)sub * ob + o_off);
      const uint32_t fa = st + f_off + (uint32_t)sub * fb;
      if constexpr (PCA) {
#pragma unroll
        for (int j = 0; j < EP; ++j)
          if (j < E) rw.q[sub][j] = lds_code<FSZ>(fa + (uint32_t)(2 * j) * fb);
      } else {
        rw.q[sub][0] = lds_code<FSZ>(fa);
        if constexpr (MODE == K7_LUT) rw.lv[sub] = lds_f32x2(lut_b + 8u * min(rw.q[sub][0], (uint32_t)(k7LutMax - 1)));
      }
    }
  };
  // decode math of a row pair: recon values and the SSIM input pairs (s, d);
  // `ok1` = the pair's second row exists (odd H)
  auto decode = [&](const Raw7<EPL> &rw, bool ok1, float &r0, float &r1, float2 &sd0, float2 &sd1) {
    float2 rv, df;
    const float2 om = make_float2(rw.om[0], rw.om[1]);
    if constexpr (PCA) {
      // both rows at once: acc = base + sum_j q_j coef_j (packed FFMA2)
      float2 acc = make_float2(base, base);
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        if (j < E) {
          qor |= rw.q[0][j] | rw.q[1][j];
          acc = __ffma2_rn(make_float2((float)rw.q[0][j], (float)rw.q[1][j]), make_float2(coef[j], coef[j]), acc);
        }
      }
      rv = acc;
      df = fsub2(om, rv);
    } else {
      qor |= rw.q[0][0] | rw.q[1][0];
      if constexpr (MODE == K7_LUT) {
        rv = make_float2(rw.lv[0].x, rw.lv[1].x);
        df = fsub2(fsub2(om, rv), make_float2(rw.lv[0].y, rw.lv[1].y));
      } else {
        const double rm0 = dequantize_fast(rw.q[0][0], dq_m, dq_span, L, args.rL);
        const double rm1 = dequantize_fast(rw.q[1][0], dq_m, dq_span, L, args.rL);
        rv = make_float2((float)rm0, (float)rm1);
        df = make_float2((float)__dsub_rn((double)om.x, rm0), (float)__dsub_rn((double)om.y, rm1));
      }
    }
    const float d0 = own ? df.x : 0.f, d1 = (own && ok1) ? df.y : 0.f;
    sse_f = fmaf(d1, d1, fmaf(d0, d0, sse_f));
    r0 = rv.x;
    r1 = rv.y;
    const float2 sv = __fadd2_rn(__fadd2_rn(om, rv), make_float2(-2.f * c0, -2.f * c0));
    sd0 = make_float2(sv.x, df.x);
    sd1 = make_float2(sv.y, df.y);
  };

  Fir2 fir;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    fir.zsd[i] = make_float2(0.f, 0.f);
    fir.zq[i] = make_float2(0.f, 0.f);
  }

  constexpr uint32_t kVbPair = 2u * k7VbRow * 16u;  // bytes of one ring slot (row pair)
  const uint32_t vb_st = opaque(vb + 16u * (uint32_t)(vb_skew(b) + vb_idx(lc)));

  // Software pipeline: iteration p holds the decoded pair p, loads the raw
  // inputs of pair p+1 (their shared-memory latency overlaps pair p's FIR),
  // stores pair p's recon, runs its vertical FIR (filtered pair p-5 goes to
  // ring slot (p-5) % 6) and decodes pair p+1 last.
  float r0, r1;
  float2 sd0, sd1;
  {
    Raw7<EPL> rw;
    mbar_wait7(full_in, 0u);
    load_raw(in_ring, rw);
    decode(rw, 1 < H32, r0, r1, sd0, sd1);
    __syncwarp();
    if (lane == 0) mbar_arrive7(empty_in);
  }
  uint32_t vs_off = 0;    // byte offset of the next ring slot to store
  int vs_slot = 0;        // its index
  uint32_t vs_phase = 0;  // its lap parity
#pragma unroll 1
  for (int p = 0; p < npairs; ++p) {
    const bool more = p + 1 < npairs;
    const int U1 = (p + 1) & (k7NS - 1);
    const uint32_t st1 = in_ring + (uint32_t)U1 * geo.stage;
    Raw7<EPL> rw;
    if (more) {
      mbar_wait7(full_in + 8 * U1, (uint32_t)((p + 1) >> 2) & 1u);
      load_raw(st1, rw);
    }
    if (wr) {  // the four bands of a pixel sit in adjacent lanes: 16-byte runs per pixel
      wq[0] = r0;
      if (2 * p + 1 < H32) wq1[0] = r1;
    }
    wq += 2 * rstride;
    wq1 += 2 * rstride;
    const float4 o0 = fir2_step(fir, sd0);
    const float4 o1 = fir2_step(fir, sd1);
    if (p >= 5) {  // column-filtered rows 2p-10, 2p-9 = pair p-5
      if (p - 5 >= k7Ring) mbar_wait7(vb_empty + 8 * vs_slot, vs_phase ^ 1u);
      const uint32_t d = vb_st + vs_off;
      sts_f32x4(d, o0);
      sts_f32x4(d + k7VbRow * 16u, o1);
      __syncwarp();
      if (lane == 0) mbar_arrive7(vb_full + 8 * vs_slot);
      vs_off += kVbPair;
      if (++vs_slot == k7Ring) {
        vs_slot = 0;
        vs_off = 0;
        vs_phase ^= 1u;
      }
    }
    if (more) {
      decode(rw, 2 * p + 3 < H32, r0, r1, sd0, sd1);  // odd H: the last pair's second row does not exist
      __syncwarp();
      if (lane == 0) mbar_arrive7(empty_in + 8 * U1);
    }
    if ((p & 3) == 3) {
      sse += (double)sse_f;
      sse_f = 0.f;
    }
  }
  sse += (double)sse_f;
  flag_warp(args.err, (qor & code_hi) != 0u, CV_FLAG_INT_RANGE);

  // deterministic CTA reduction: per band, fixed order over warps and lanes
  asm volatile("bar.sync 1, %0;\n" ::"n"(k7Threads) : "memory");  // the ring is idle
  red[w * 32 + lane] = make_double2(sse, 0.0);
  asm volatile("bar.sync 1, %0;\n" ::"n"(k7Threads) : "memory");  // all partials written
  if (threadIdx.x < nb) {
    const int bq = threadIdx.x;
    const double *hred = reinterpret_cast<const double *>(red + k7VW * 32);
    double s1 = 0.0, s2 = 0.0;
    for (int ww = 0; ww < k7VW; ++ww)
      for (int l = bq; l < 32; l += 4) s1 += red[ww * 32 + l].x;
    for (int i = 0; i < k7HW * 32; ++i) s2 += hred[i * k7GB + bq];
    double *pp = args.part + ((a * T + t) * args.nstrips + strip) * 2 * C;
    pp[g * k7GB + bq] = s1;
    pp[C + g * k7GB + bq] = s2;
  }
}

}  // namespace cvb
