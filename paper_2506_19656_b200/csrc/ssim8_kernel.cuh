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
// inside the strip) and a group of up to four bands g*4 .. g*4+3; it walks the
// frame top to bottom in row pairs. 32 warps in two roles:
//   * 16 "vertical" warps (88 registers); lane = (column 8w + lane/4, band
//     lane%4): conflict-free reads of the channel-last original, 16-byte recon
//     runs. Per row pair a lane decodes its two elements (float2 lookup table
//     of the exact float64 dequantisation for <= 10 bits; exact float64 for
//     12/16-bit without PCA; float32 inverse PCA with the dequantisation
//     folded into the coefficients), stores the recon, adds the squared error
//     and steps the VERTICAL 11-tap filter of (s, d) and (s^2, d^2), a
//     transposed-form FIR on packed FFMA2 (s = x'+y', d = x-y, x' = x - peak).
//     Column-filtered row pairs go to a 5-slot shared ring.
//   * 15 "horizontal" workers (40 registers; their float64 SSIM sums live in
//     shared memory) take the (row, band) tasks of the filtered pairs
//     round-robin. Lane q filters columns 4q .. 4q+13 of a row into outputs
//     4q .. 4q+3 (14 LDS.128, 22 FFMA2 per output) and scores them. The
//     horizontal role has slack: it waits on "filled" rather than making the
//     vertical warps wait on "drained".
//   * 1 loader warp (in the horizontal warpgroups) feeds the input ring:
//     mbarrier-tracked bulk copies (cp.async.bulk, the TMA path), one per
//     original row segment (all C bands of 128 pixels) and per frame-plane row
//     segment, as far ahead as the ring (up to 5 row pairs) allows.
// The filtered-row ring is handed over through mbarriers in both directions (see
// "Hand-offs" below), the input stages are released to the loader through named
// barriers. Gaussian weights are compile-time immediates.
#pragma once
#include "eval_kernel.cuh"
#include "ssim_kernel.cuh"

namespace cvb {

constexpr int k8Cols = 128;
constexpr int k8Out = k8Cols - 2 * kSsimRadius;  // 118
constexpr int k8GB = 4;                          // bands per CTA
constexpr int k8VW = 16;                         // vertical warps (warpgroups 0-3)
constexpr int k8HW = 16;                         // horizontal warpgroups' warps (4-7): 15 workers + the loader
constexpr int k8HWork = k8HW - 1;
constexpr int k8Threads = 32 * (k8VW + k8HW);
constexpr int k8RegsV = 88;                      // setmaxnreg: vertical warpgroups
constexpr int k8RegsH = 40;                      // setmaxnreg: horizontal warpgroups (512 x 88 + 512 x 40 = the register file)
constexpr int k8NSMax = 5;                       // input ring stages (row pairs)
constexpr int k8SmemMax = 227 * 1024;
constexpr int k8Ring = 5;                        // filtered-row ring slots (row pairs) = pairs per unrolled group
constexpr int k8PcaMax = 12;
constexpr int k8LutMax = 1024;
constexpr int k8VbBand = 144;                    // float4 per band row (136 used + skew)
constexpr int k8VbRow = k8GB * k8VbBand;         // float4 per filtered row (4 bands)
constexpr int k8Bars = 192;                      // bytes of mbarriers: full_in[3] at 0, drained[6] at 64, filled[6] at 128
constexpr int k8Desc = k8GB * 16;                // bytes of the per-band SSIM constants (c0, C1, C2)
constexpr int k8Coef = k8GB * k8PcaMax * 4;      // bytes of the inverse-PCA coefficients [band][plane]
constexpr int k8HsBytes = k8HW * 32 * k8GB * 8;  // per-thread float64 SSIM sums of the horizontal warps [thread][band]
// Hand-offs:
//   filled[slot]   mbarrier, one arrival per vertical warp (lane 0 after __syncwarp);
//                  a horizontal worker waits for it alone (try_wait suspends the warp in
//                  hardware). As a named barrier (bar.sync over 16 + 8 warps) it completed
//                  only when ALL eight workers of the pair had reached it, so the workers ran
//                  pair by pair in step, three of the eleven idle: 68.7 -> 58.8 ms on config 5.
//   drained[slot]  mbarrier, one arrival per (row, band) task; a vertical warp waits for it
//                  on its own before it overwrites the slot (no vertical-vertical lock-step).
//   k8BarStage + stage   named barrier: the vertical warps arrive when they have read an
//                  input stage, the loader waits parked before refilling it.
constexpr int k8BarStage = 1;
static_assert(k8BarStage + k8NSMax <= 16, "named barrier ids");
enum { K8_LUT = 0, K8_F64 = 1, K8_PCA = 2 };

__host__ __device__ inline int ssim8_strips(int64_t W) { return (int)((W - 2 * kSsimRadius + k8Out - 1) / k8Out); }

struct Ssim8Geom {
  int ob, fb, np, ns, stage, off_desc, off_coef, off_in, off_vb, off_lut, off_hs, total;
};

// shared-memory geometry: np frame planes per row (PCA: E; else the group's bands)
__host__ __device__ inline Ssim8Geom ssim8_geom(int C, int np, int fsz, bool lut) {
  Ssim8Geom g;
  g.ob = ((k8Cols * C * 4 + 15) & ~15) + 32;  // 16-byte aligned copy of 128 pixels + slack
  g.fb = ((k8Cols * fsz + 15) & ~15) + 32;
  g.np = np;
  g.stage = 2 * g.ob + 2 * np * g.fb;
  g.off_desc = k8Bars;
  g.off_coef = g.off_desc + k8Desc;
  g.off_in = g.off_coef + k8Coef;
  const int rest = g.off_in + k8Ring * 2 * k8VbRow * 16 + (lut ? k8GB * k8LutMax * 8 : 0) + k8HsBytes;
  g.ns = (k8SmemMax - rest) / g.stage;
  g.ns = g.ns > k8NSMax ? k8NSMax : g.ns;  // < 2: the kernel cannot run (the launcher checks)
  g.off_vb = g.off_in + g.ns * g.stage;
  g.off_lut = g.off_vb + k8Ring * 2 * k8VbRow * 16;
  g.off_hs = g.off_lut + (lut ? k8GB * k8LutMax * 8 : 0);
  g.total = g.off_hs + k8HsBytes;
  return g;
}

__device__ __forceinline__ void mbar_init8(uint32_t b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx8(uint32_t b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(tx) : "memory");
}
// try_wait suspends the thread in hardware for a bounded time; looping on it is
// the nearest thing to a parked wait an mbarrier offers (the time hint keeps the polls
// rare: without it 13 % of the issued instructions of the kernel were polls)
__device__ __forceinline__ void mbar_wait8(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n}\n" ::"r"(b), "r"(parity), "r"(0x989680u)
      : "memory");
}
// (Sleeping between the workers' polls measured no better: nanosleep 400 -> 53.7 ms, nanosleep 48
// -> 53.3 ms, tight try_wait loop 53.1 ms on config 5.)
// global -> shared bulk copy (TMA engine), completion counted on `bar` in bytes
__device__ __forceinline__ void bulk_g2s8(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// named barriers: producers arrive, consumers sync (both count towards `n` threads)
__device__ __forceinline__ void nbar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
// Ring data is read through volatile asm so that no load is hoisted above the
// barrier that publishes it.
__device__ __forceinline__ float lds8_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds8_f32x2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds8_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts8_f32x4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
template <int FSZ>
__device__ __forceinline__ uint32_t lds8_code(uint32_t a) {
  uint32_t v;
  if constexpr (FSZ == 2) asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(v) : "r"(a));
  else asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}

// a value the compiler must keep in a register (it cannot rematerialise it
// from thread indices inside the hot loop)
__device__ __forceinline__ uint32_t opaque8(uint32_t x) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;\n" : "=r"(r) : "r"(x));
  return r;
}

// a - b on packed pairs (one rounding: b * -1 + a)
__device__ __forceinline__ float2 fsub2_8(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }

// Transposed-form 11-tap FIR on packed pairs, updated IN PLACE: zsd = (s, d),
// zq = (s^2, d^2). The output row born at step i lives in slot i % 10 for its
// ten following steps; step S (= row index mod 10, a compile-time constant of
// the 5-pair unrolled loop) completes and restarts slot S and adds the row to
// the nine others with the weight of their age. Every FFMA2 has its
// accumulator as destination: the shifting form (z[k-1] = p w + z[k]) made the
// compiler rotate the 40 state registers with ~15 MOV / IMAD.MOV per row.
struct Fir8 {
  float2 zsd[10], zq[10];
};

template <int S>
__device__ __forceinline__ float4 fir8_step(Fir8 &f, float2 p) {
  const float2 q = __fmul2_rn(p, p);
  const float w0 = gtap(5);
  const float2 osd = __ffma2_rn(p, make_float2(w0, w0), f.zsd[S]);
  const float2 oq = __ffma2_rn(q, make_float2(w0, w0), f.zq[S]);
  f.zsd[S] = __fmul2_rn(p, make_float2(w0, w0));
  f.zq[S] = __fmul2_rn(q, make_float2(w0, w0));
#pragma unroll
  for (int age = 1; age < 10; ++age) {
    const int j = (S - age + 10) % 10;
    const float wt = gtap(age < 5 ? 5 - age : age - 5);
    f.zsd[j] = __ffma2_rn(p, make_float2(wt, wt), f.zsd[j]);
    f.zq[j] = __ffma2_rn(q, make_float2(wt, wt), f.zq[j]);
  }
  return make_float4(osd.x, osd.y, oq.x, oq.y);
}

template <int U>
struct PairIdx8 {
  static constexpr int value = U;
};

__device__ __forceinline__ int vb8_skew(int b) { return b * k8VbBand + ((b & 1) | ((b & 2) << 1)); }  // {0,1,4,5} mod 8
__device__ __forceinline__ int vb8_idx(int col) { return (col & 3) * 34 + (col >> 2); }

// EP: PCA planes the loops are unrolled for; EXACT: E == EP (6 and 9), else
// k8PcaMax with runtime guards; 0 without PCA.
template <int RS, int MODE, int EP, bool EXACT, bool CHKQ = true>
__global__ void __launch_bounds__(k8Threads, 1)
k_eval_ssim8(const EvalArgs args, const PcaParams inv) {
  using R = typename RawT<RS>::type;
  constexpr int FSZ = (int)sizeof(R);
  constexpr bool PCA = MODE == K8_PCA;
  constexpr int EPL = PCA ? EP : 1;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int C = args.C, E = EXACT ? EP : args.E;
  const int ngrp = (C + k8GB - 1) / k8GB;
  const int strip = blockIdx.x / ngrp, g = blockIdx.x % ngrp;
  const int nb = min(k8GB, C - g * k8GB);
  const int64_t T = args.T, H = args.H, W = args.W, HW = H * W;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int64_t x0 = (int64_t)strip * k8Out;
  const int nstr = gridDim.x / ngrp;
  const bool last_strip = strip == nstr - 1;
  const int H32 = (int)H, W32 = (int)W;
  const int npairs = (H32 + 1) >> 1;
  const int nfe = npairs - 5;  // filtered pairs (output rows 2e, 2e+1)
  const int np = PCA ? E : nb;
  const Ssim8Geom geo = ssim8_geom(C, PCA ? E : k8GB, FSZ, MODE == K8_LUT);

  const uint32_t s0 = smem_u32(smem);
  const int ns = geo.ns;
  const uint32_t full_in = s0;  // + 8 * stage
  const uint32_t in_ring = s0 + geo.off_in;
  const uint32_t vb = s0 + geo.off_vb;
  float2 *lut = reinterpret_cast<float2 *>(smem + geo.off_lut);
  const double L = args.L;

  if (threadIdx.x < k8NSMax) mbar_init8(full_in + 8 * threadIdx.x, 1);  // the loader's expect_tx arrival + bytes
  if (threadIdx.x >= 32 && threadIdx.x < 32 + k8Ring)
    mbar_init8(s0 + 64 + 8 * (threadIdx.x - 32), 2 * k8GB);  // one arrival per (row, band) task of the pair
  if (threadIdx.x >= 64 && threadIdx.x < 64 + k8Ring)
    mbar_init8(s0 + 128 + 8 * (threadIdx.x - 64), k8VW);  // one arrival per vertical warp
  if (threadIdx.x < k8GB) {  // per-band SSIM constants for the horizontal warps
    const double pk = (int)threadIdx.x < nb ? args.peaks[a * C + g * k8GB + threadIdx.x] : 1.0;
    reinterpret_cast<float4 *>(smem + geo.off_desc)[threadIdx.x] =
        make_float4((float)pk, fmaxf((float)((0.01 * pk) * (0.01 * pk)), 1e-30f),
                    fmaxf((float)((0.03 * pk) * (0.03 * pk)), 1e-30f), 0.f);
  }
  if constexpr (PCA) {
    if (w == 2) {
      for (int i = lane; i < k8GB * k8PcaMax; i += 32) {
        const int bq = i / k8PcaMax, j = i % k8PcaMax;
        float cf = 0.f;
        if (bq < nb && j < E) {
          const double m = args.qmins[a * E + j];
          const double sp = __dsub_rn(args.qmaxs[a * E + j], m);
          cf = (float)((sp / L) * inv.W[j * kMaxC + g * k8GB + bq]);
        }
        reinterpret_cast<float *>(smem + geo.off_coef)[i] = cf;
      }
    }
  }
  if constexpr (MODE == K8_LUT) {
    // (hi, lo) float pair of the exact float64 dequantisation of every code
    for (int i = threadIdx.x; i < k8GB * k8LutMax; i += blockDim.x) {
      const int b = i / k8LutMax, q = i % k8LutMax;
      if (b < nb && q <= (int)args.Li) {
        const double m = args.qmins[a * C + g * k8GB + b];
        const double sp = __dsub_rn(args.qmaxs[a * C + g * k8GB + b], m);
        const double v = dequantize_fast((uint32_t)q, m, sp, L, args.rL);
        const float hi = (float)v;
        lut[i] = make_float2(hi, (float)(v - (double)hi));
      }
    }
  }
  // the input ring starts zeroed: bytes no copy ever writes (columns past the
  // frame edge) read as 0, so the decode needs no per-element masking
  for (int i = threadIdx.x; i < ns * geo.stage / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(smem + geo.off_in)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // zeros before the first bulk copies
  __syncthreads();
  double *red = reinterpret_cast<double *>(smem + geo.off_vb);  // end-of-kernel partials [32 warps][32]

  if (w >= k8VW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(k8RegsH));
    // ------------------------------------------------------------------ horizontal warpgroups
    const int h = w - k8VW;
    // a worker's tasks cycle through the bands: its four float64 sums live in shared memory
    double *hsl = reinterpret_cast<double *>(smem + geo.off_hs) + (size_t)(h * 32 + lane) * k8GB;
#pragma unroll
    for (int bq = 0; bq < k8GB; ++bq) hsl[bq] = 0.0;
    if (h == k8HWork) {
      // ---------------------------------------------------------------- loader warp
      // copy k of a pair (lane k): row k / ncp of the pair, piece k % ncp
      // (piece 0: the original's row segment, piece j+1: frame plane j)
      const int ncp = 1 + np;
      const int64_t rowb = W * C * 4;
      const int64_t xe = min(x0 + k8Cols, W);
      const int64_t oa0 = (x0 * C * 4) & ~15ll, oa1 = (xe * C * 4 + 15) & ~15ll;
      const int64_t fa0 = (x0 * FSZ) & ~15ll, fa1 = (xe * FSZ + 15) & ~15ll;
      const uint32_t obytes = (uint32_t)(oa1 - oa0), fbytes = (uint32_t)(fa1 - fa0);
      const char *src = nullptr;
      uint32_t dst = 0, bytes = 0;
      int64_t stride2 = 0;
      if (lane < 2 * ncp) {
        const int row_k = lane / ncp, piece = lane % ncp;
        if (piece == 0) {
          src = reinterpret_cast<const char *>(args.orig) + (a * T + t) * H * rowb + oa0 + row_k * rowb;
          dst = in_ring + row_k * geo.ob;
          bytes = obytes;
          stride2 = 2 * rowb;
        } else {
          const int j = PCA ? piece - 1 : g * k8GB + piece - 1;  // frame plane
          src = reinterpret_cast<const char *>(args.frames) +
                ((((a * args.G + j / 3) * T + t) * 3 + j % 3) * HW) * FSZ + fa0 + row_k * W * FSZ;
          dst = in_ring + 2 * geo.ob + ((piece - 1) * 2 + row_k) * geo.fb;
          bytes = fbytes;
          stride2 = 2 * W * FSZ;
        }
      }
      const uint32_t tx = obytes + (uint32_t)np * fbytes;
      int st = 0;
#pragma unroll 1
      for (int p = 0; p < npairs; ++p) {
        if (p >= ns) nbar_sync(k8BarStage + st, 32 * (k8VW + 1));  // parked until the 16 vertical warps released it
        const int rows = min(2, H32 - 2 * p);
        if (lane == 0) mbar_arrive_tx8(full_in + 8 * st, (uint32_t)rows * tx);
        __syncwarp();
        if (lane < rows * ncp) bulk_g2s8(dst + (uint32_t)st * geo.stage, src, bytes, full_in + 8 * st);
        src += stride2;
        if (++st == ns) st = 0;
      }
    } else {
      // ---------------------------------------------------------------- horizontal workers
      // task k = (filtered pair k / 8, row (k / 4) % 2, band k % 4); worker h takes h, h + 11, ...
      const int hlim = min(k8Out, W32 - kSsimTaps - (int)x0 + 1);  // valid output columns of the strip
      const bool hv_any = 4 * lane < hlim;
      constexpr uint32_t kVbPair = 2u * k8VbRow * 16u;
      const uint32_t cst = s0 + geo.off_desc;
      float hs4 = 0.f;
      const int ntask = nfe * 2 * k8GB;
#pragma unroll 1
      for (int k = h; k < ntask; k += k8HWork) {
        const int e = k >> 3, hsub = (k >> 2) & 1, bb = k & 3;
        const int slot = e % k8Ring;
        mbar_wait8(s0 + 128u + 8u * (uint32_t)slot, (uint32_t)((e / k8Ring) & 1));
        if (bb < nb && hv_any && 2 * e + hsub <= H32 - kSsimTaps) {
          const float4 cc = lds8_f32x4(cst + 16u * (uint32_t)bb);
          const uint32_t hv = vb + 16u * (uint32_t)(vb8_skew(bb) + lane) + (uint32_t)slot * kVbPair +
                              (uint32_t)hsub * (k8VbRow * 16u);
          float2 asd[4], aq[4];
          // loads run kHPf columns ahead of the filter (the chain is otherwise bound
          // by one shared-memory latency per column)
          constexpr int kHPf = 3;
          float4 pf[kHPf];
#pragma unroll
          for (int kk = 0; kk < kHPf; ++kk) pf[kk] = lds8_f32x4(hv + 16u * (uint32_t)((kk & 3) * 34 + (kk >> 2)));
#pragma unroll
          for (int kk = 0; kk < 14; ++kk) {
            const float4 v = pf[kk % kHPf];
            if (kk + kHPf < 14)
              pf[kk % kHPf] = lds8_f32x4(hv + 16u * (uint32_t)(((kk + kHPf) & 3) * 34 + ((kk + kHPf) >> 2)));
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
          float ts = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float s1 = ssim_px(asd[i].x, asd[i].y, aq[i].x, aq[i].y, cc.x, cc.y, cc.z);
            ts += 4 * lane + i < hlim ? s1 : 0.f;
          }
          hs4 += ts;
        }
        if (e + k8Ring < nfe) {  // the slot will be refilled: one arrival per task, by lane 0 after the warp's reads
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(s0 + 64u + 8u * (uint32_t)slot) : "memory");
        }
        hsl[bb] += (double)hs4;
        hs4 = 0.f;
      }
    }
    __syncthreads();  // the ring is idle
    __syncthreads();  // all partials written
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(k8RegsV));

  // ------------------------------------------------------------------ vertical warps
  const int b = lane & 3, cl = lane >> 2;
  const int lc = 8 * w + cl;  // local input column
  const int c = g * k8GB + b;
  const bool bact = b < nb;
  const int xv = (int)x0 + lc;
  const bool own = bact && xv < W32 && (lc < k8Out || last_strip);
  const float c0 = bact ? (float)args.peaks[a * C + c] : 1.f;

  // decode constants
  double dq_m = 0.0, dq_span = 0.0;
  float base = 0.f;
  if constexpr (MODE == K8_F64) {
    if (bact) {
      dq_m = args.qmins[a * C + c];
      dq_span = __dsub_rn(args.qmaxs[a * C + c], dq_m);
    }
  }
  if constexpr (PCA) {
    // recon_c = mean_c + sum_j (min_j + q_j span_j / L) W[j][c]
    //         = base_c + sum_j q_j coef_cj   (float32; |error| << one code step);
    // the coefficients live in shared memory (table written before the first barrier)
    double bd = inv.mean[bact ? c : 0];
#pragma unroll
    for (int j = 0; j < EP; ++j)
      if ((EXACT || j < E) && bact) bd = __fma_rn(args.qmins[a * E + j], inv.W[j * kMaxC + c], bd);
    base = (float)bd;
  }
  const uint32_t coef_b = opaque8(s0 + geo.off_coef + (uint32_t)(b * k8PcaMax * 4));

  // per-lane shared-memory byte offsets inside a stage. Lanes of an absent
  // band (b >= nb) read the neighbouring band's finite values, lanes past the
  // frame edge read zeros: neither reaches a counted output, so only the
  // squared error and the recon store are masked.
  const uint32_t o_off = opaque8(in_ring + (uint32_t)((x0 * C * 4) & 15) + (uint32_t)(lc * C + min(c, C - 1)) * 4u);
  const uint32_t f_off = opaque8(in_ring + 2u * geo.ob + (uint32_t)((PCA ? 0 : 2 * min(b, nb - 1)) * geo.fb) +
                                 (uint32_t)((x0 * FSZ) & 15) + (uint32_t)(lc * FSZ));
  const uint32_t ob = opaque8(geo.ob), fb = opaque8(geo.fb), stage_b = opaque8(geo.stage);
  const uint32_t lut_b = opaque8(s0 + geo.off_lut + (uint32_t)(b * k8LutMax * 8));
  const uint32_t bars = opaque8(s0);  // full_in at +8*stage, empty_in at +8*(NS+stage)
  uint32_t qor = 0;
  float sse_f = 0.f;
  double sse = 0.0;
  const bool wr = args.recon_out != nullptr && own;
  // recon stores: frame base (uniform) + 32-bit element offset inside the frame
  float *const rbase = args.recon_out + (a * T + t) * HW * C;
  uint32_t woff = (uint32_t)(xv * C + c);
  const uint32_t rstride = (uint32_t)(W32 * C);  // recon row stride (floats); H W C < 2^31

  Fir8 fir;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    fir.zsd[i] = make_float2(0.f, 0.f);
    fir.zq[i] = make_float2(0.f, 0.f);
  }

  constexpr uint32_t kVbPair = 2u * k8VbRow * 16u;  // bytes of one ring slot (row pair)
  const uint32_t vb_st = opaque8(vb + 16u * (uint32_t)(vb8_skew(b) + vb8_idx(lc)));

  int in_st = 0;          // input ring stage of the next pair
  uint32_t in_off = 0;    // its byte offset
  uint32_t in_ph = 0;     // parity of its "copies landed" completion
  int vs_slot = 0;        // ring slot of the next filtered pair
  uint32_t vs_off = 0;    // its byte offset
  uint32_t dr_par = 1;    // parity of the slot's "drained" completion (first reuse waits for phase 0)
  // one row pair; UU = pair index mod 5 (the FIR slots of its rows are 2 UU, 2 UU + 1)
  // FIRST: pairs 0 .. 4, whose filtered rows do not exist yet (no ring writes)
  // SR ("static rings"): with ns == 5 input stages and the 5-slot filtered ring, pair p = 5 gi + UU
  // uses stage UU and slot UU, and every phase parity is gi & 1: the ring bookkeeping (about 20
  // uniform-datapath instructions per pair) folds into immediates.
  auto pair_step = [&](auto uu, auto first, auto srt, const int p, const int gi) {
    constexpr int UU = decltype(uu)::value;
    constexpr bool FIRST = decltype(first)::value != 0;
    constexpr bool SR = decltype(srt)::value != 0;
    int U;
    uint32_t st;
    if constexpr (SR) {
      U = UU;
      st = (uint32_t)UU * stage_b;
      mbar_wait8(bars + 8 * UU, (uint32_t)(gi & 1));
    } else {
      U = in_st;
      st = in_off;
      mbar_wait8(bars + 8 * U, in_ph);
      in_off += stage_b;
      if (++in_st == ns) {
        in_st = 0;
        in_off = 0;
        in_ph ^= 1u;
      }
    }
    const bool rel = p + ns < npairs;  // the loader refills this stage: tell it when the reads are done
    // raw inputs of the pair: original values and codes
    float2 om;
    om.x = lds8_f32(st + o_off);
    om.y = lds8_f32(st + ob + o_off);
    float2 rv, df;
    if constexpr (PCA) {
      uint32_t q0[EPL], q1[EPL];
#pragma unroll
      for (int j = 0; j < EP; ++j)
        if (EXACT || j < E) {
          q0[j] = lds8_code<FSZ>(st + f_off + (uint32_t)(2 * j) * fb);
          q1[j] = lds8_code<FSZ>(st + f_off + (uint32_t)(2 * j + 1) * fb);
        }
      if (rel) nbar_arrive(k8BarStage + U, 32 * (k8VW + 1));
      // both rows at once: acc = base + sum_j q_j coef_j (packed FFMA2)
      float2 acc = make_float2(base, base);
#pragma unroll
      for (int j = 0; j < EP; j += 2) {
        const float2 cf = lds8_f32x2(coef_b + 4u * (uint32_t)j);
        if (EXACT || j < E) {
          if (CHKQ) qor |= q0[j] | q1[j];
          acc = __ffma2_rn(make_float2((float)q0[j], (float)q1[j]), make_float2(cf.x, cf.x), acc);
        }
        if (j + 1 < EP && (EXACT || j + 1 < E)) {
          if (CHKQ) qor |= q0[j + 1] | q1[j + 1];
          acc = __ffma2_rn(make_float2((float)q0[j + 1], (float)q1[j + 1]), make_float2(cf.y, cf.y), acc);
        }
      }
      rv = acc;
    } else {
      const uint32_t q0 = lds8_code<FSZ>(st + f_off), q1 = lds8_code<FSZ>(st + f_off + fb);
      qor |= q0 | q1;
      if constexpr (MODE == K8_LUT) {
        const float2 l0 = lds8_f32x2(lut_b + 8u * min(q0, (uint32_t)(k8LutMax - 1)));
        const float2 l1 = lds8_f32x2(lut_b + 8u * min(q1, (uint32_t)(k8LutMax - 1)));
        if (rel) nbar_arrive(k8BarStage + U, 32 * (k8VW + 1));
        rv = make_float2(l0.x, l1.x);
        df = make_float2(l0.y, l1.y);  // the low halves; subtracted from (o - hi) below
      } else {
        if (rel) nbar_arrive(k8BarStage + U, 32 * (k8VW + 1));
        const double rm0 = dequantize_fast(q0, dq_m, dq_span, L, args.rL);
        const double rm1 = dequantize_fast(q1, dq_m, dq_span, L, args.rL);
        rv = make_float2((float)rm0, (float)rm1);
        df = make_float2((float)__dsub_rn((double)om.x, rm0), (float)__dsub_rn((double)om.y, rm1));
      }
    }
    const bool ok1 = 2 * p + 1 < H32;  // odd H: the last pair's second row does not exist
    if (wr) {  // the four bands of a pixel sit in adjacent lanes: 16-byte runs per pixel
      rbase[woff] = rv.x;
      if (ok1) rbase[woff + rstride] = rv.y;
    }
    woff += 2u * rstride;
    // FIR inputs (s, d) = (x' + y', x - y) per row
    float2 p0, p1;
    if constexpr (PCA) {
      // straight into (s, d) pairs from the row-packed decode, with broadcast
      // operands: (o - 2 c0, o) + r (1, -1); no repacking moves
      const float2 kpm = make_float2(1.f, -1.f), kc = make_float2(-2.f * c0, 0.f);
      p0 = __ffma2_rn(make_float2(rv.x, rv.x), kpm, __fadd2_rn(make_float2(om.x, om.x), kc));
      p1 = __ffma2_rn(make_float2(rv.y, rv.y), kpm, __fadd2_rn(make_float2(om.y, om.y), kc));
      df = make_float2(p0.y, p1.y);
    } else if constexpr (MODE == K8_LUT) {
      // same pairs from the (hi, lo) table entries: d = (o - hi) - lo
      const float2 kpm = make_float2(1.f, -1.f), kc = make_float2(-2.f * c0, 0.f);
      p0 = __ffma2_rn(make_float2(rv.x, rv.x), kpm, __fadd2_rn(make_float2(om.x, om.x), kc));
      p1 = __ffma2_rn(make_float2(rv.y, rv.y), kpm, __fadd2_rn(make_float2(om.y, om.y), kc));
      // d -= lo as a packed fma (lo * (0, -1) + p): the pair stays one FFMA2 result
      const float2 k0m = make_float2(0.f, -1.f);
      p0 = __ffma2_rn(make_float2(df.x, df.x), k0m, p0);
      p1 = __ffma2_rn(make_float2(df.y, df.y), k0m, p1);
      df = make_float2(p0.y, p1.y);
    } else {
      p0 = make_float2(__fadd_rn(__fadd_rn(om.x, rv.x), -2.f * c0), df.x);
      p1 = make_float2(__fadd_rn(__fadd_rn(om.y, rv.y), -2.f * c0), df.y);
    }
    const float d0 = own ? df.x : 0.f, d1 = (own && ok1) ? df.y : 0.f;
    sse_f = fmaf(d1, d1, fmaf(d0, d0, sse_f));
    const float4 o0 = fir8_step<2 * UU>(fir, p0);
    const float4 o1 = fir8_step<2 * UU + 1>(fir, p1);
    if constexpr (!FIRST && SR) {  // column-filtered pair p - 5 = 5 (gi - 1) + UU: slot UU, reuse gi - 1
      if (gi >= 2) mbar_wait8(bars + 64u + 8u * UU, (uint32_t)(gi & 1));
      const uint32_t d = vb_st + (uint32_t)UU * kVbPair;
      sts8_f32x4(d, o0);
      sts8_f32x4(d + k8VbRow * 16u, o1);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bars + 128u + 8u * UU) : "memory");
    } else if constexpr (!FIRST) {  // column-filtered rows 2p-10, 2p-9 = pair p-5
      if (p - 5 >= k8Ring) mbar_wait8(bars + 64u + 8u * (uint32_t)vs_slot, dr_par);
      const uint32_t d = vb_st + vs_off;
      sts8_f32x4(d, o0);
      sts8_f32x4(d + k8VbRow * 16u, o1);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bars + 128u + 8u * (uint32_t)vs_slot) : "memory");
      vs_off += kVbPair;
      if (++vs_slot == k8Ring) {
        vs_slot = 0;
        vs_off = 0;
        dr_par ^= 1u;
      }
    }
  };
  // Straight-line groups of five pairs (ten rows = one turn of the FIR slots; no
  // branch between the steps, so the 40 state registers keep their places):
  // group 0 without ring writes, whole groups, then the npairs % 5 tail.
  // H >= 11 rows, so there are at least six pairs.
  auto flush_sse = [&]() {
    sse += (double)sse_f;  // ten squared differences per float32 partial
    sse_f = 0.f;
  };
  auto run_all = [&](auto srt) {
    pair_step(PairIdx8<0>{}, PairIdx8<1>{}, srt, 0, 0);
    pair_step(PairIdx8<1>{}, PairIdx8<1>{}, srt, 1, 0);
    pair_step(PairIdx8<2>{}, PairIdx8<1>{}, srt, 2, 0);
    pair_step(PairIdx8<3>{}, PairIdx8<1>{}, srt, 3, 0);
    pair_step(PairIdx8<4>{}, PairIdx8<1>{}, srt, 4, 0);
    flush_sse();
    const int ngroups = npairs / 5;
#pragma unroll 1
    for (int gi = 1; gi < ngroups; ++gi) {
      const int p0 = 5 * gi;
      pair_step(PairIdx8<0>{}, PairIdx8<0>{}, srt, p0, gi);
      pair_step(PairIdx8<1>{}, PairIdx8<0>{}, srt, p0 + 1, gi);
      pair_step(PairIdx8<2>{}, PairIdx8<0>{}, srt, p0 + 2, gi);
      pair_step(PairIdx8<3>{}, PairIdx8<0>{}, srt, p0 + 3, gi);
      pair_step(PairIdx8<4>{}, PairIdx8<0>{}, srt, p0 + 4, gi);
      flush_sse();
    }
    {
      const int p0 = 5 * ngroups, rem = npairs - p0;
      if (rem > 0) pair_step(PairIdx8<0>{}, PairIdx8<0>{}, srt, p0, ngroups);
      if (rem > 1) pair_step(PairIdx8<1>{}, PairIdx8<0>{}, srt, p0 + 1, ngroups);
      if (rem > 2) pair_step(PairIdx8<2>{}, PairIdx8<0>{}, srt, p0 + 2, ngroups);
      if (rem > 3) pair_step(PairIdx8<3>{}, PairIdx8<0>{}, srt, p0 + 3, ngroups);
      flush_sse();
    }
  };
  if (ns == k8Ring) run_all(PairIdx8<1>{});  // five input stages: static rings
  else run_all(PairIdx8<0>{});
  flag_warp(args.err, (qor & ~args.Li) != 0u, CV_FLAG_INT_RANGE);

  // deterministic CTA reduction: per band, fixed order over warps and lanes
  __syncthreads();  // the ring is idle
  red[w * 32 + lane] = sse;
  __syncthreads();  // all partials written
  if (threadIdx.x < nb) {
    const int bq = threadIdx.x;
    double s1 = 0.0, s2 = 0.0;
    for (int ww = 0; ww < k8VW; ++ww)
      for (int l = bq; l < 32; l += 4) s1 += red[ww * 32 + l];
    const double *hs = reinterpret_cast<const double *>(smem + geo.off_hs);
    for (int i = 0; i < k8HW * 32; ++i) s2 += hs[i * k8GB + bq];
    double *pp = args.part + ((a * T + t) * args.nstrips + strip) * 2 * C;
    pp[g * k8GB + bq] = s1;
    pp[C + g * k8GB + bq] = s2;
  }
}

}  // namespace cvb
