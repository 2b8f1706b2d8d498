// K4 planar quantiser (the encode-prep kernel of the benchmark).
//
// A CTA owns P = blockDim.x pixels of one cube for one time segment. Each time
// step's source chunk (P*C contiguous elements) streams through a 4-stage
// cp.async ring in shared memory (16-byte copies, 3 steps ahead). Per step:
//   1. every thread forward-fills the vectors it copied (carries stay in
//      registers: the thread <-> element ownership is fixed across steps),
//      writes them back in place and to the filled cube (16-byte stores);
//   2. barrier; thread p takes pixel p: reads its C values from shared memory,
//      (projects them onto the PCA components), quantises each band with the
//      float32 fast path / exact float64 fallback, and writes its sample of
//      every plane of the planar frames (coalesced across the warp).
#pragma once
#include "common.cuh"
#include "pca_params.cuh"

namespace cvb {

#ifndef CVB_QSTAGES
#define CVB_QSTAGES 4
#endif
constexpr int kQStages = CVB_QSTAGES;

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit_q() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_q() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// PX2 (non-PCA, C <= kQRegC, even H*W): thread p takes the pixel pair 2p,
// 2p+1, keeps every band's float32 quantiser constants in registers and
// stores both samples of a plane with one 32-bit (u16) / 16-bit (u8) store.
constexpr int kQRegC = 8;
constexpr int kQPcaC = 16;  // PCA register path: channels and components
// C = 12 PCA path: float64 tables in shared memory behind the band constants:
// weights [12][12], means [12], K = L / span [12]
constexpr int kQP12 = 12;
constexpr int kQP12Tab = (kQP12 * kQP12 + 2 * kQP12) * 8;

__device__ __forceinline__ double lds_f64_q(uint32_t a) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}

// C = 12 PCA path, quantize (transform.py:98-105) of a float64 component. Fast path: one
// fma, t = (v - m) K + 0.5 with K = RN(L / span); it differs from the reference's
// RN(RN(RN(v - m) / span) L) + 0.5 by less than 4 L 2^-53 < 4e-11, so whenever frac(t) is
// more than 2^-28 away from an integer both floors agree; otherwise the reference's own
// operation order decides (one branch per group of six values). A constant band has span 1
// and v = m: t = 0.5, code 0. Clamped streams take the generic kernel; out-of-range / NaN
// values set the RANGE flag (transform.py:92-97 raises).

// EE: compile-time component count of the C = 12 PCA path (6 / 9; 0 = runtime): the plane
// guards and pad selects (52 SEL + 68 IMAD.MOV of 731 instructions per pixel pair) fold away.
template <typename TIn, typename TOut, bool FILL, bool PCA, int MAXV, bool PX2 = false, int CX = 0, int EE = 0>
__global__ void __launch_bounds__(256)
k_quantize_planar(const TIn *__restrict__ src, TOut *__restrict__ out, const QuantArgs args,
                  const PcaParams pca) {
  constexpr int VE = 16 / sizeof(TIn);  // elements per 16-byte copy
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = blockDim.x, tid = threadIdx.x;
  const int C = CX ? CX : args.C, E = EE ? EE : args.E;  // CX: compile-time band count (PCA, C = 12)
  const int GG = EE ? (EE + 2) / 3 : (CX && !PCA) ? (CX + 2) / 3 : args.G;  // videos of the stream
  const int64_t T = args.T, HW = args.HW, inner = HW * C;
  const int P = PX2 ? 2 * NT : NT;          // pixels per chunk
  const int NE = P * C;                     // elements per full chunk
  const int64_t a = blockIdx.z, seg = blockIdx.y, nseg = gridDim.y;
  const int64_t pix0 = (int64_t)blockIdx.x * P;
  const int64_t e0 = pix0 * C;
  const int npix = (int)min((int64_t)P, HW - pix0);
  const int ne = npix * C;
  const int nvec = (ne + VE - 1) / VE;      // whole row end is vector aligned (host check)
  const int64_t t0 = seg * args.seg_len;
  const int64_t t1 = min(T, t0 + (int64_t)args.seg_len);
  const TIn *cube = src + a * T * inner;
  TIn *stage = reinterpret_cast<TIn *>(smem);  // [kQStages][NE + pad]
  const int SP = (NE + VE - 1) / VE * VE;       // stage pitch (elements)
  QBand *qtab = reinterpret_cast<QBand *>(smem + (size_t)kQStages * SP * sizeof(TIn));
  QBand32 *qtab32 = reinterpret_cast<QBand32 *>(qtab + kMaxC);
  for (int j = tid; j < E; j += NT) {
    qtab[j] = make_qband(args.mins[a * E + j], args.maxs[a * E + j], args.bit_depth);
    qtab32[j] = make_qband32(qtab[j], args.clamp);
  }
  double *wsm = reinterpret_cast<double *>(qtab32 + kMaxC);  // [12][12] weights, [12] means, [12] K
  if constexpr (PX2 && PCA && CX == kQP12) {
    for (int i = tid; i < kQP12 * kQP12; i += NT) wsm[i] = i < E * kQP12 ? pca.W[(i / kQP12) * kMaxC + i % kQP12] : 0.0;
    if (tid < kQP12) wsm[kQP12 * kQP12 + tid] = pca.mean[tid];
    for (int j = tid; j < E; j += NT) wsm[kQP12 * kQP12 + kQP12 + j] = __ddiv_rn(qtab[j].L, qtab[j].s);
  }
  __syncthreads();

  // vectors owned by this thread: v = tid + i*NT (fixed across steps), at most
  // MAXV = ceil(C / VE) (host-selected bound)
  const int nv_mine = nvec > tid ? (nvec - tid + NT - 1) / NT : 0;

  float carry[FILL ? MAXV * 4 : 1];
  if constexpr (FILL) {
    const float *sl = args.seg_last + a * nseg * inner;
    const float *ci = args.carry_in ? args.carry_in + a * inner : nullptr;
#pragma unroll
    for (int i = 0; i < MAXV; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int el = (tid + i * NT) * 4 + j;
        carry[i * 4 + j] = (i < nv_mine && el < ne) ? segment_carry(sl, seg, inner, e0 + el, ci, args.fill) : args.fill;
      }
  }

  auto issue = [&](int64_t t) {
    TIn *st = stage + (size_t)(t % kQStages) * SP;
    const TIn *row = cube + t * inner + e0;
    for (int i = 0; i < nv_mine; ++i) {
      const int v = tid + i * NT;
      cp_async16(st + v * VE, row + (int64_t)v * VE);
    }
  };
#pragma unroll
  for (int s = 0; s < kQStages - 1; ++s) {
    if (t0 + s < t1) issue(t0 + s);
    cp_async_commit_q();
  }

  // per-pixel constants
  const int p = PX2 ? 2 * tid : tid;
  const bool pvalid = p < npix;
  bool bad = false, nanbad = false;
  TOut *obase = out + (a * args.G * T) * 3 * HW + pix0 + p;
  QBand32 rb[PX2 ? kQRegC : 1];
  const int64_t gjump = (3 * T - 2) * HW;  // plane 2 of video g -> plane 0 of video g+1
  if constexpr (PX2) obase += t0 * 3 * HW;
  if constexpr (PX2 && !PCA) {
#pragma unroll
    for (int c = 0; c < kQRegC; ++c) rb[c] = qtab32[c < C ? c : 0];  // C is static with CX (7: minicubes, 4: RGB+NIR)
  }

  for (int64_t t = t0; t < t1; ++t) {
    cp_async_wait_q<kQStages - 2>();
    TIn *st = stage + (size_t)(t % kQStages) * SP;
    if constexpr (FILL) {
      // forward fill of the owned vectors, in place, + the filled cube
      float *fo = args.filled_out ? args.filled_out + (a * T + t) * inner + e0 : nullptr;
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        if (i < nv_mine) {
          const int v = tid + i * NT;
          float4 x = *reinterpret_cast<float4 *>(st + v * 4);
          float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (isnan(xv[j])) xv[j] = carry[i * 4 + j];
            else carry[i * 4 + j] = xv[j];
          }
          x = make_float4(xv[0], xv[1], xv[2], xv[3]);
          *reinterpret_cast<float4 *>(st + v * 4) = x;
          if (fo) *reinterpret_cast<float4 *>(fo + v * 4) = x;
        }
      }
    }
    __syncthreads();
    // refill the stage consumed one step ago (every thread is past it now)
    if (t + kQStages - 1 < t1) issue(t + kQStages - 1);
    cp_async_commit_q();
    if constexpr (PX2 && PCA && CX == kQP12) {
      if (pvalid) {
        // C = 12 pixel pair: weights / means / per-component constants through
        // broadcast LDS.64 (one load serves both pixels; as kernel parameters the
        // 72 weights overflow the uniform registers and spill), one fma per code
        const TIn *px = st + p * kQP12;
        TOut *op = obase + (t - t0) * 3 * HW;
        using W2 = typename std::conditional<sizeof(TOut) == 1, uint16_t, uint32_t>::type;
        const uint32_t wb = (uint32_t)__cvta_generic_to_shared(wsm);
        const uint32_t qb = (uint32_t)__cvta_generic_to_shared(qtab);
        double d0[kQP12], d1[kQP12];
        if constexpr (std::is_same<TIn, float>::value) {
          // the pair's 24 floats as six 16-byte loads (p is even: 96-byte aligned)
          float xv[2 * kQP12];
#pragma unroll
          for (int q4 = 0; q4 < 2 * kQP12 / 4; ++q4) {
            const float4 v4 = *reinterpret_cast<const float4 *>(px + 4 * q4);
            xv[4 * q4] = v4.x, xv[4 * q4 + 1] = v4.y, xv[4 * q4 + 2] = v4.z, xv[4 * q4 + 3] = v4.w;
          }
#pragma unroll
          for (int c = 0; c < kQP12; ++c) {
            const double mu = lds_f64_q(wb + 8u * (kQP12 * kQP12 + c));
            d0[c] = __dsub_rn((double)xv[c], mu);
            d1[c] = __dsub_rn((double)xv[kQP12 + c], mu);
          }
        } else {
#pragma unroll
          for (int c = 0; c < kQP12; ++c) {
            const double mu = lds_f64_q(wb + 8u * (kQP12 * kQP12 + c));
            d0[c] = __dsub_rn((double)px[c], mu);
            d1[c] = __dsub_rn((double)px[kQP12 + c], mu);
          }
        }
        uint32_t l0 = 0, l1 = 0, badi = 0;
#pragma unroll
        for (int g = 0; g < kQP12 / 3; ++g) {
          if (g < GG) {
            // the three components of a video together: six independent fma chains
            double a0[3] = {0.0, 0.0, 0.0}, a1[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int c = 0; c < kQP12; ++c) {
#pragma unroll
              for (int jp = 0; jp < 3; ++jp) {
                const double w = lds_f64_q(wb + 8u * (uint32_t)((3 * g + jp) * kQP12 + c));
                a0[jp] = __fma_rn(d0[c], w, a0[jp]);
                a1[jp] = __fma_rn(d1[c], w, a1[jp]);
              }
            }
            // fast codes of the group's six values; ONE rare branch recomputes the group in the
            // reference's operation order when any of them is within 2^-28 of a rounding tie
            uint32_t qq0[3], qq1[3];
            bool near = false;
            const double eps = 3.725290298461914e-09;  // 2^-28
#pragma unroll
            for (int jp = 0; jp < 3; ++jp) {
              const int pl = 3 * g + jp;
              qq0[jp] = qq1[jp] = 0u;
              if (pl < E) {
                const uint32_t bq = qb + (uint32_t)(pl * sizeof(QBand));
                const double bm = lds_f64_q(bq), bM = lds_f64_q(bq + 8);
                const double bK = lds_f64_q(wb + 8u * (uint32_t)(kQP12 * kQP12 + kQP12 + pl));
                if (!(a0[jp] >= bm && a0[jp] <= bM)) badi = 1u;
                if (!(a1[jp] >= bm && a1[jp] <= bM)) badi = 1u;
                const double t0 = __fma_rn(__dsub_rn(a0[jp], bm), bK, 0.5), t1 = __fma_rn(__dsub_rn(a1[jp], bm), bK, 0.5);
                const double f0 = floor(t0), f1 = floor(t1);
                const double r0 = __dsub_rn(t0, f0), r1 = __dsub_rn(t1, f1);
                near |= (r0 < eps) | (r0 > 1.0 - eps) | (r1 < eps) | (r1 > 1.0 - eps);
                qq0[jp] = min((uint32_t)f0, 65535u);
                qq1[jp] = min((uint32_t)f1, 65535u);
              }
            }
            if (near) {
#pragma unroll
              for (int jp = 0; jp < 3; ++jp) {
                const int pl = 3 * g + jp;
                if (pl < E) {
                  const uint32_t bq = qb + (uint32_t)(pl * sizeof(QBand));
                  const double bm = lds_f64_q(bq), bs = lds_f64_q(bq + 16), bL = lds_f64_q(bq + 32);
                  const double x0 = __dmul_rn(__ddiv_rn(__dsub_rn(a0[jp], bm), bs), bL);
                  const double x1 = __dmul_rn(__ddiv_rn(__dsub_rn(a1[jp], bm), bs), bL);
                  qq0[jp] = min((uint32_t)floor(__dadd_rn(x0, 0.5)), 65535u);
                  qq1[jp] = min((uint32_t)floor(__dadd_rn(x1, 0.5)), 65535u);
                }
              }
            }
#pragma unroll
            for (int jp = 0; jp < 3; ++jp) {
              const int pl = 3 * g + jp;
              uint32_t q0, q1;
              if (pl < E) {
                q0 = qq0[jp];
                q1 = qq1[jp];
                l0 = q0;
                l1 = q1;
              } else {
                const bool rep = args.pad_mode == CV_PAD_REPEAT;
                q0 = rep ? l0 : 0u;
                q1 = rep ? l1 : 0u;
              }
              *reinterpret_cast<W2 *>(op) = (W2)(q0 | (q1 << (8 * sizeof(TOut))));
              op += jp == 2 ? gjump : HW;
            }
          }
        }
        bad |= badi != 0u;
      }
    } else if (PX2 && PCA && pvalid) {
      // PCA pixel pair (p, p+1): both projections in registers (two independent
      // float64 chains), one 32-bit / 16-bit store per component plane
      const TIn *px = st + p * C;
      TOut *op = obase + (t - t0) * 3 * HW;
      using W2 = typename std::conditional<sizeof(TOut) == 1, uint16_t, uint32_t>::type;
      double d0[kQPcaC], d1[kQPcaC];
#pragma unroll
      for (int c = 0; c < kQPcaC; ++c) {
        d0[c] = c < C ? __dsub_rn((double)px[c], pca.mean[c]) : 0.0;
        d1[c] = c < C ? __dsub_rn((double)px[C + c], pca.mean[c]) : 0.0;
      }
      uint32_t l0 = 0, l1 = 0;
#pragma unroll
      for (int pl = 0; pl < 3 * ((kQPcaC + 2) / 3); ++pl) {
        if (pl < 3 * args.G) {
          uint32_t q0, q1;
          if (pl < E) {
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int c = 0; c < kQPcaC; ++c)
              if (c < C) {
                a0 = __fma_rn(d0[c], pca.W[pl * kMaxC + c], a0);
                a1 = __fma_rn(d1[c], pca.W[pl * kMaxC + c], a1);
              }
            const QBand b = qtab[pl];
            q0 = quantize_value(range_prep(a0, b, args.clamp, bad), b);
            q1 = quantize_value(range_prep(a1, b, args.clamp, bad), b);
            l0 = q0;
            l1 = q1;
          } else {
            const bool rep = args.pad_mode == CV_PAD_REPEAT;
            q0 = rep ? l0 : 0u;
            q1 = rep ? l1 : 0u;
          }
          *reinterpret_cast<W2 *>(op) = (W2)(q0 | (q1 << (8 * sizeof(TOut))));
          op += (pl % 3 == 2) ? gjump : HW;
        }
      }
    } else if (PX2 && !PCA && pvalid) {
      // pixel pair (p, p+1); npix and p are even
      const TIn *px = st + p * C;
      TOut *op = obase + (t - t0) * 3 * HW;  // plane 0 of video 0 at time t
      using W2 = typename std::conditional<sizeof(TOut) == 1, uint16_t, uint32_t>::type;
      uint32_t l0 = 0, l1 = 0;
#pragma unroll
      for (int pl = 0; pl < 3 * ((kQRegC + 2) / 3); ++pl) {
        if (pl < 3 * GG) {
          const int c = pl;
          uint32_t q0, q1;
          if (c < C) {
            const float v0 = (float)px[c], v1 = (float)px[C + c];
            if constexpr (!FILL) nanbad |= (v0 != v0) | (v1 != v1);
            const QBand32 b32 = rb[c];
            const bool f0 = b32.use32 && quantize_fast32(v0, b32, q0, bad);
            const bool f1 = b32.use32 && quantize_fast32(v1, b32, q1, bad);
            if (!(f0 && f1)) {
              const QBand b = qtab[c];
              if (!f0) q0 = quantize_value(range_prep((double)v0, b, args.clamp, bad), b);
              if (!f1) q1 = quantize_value(range_prep((double)v1, b, args.clamp, bad), b);
            }
            l0 = q0;
            l1 = q1;
          } else {
            const bool rep = args.pad_mode == CV_PAD_REPEAT;
            q0 = rep ? l0 : 0u;
            q1 = rep ? l1 : 0u;
          }
          *reinterpret_cast<W2 *>(op) = (W2)(q0 | (q1 << (8 * sizeof(TOut))));
          op += (pl % 3 == 2) ? gjump : HW;  // next plane / next video
        }
      }
    } else if (!PX2 && pvalid) {
      const TIn *px = st + p * C;
      TOut *o = obase + t * 3 * HW;
      if constexpr (!PCA) {
        uint32_t last = 0;
        const int64_t gstride = 3 * T * HW;  // next video (group of three planes)
        for (int g = 0; g < args.G; ++g) {
#pragma unroll
          for (int jp = 0; jp < 3; ++jp) {
            const int c = 3 * g + jp;
            uint32_t q;
            if (c < C) {
              const float v = (float)px[c];
              if constexpr (!FILL) nanbad |= (v != v);
              const QBand32 b32 = qtab32[c];
              if (!(b32.use32 && quantize_fast32(v, b32, q, bad))) {
                const QBand b = qtab[c];
                const double d = range_prep((double)v, b, args.clamp, bad);
                q = quantize_value(d, b);
              }
              last = q;
            } else {
              q = args.pad_mode == CV_PAD_REPEAT ? last : 0u;
            }
            o[jp * HW] = (TOut)q;
          }
          o += gstride;
        }
      } else if (C <= kQPcaC && E <= kQPcaC) {
        // registers only: C differences, K components with constant-bank
        // weights (static indices), incremental plane pointer
        double d[kQPcaC];
#pragma unroll
        for (int c = 0; c < kQPcaC; ++c) d[c] = c < C ? __dsub_rn((double)px[c], pca.mean[c]) : 0.0;
        uint32_t last = 0;
        TOut *op = o;
#pragma unroll
        for (int pl = 0; pl < 3 * ((kQPcaC + 2) / 3); ++pl) {
          if (pl < 3 * args.G) {
            uint32_t q;
            if (pl < E) {
              double pc = 0.0;
#pragma unroll
              for (int c = 0; c < kQPcaC; ++c)
                if (c < C) pc = __fma_rn(d[c], pca.W[pl * kMaxC + c], pc);
              const QBand b = qtab[pl];
              q = quantize_value(range_prep(pc, b, args.clamp, bad), b);
              last = q;
            } else {
              q = args.pad_mode == CV_PAD_REPEAT ? last : 0u;
            }
            *op = (TOut)q;
            op += (pl % 3 == 2) ? gjump : HW;
          }
        }
      } else {
        double d[kMaxC];
#pragma unroll
        for (int c = 0; c < kMaxC; ++c)
          if (c < C) d[c] = __dsub_rn((double)px[c], pca.mean[c]);
        uint32_t last = 0;
        const int64_t gstride = 3 * T * HW;
        for (int g = 0; g < args.G; ++g) {
#pragma unroll
          for (int jp = 0; jp < 3; ++jp) {
            const int j = 3 * g + jp;
            uint32_t q;
            if (j < E) {
              const double pc = project_one(d, pca, j);
              const QBand b = qtab[j];
              const double dv = range_prep(pc, b, args.clamp, bad);
              q = quantize_value(dv, b);
              last = q;
            } else {
              q = args.pad_mode == CV_PAD_REPEAT ? last : 0u;
            }
            o[jp * HW] = (TOut)q;
          }
          o += gstride;
        }
      }
    }
  }
  cp_async_wait_q<0>();
  flag_warp(args.err, bad, CV_FLAG_RANGE);
  flag_warp(args.err, nanbad, CV_FLAG_NAN);
}

}  // namespace cvb
