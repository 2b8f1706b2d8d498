// Shared device helpers for the cvb200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#include "cvb200.h"

namespace cvb {

// ----------------------------------------------------------------- errors
void set_last_error(const std::string &msg);
int fail(int status, const char *fmt, ...);
int check_launch(const char *what);

// Kernel-variant selection for A/B measurements and tests (cv_set_variant);
// plain ints read by the launchers, never the environment.
struct Variants {
  int gram_tiles = 0;    // 1: tiled k_gram instead of the pixel-per-lane k_gram_px
  int gram_nt = 64;      // k_gram_px CTA size: 64 or 256
  int proj_nopf = 0;     // 1: no next-pixel prefetch in k_pca_project_px (C = 12)
  int proj12 = 1;        // 0: k_pca_project_px instead of k_pca_project12 (float32, C = 12, K in {6, 9})
  int gram12 = 1;        // 0: k_gram_px instead of k_gram12 (float32, C = 12)
  int gram_checks = 0;   // 1: per-element finite tests in k_gram_px (else NaN / inf are read off the sums)
  int qp_px1 = 0;        // 1: one pixel per thread in k_quantize_planar
  int qp_runtime_c = 0;  // 1: runtime band count for the C = 12 PCA quantiser
  int eval_kernel = 0;   // SSIM kernel: 0 / 8 = k_eval_ssim8 (default), 7 = k_eval_ssim7
};
extern Variants g_variants;

// ----------------------------------------------------------------- limits
constexpr int kMaxC = 32;        // channels per stream handled by one CTA row
constexpr int kSsimRadius = 5;   // 11x11 window
constexpr int kSsimTaps = 2 * kSsimRadius + 1;

// threads per CTA for the "thread owns band tid % C" mapping: a multiple of C
// (and of 32) between 128 and 1024.
__host__ __device__ inline int threads_for_channels(int C) {
  int nt = 32 * C;
  while (nt < 128) nt *= 2;
  return nt;
}

// ----------------------------------------------------------------- typed loads
template <typename T> __device__ __forceinline__ T ldg(const T *p) { return __ldg(p); }

template <typename T> struct is_float_t { static constexpr bool value = false; };
template <> struct is_float_t<float> { static constexpr bool value = true; };
template <> struct is_float_t<double> { static constexpr bool value = true; };

// ----------------------------------------------------------------- ordered keys
// Monotone map double -> u64 so atomicMin/atomicMax on keys order like the
// doubles (-0.0 canonicalised to +0.0).
__device__ __forceinline__ unsigned long long dkey(double v) {
  if (v == 0.0) v = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
#endif
}

// statistics workspace entry, one per (cube, band)
struct StatsEntry {
  unsigned long long min_key;
  unsigned long long max_key;
  unsigned long long nan_count;
  unsigned int lead;   // some t=0 cell of the band is NaN (leading fill used)
  unsigned int pad;
};

// Commit per-thread band statistics (band = tid % C; NT = blockDim.x is a
// multiple of C) into the (cube-local) workspace: block reduce in shared
// memory, then one ordered-key atomic per band. `scratch` needs
// NT*(2*sizeof(Acc)+8) bytes and all threads must call this.
template <typename Acc>
__device__ void commit_band_stats(Acc mn, Acc mx, unsigned nanc, bool lead, int C,
                                  StatsEntry *ws_cube, unsigned char *scratch) {
  const int NT = blockDim.x, tid = threadIdx.x;
  Acc *smn = reinterpret_cast<Acc *>(scratch);
  Acc *smx = smn + NT;
  unsigned *snan = reinterpret_cast<unsigned *>(smx + NT);
  unsigned *slead = snan + NT;
  __syncthreads();
  smn[tid] = mn;
  smx[tid] = mx;
  snan[tid] = nanc;
  slead[tid] = lead ? 1u : 0u;
  __syncthreads();
  if (tid < C) {
    Acc bmn = smn[tid], bmx = smx[tid];
    unsigned long long bn = 0;
    unsigned bl = 0;
    for (int i = tid; i < NT; i += C) {
      bmn = min(bmn, smn[i]);
      bmx = max(bmx, smx[i]);
      bn += snan[i];
      bl |= slead[i];
    }
    StatsEntry *en = ws_cube + tid;
    if (bmn <= bmx) {
      atomicMin(&en->min_key, dkey((double)bmn));
      atomicMax(&en->max_key, dkey((double)bmx));
    }
    if (bn) atomicAdd(&en->nan_count, bn);
    if (bl) atomicOr(&en->lead, 1u);
  }
  __syncthreads();
}

__device__ __forceinline__ void flag(uint32_t *err, uint32_t f) {
  if (err) atomicOr(err, f);
}

// warp-aggregated flag: one atomic per warp
__device__ __forceinline__ void flag_warp(uint32_t *err, bool cond, uint32_t f) {
  unsigned m = __ballot_sync(__activemask(), cond);
  if (m && (threadIdx.x & 31) == (unsigned)(__ffs(m) - 1)) flag(err, f);
}

// --------------------------------------------------------------- fill carries
// Forward-fill value entering time segment `seg` for element e: the last
// observation of an earlier local segment, else the carry handed over by
// earlier time shards (carry_in, NaN = none; multi-GPU T-sharding), else the
// leading fill constant (cube.py:236-242 semantics).
__device__ __forceinline__ float segment_carry(const float *__restrict__ sl_cube, int64_t seg,
                                               int64_t inner, int64_t e,
                                               const float *__restrict__ carry_in_cube, float fill) {
  for (int64_t s = seg - 1; s >= 0; --s) {
    const float v = sl_cube[s * inner + e];
    if (!isnan(v)) return v;
  }
  if (carry_in_cube) {
    const float v = carry_in_cube[e];
    if (!isnan(v)) return v;
  }
  return fill;
}

// --------------------------------------------------------------- fill lookback
// Forward-fill value of element `e` at time t of cube `a` when src[t][e] is
// NaN: walk back inside the current segment, then over the per-segment
// last-observed map; no observation -> the leading fill constant
// (cube.py:236-242 semantics).
template <typename TIn>
__device__ __forceinline__ float fill_lookback(const TIn *__restrict__ cube, int64_t t,
                                               int64_t inner, int64_t e, int seg_len,
                                               const float *__restrict__ seg_last_cube,
                                               float fill) {
  const int64_t seg = t / seg_len;
  const int64_t t_lo = seg * seg_len;
  for (int64_t u = t - 1; u >= t_lo; --u) {
    float v = (float)cube[u * inner + e];
    if (!isnan(v)) return v;
  }
  for (int64_t s = seg - 1; s >= 0; --s) {
    float v = seg_last_cube[s * inner + e];
    if (!isnan(v)) return v;
  }
  return fill;
}

// ----------------------------------------------------------------- quantiser
// Per-band constants of quantize (transform.py:89-101).
struct QBand {
  double m, M, s, r, L;
  bool constant;
};

__device__ __forceinline__ QBand make_qband(double m, double M, int bit_depth) {
  QBand q;
  q.m = m;
  q.M = M;
  double span = __dsub_rn(M, m);
  q.constant = (span == 0.0);
  q.s = q.constant ? 1.0 : span;
  q.r = __drcp_rn(q.s);
  q.L = (double)((1u << bit_depth) - 1u);
  return q;
}

// q = floor(((v - m) / s) * L + 0.5) exactly as IEEE float64 evaluates it in
// the reference. Fast path: multiply by the rounded reciprocal; its result is
// within 6 ulp(L) (< 5e-11) of the reference x, so whenever x+0.5 is more than
// 2^-28 away from an integer both floors agree. Otherwise recompute with the
// correctly-rounded division in the reference's operation order.
__device__ __forceinline__ uint32_t quantize_value(double v, const QBand &b) {
  const double diff = __dsub_rn(v, b.m);
  double x = __dmul_rn(__dmul_rn(diff, b.r), b.L);
  double t = __dadd_rn(x, 0.5);
  double q = floor(t);
  double fr = __dsub_rn(t, q);
  const double eps = 3.725290298461914e-09;  // 2^-28
  if (fr < eps || fr > 1.0 - eps) {
    x = __dmul_rn(__ddiv_rn(diff, b.s), b.L);
    q = floor(__dadd_rn(x, 0.5));
  }
  if (b.constant) q = 0.0;
  // out-of-range values are flagged by the caller; keep the cast defined
  q = fmin(fmax(q, 0.0), 65535.0);
  return (uint32_t)q;
}

// Float32 fast path of the quantiser for float32 / integer sources.
// x32 = RN32(fma(v, RN32(K), RN32(-m K))), K = L/span, satisfies
//   |x32 + 0.5 - (x_ref + 0.5)| <= eps = 2^-24 (2L + 1 + 2 K A) + 2^-40 L,
// A = max(|min|, |max|), for every in-range v (x_ref: the reference's float64
// value). When frac(x32 + 0.5) is more than eps away from an integer the
// floor is the reference's; otherwise the element takes the exact float64
// path. Bands with eps > 2^-9 (huge offsets, 16-bit) always use float64.
// Range checks use the float neighbours of min/max, exact for float v.
struct QBand32 {
  float k, b, eps, lo, hi;
  bool use32;
};

__device__ __forceinline__ QBand32 make_qband32(const QBand &q, int clamp) {
  QBand32 r;
  const double K = q.L / q.s;
  const double A = fmax(fabs(q.m), fabs(q.M));
  const double eps = 5.9604644775390625e-08 * (2.0 * q.L + 1.0 + 2.0 * K * A) + 1e-12 * q.L;
  r.k = (float)K;
  r.b = (float)(-q.m * K);
  r.eps = (float)eps;
  r.lo = __double2float_ru(q.m);
  r.hi = __double2float_rd(q.M);
  r.use32 = !clamp && !q.constant && eps < 0.001953125;
  return r;
}

// Returns true and the code in q when the float32 path decides the element.
__device__ __forceinline__ bool quantize_fast32(float v, const QBand32 &b, uint32_t &q, bool &bad) {
  const float t = fmaf(v, b.k, b.b) + 0.5f;
  const float fl = floorf(t);
  const float fr = t - fl;
  bad |= (v < b.lo) || (v > b.hi);
  q = (uint32_t)fminf(fmaxf(fl, 0.f), 65535.f);
  return fr > b.eps && fr < 1.f - b.eps;
}

// RN(q / L) without a division: q0 = RN(q*rL), e = fma(-q0, L, q) (exact),
// RN(q0 + e*rL). Equal to the IEEE quotient for every q in [0, L] at all four
// bit depths (exhaustive proof: tests/test_exactness.py).
__device__ __forceinline__ double div_by_levels(double q, double L, double rL) {
  const double q0 = __dmul_rn(q, rL);
  const double e = __fma_rn(-q0, L, q);
  return __fma_rn(e, rL, q0);
}

// dequantize (transform.py:122-125): min + (q / L) * (max - min), same rounding
// as numpy's float64 evaluation order.
__device__ __forceinline__ double dequantize_value(uint32_t q, double m, double span, double L,
                                                   bool constant) {
  if (constant) return m;
  return __dadd_rn(m, __dmul_rn(div_by_levels((double)q, L, __drcp_rn(L)), span));
}

__device__ __forceinline__ double dequantize_fast(uint32_t q, double m, double span, double L,
                                                  double rL) {
  return __dadd_rn(m, __dmul_rn(div_by_levels((double)q, L, rL), span));
}

}  // namespace cvb
