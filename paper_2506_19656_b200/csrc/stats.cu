// K1 — per-band statistics with the forward-fill policy, and forward_fill_time.
//
// Replaces, for the array path:
//   fit_quant            /root/reference/pkg/src/cubevid/transform.py:61-70
//   forward_fill_time    /root/reference/pkg/src/cubevid/cube.py:213-246
//
// Work decomposition ("column chunk x time segment"): a CTA owns a contiguous
// chunk of NT*K elements of the inner (H*W*C) row and a segment of seg_len
// time steps; every thread owns K elements (tid + k*NT) and walks t inside the
// segment, so each time step is one fully coalesced sweep of the chunk and the
// per-element forward-fill carry lives in registers. NT is a multiple of C, so
// a thread's band is tid % C for all its elements.
#include <type_traits>
#include "common.cuh"

#ifndef CVB_STATS_KV
#define CVB_STATS_KV 2  // float4 vectors per thread and time step
#endif

namespace cvb {

constexpr int kStatsK = 4;

template <typename T> struct AccT { using type = float; };
template <> struct AccT<double> { using type = double; };

__global__ void k_stats_reset(StatsEntry *ws, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    ws[i].min_key = ~0ull;
    ws[i].max_key = 0ull;
    ws[i].nan_count = 0ull;
    ws[i].lead = 0u;
    ws[i].pad = 0u;
  }
}

template <typename TIn, int K>
__global__ void __launch_bounds__(1024)
k_stats(const TIn *__restrict__ src, int64_t T, int64_t inner, int C, int fill_mode, int seg_len,
        StatsEntry *__restrict__ ws, float *__restrict__ seg_last, uint32_t *err) {
  using Acc = typename AccT<TIn>::type;
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t a = blockIdx.z;
  const int64_t seg = blockIdx.y;
  const int64_t nseg = gridDim.y;
  const int64_t e0 = (int64_t)blockIdx.x * NT * K + tid;
  const int64_t t0 = seg * seg_len;
  const int64_t t1 = min(T, t0 + (int64_t)seg_len);
  const TIn *cube = src + a * T * inner;

  Acc mn = (Acc)INFINITY, mx = (Acc)-INFINITY;
  unsigned nanc = 0;
  bool lead = false, inf_seen = false;
  float last[K];
#pragma unroll
  for (int k = 0; k < K; ++k) last[k] = __int_as_float(0x7fc00000);

  for (int64_t t = t0; t < t1; ++t) {
    const TIn *row = cube + t * inner;
    TIn v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t e = e0 + (int64_t)k * NT;
      v[k] = (e < inner) ? ldg(row + e) : TIn(0);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t e = e0 + (int64_t)k * NT;
      if (e >= inner) continue;
      if constexpr (is_float_t<TIn>::value) {
        const TIn x = v[k];
        if (isnan(x)) {
          ++nanc;
          if (t == 0) lead = true;
        } else if (isinf(x)) {
          inf_seen = true;
        } else {
          mn = min(mn, (Acc)x);
          mx = max(mx, (Acc)x);
          last[k] = (float)x;
        }
      } else {
        mn = min(mn, (Acc)v[k]);
        mx = max(mx, (Acc)v[k]);
      }
    }
  }
  if (seg_last) {
    float *sl = seg_last + (a * nseg + seg) * inner;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t e = e0 + (int64_t)k * NT;
      if (e < inner) sl[e] = last[k];
    }
  }
  flag_warp(err, inf_seen, CV_FLAG_NONFINITE);
  flag_warp(err, fill_mode == 0 && nanc > 0, CV_FLAG_NAN);

  commit_band_stats<Acc>(mn, mx, nanc, lead, C, ws + a * C, smem);
}

// Vectorised K1 for rows whose length is a multiple of 4 (16 B loads of f32,
// 8 B of u16): thread lane j of a vector always sees band (4*tid + j) % C;
// the next time step's vectors are in flight while the current one is reduced.
template <typename TIn> struct SVec4T;
template <> struct SVec4T<float> { using type = float4; };
template <> struct SVec4T<uint16_t> { using type = ushort4; };

template <typename TIn, int KV>
__global__ void __launch_bounds__(1024)
k_stats_vec(const TIn *__restrict__ src, int64_t T, int64_t inner, int C, int fill_mode,
            int seg_len, StatsEntry *__restrict__ ws, float *__restrict__ seg_last, uint32_t *err) {
  using V = typename SVec4T<TIn>::type;
  constexpr int VEC = 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = blockDim.x, tid = threadIdx.x;
  const int64_t a = blockIdx.z, seg = blockIdx.y, nseg = gridDim.y;
  const int64_t e0 = (int64_t)blockIdx.x * NT * VEC * KV;
  const int64_t t0 = seg * seg_len;
  const int64_t t1 = min(T, t0 + (int64_t)seg_len);
  const TIn *cube = src + a * T * inner;
  int64_t voff[KV];
  bool vok[KV];
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    voff[k] = e0 + (int64_t)VEC * (tid + k * NT);
    vok[k] = voff[k] < inner;
  }
  float mn[VEC], mx[VEC];
  unsigned nanc[VEC];
  bool lead[VEC];
  float last[KV][VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    mn[j] = INFINITY;
    mx[j] = -INFINITY;
    nanc[j] = 0;
    lead[j] = false;
#pragma unroll
    for (int k = 0; k < KV; ++k) last[k][j] = __int_as_float(0x7fc00000);
  }
  V cur[KV], nxt[KV];
#pragma unroll
  for (int k = 0; k < KV; ++k)
    if (vok[k] && t0 < t1) cur[k] = __ldg(reinterpret_cast<const V *>(cube + t0 * inner + voff[k]));
  // leading gap flag: NaN in the cube's first frame
  if (t0 == 0 && t0 < t1) {
#pragma unroll
    for (int k = 0; k < KV; ++k)
      if (vok[k]) {
        const float x[VEC] = {(float)cur[k].x, (float)cur[k].y, (float)cur[k].z, (float)cur[k].w};
#pragma unroll
        for (int j = 0; j < VEC; ++j) lead[j] |= isnan(x[j]);
      }
  }
  // per element: min/max (fminf/fmaxf skip NaN; an infinity ends up as the
  // band's min or max and is flagged below), NaN count, last observation
  for (int64_t t = t0; t < t1; ++t) {
    if (t + 1 < t1) {
#pragma unroll
      for (int k = 0; k < KV; ++k)
        if (vok[k]) nxt[k] = __ldg(reinterpret_cast<const V *>(cube + (t + 1) * inner + voff[k]));
    }
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      if (!vok[k]) continue;
      const float x[VEC] = {(float)cur[k].x, (float)cur[k].y, (float)cur[k].z, (float)cur[k].w};
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const bool nan = x[j] != x[j];
        mn[j] = fminf(mn[j], x[j]);
        mx[j] = fmaxf(mx[j], x[j]);
        nanc[j] += nan ? 1u : 0u;
        last[k][j] = nan ? last[k][j] : x[j];
      }
    }
#pragma unroll
    for (int k = 0; k < KV; ++k) cur[k] = nxt[k];
  }
  bool inf_seen = false;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    // an infinity is the band's extreme once seen (the initial +/-INF of an
    // empty range sit on the opposite sides); it is an error either way
    inf_seen |= (mn[j] == -INFINITY) || (mx[j] == INFINITY);
  }
  if (seg_last && t0 < t1) {
    float *sl = seg_last + (a * nseg + seg) * inner;
#pragma unroll
    for (int k = 0; k < KV; ++k)
      if (vok[k])
        *reinterpret_cast<float4 *>(sl + voff[k]) = make_float4(last[k][0], last[k][1], last[k][2], last[k][3]);
  }
  flag_warp(err, inf_seen, CV_FLAG_NONFINITE);
  unsigned tn = nanc[0] + nanc[1] + nanc[2] + nanc[3];
  flag_warp(err, fill_mode == 0 && tn > 0, CV_FLAG_NAN);

  // per-band reduction over the 4*NT (thread, lane) entries; entry i has band i % C
  float *smn = reinterpret_cast<float *>(smem);
  float *smx = smn + VEC * NT;
  unsigned *snan = reinterpret_cast<unsigned *>(smx + VEC * NT);
  unsigned *slead = snan + VEC * NT;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    smn[VEC * tid + j] = mn[j];
    smx[VEC * tid + j] = mx[j];
    snan[VEC * tid + j] = nanc[j];
    slead[VEC * tid + j] = lead[j] ? 1u : 0u;
  }
  __syncthreads();
  if (tid < C) {
    float bmn = INFINITY, bmx = -INFINITY;
    unsigned long long bn = 0;
    unsigned bl = 0;
    for (int i = tid; i < VEC * NT; i += C) {
      bmn = fminf(bmn, smn[i]);
      bmx = fmaxf(bmx, smx[i]);
      bn += snan[i];
      bl |= slead[i];
    }
    StatsEntry *en = ws + a * C + tid;
    if (bmn <= bmx) {
      atomicMin(&en->min_key, dkey((double)bmn));
      atomicMax(&en->max_key, dkey((double)bmx));
    }
    if (bn) atomicAdd(&en->nan_count, bn);
    if (bl) atomicOr(&en->lead, 1u);
  }
}

__global__ void k_stats_lead(const StatsEntry *__restrict__ ws, int64_t n, int32_t *__restrict__ lead) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lead[i] = ws[i].lead ? 1 : 0;
}

__global__ void k_stats_finalize(const StatsEntry *__restrict__ ws, int64_t n, int fill_mode,
                                 float fill, double *mins, double *maxs, int64_t *nan_counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const StatsEntry e = ws[i];
  double mn = INFINITY, mx = -INFINITY;
  if (e.max_key != 0ull) {
    mn = dkey_inv(e.min_key);
    mx = dkey_inv(e.max_key);
  }
  if (fill_mode && e.lead) {
    mn = fmin(mn, (double)fill);
    mx = fmax(mx, (double)fill);
  }
  if (mins) mins[i] = mn;
  if (maxs) maxs[i] = mx;
  if (nan_counts) nan_counts[i] = (int64_t)e.nan_count;
}

// forward_fill_time body: filled values + validity mask, carries in registers.
template <int K>
__global__ void __launch_bounds__(256)
k_forward_fill(const float *__restrict__ src, int64_t T, int64_t inner, float fill, int seg_len,
               const float *__restrict__ seg_last, const float *__restrict__ carry_in,
               float *__restrict__ out, uint8_t *__restrict__ mask, uint32_t *err) {
  const int NT = blockDim.x;
  const int64_t a = blockIdx.z;
  const int64_t seg = blockIdx.y;
  const int64_t nseg = gridDim.y;
  const int64_t e0 = (int64_t)blockIdx.x * NT * K + threadIdx.x;
  const int64_t t0 = seg * seg_len;
  const int64_t t1 = min(T, t0 + (int64_t)seg_len);
  const float *cube = src + a * T * inner;
  const float *sl = seg_last + a * nseg * inner;
  const float *ci = carry_in ? carry_in + a * inner : nullptr;
  float carry[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t e = e0 + (int64_t)k * NT;
    carry[k] = e < inner ? segment_carry(sl, seg, inner, e, ci, fill) : fill;
  }
  bool inf_seen = false;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t off = (a * T + t) * inner;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t e = e0 + (int64_t)k * NT;
      if (e >= inner) continue;
      float v = __ldg(cube + t * inner + e);
      const bool ok = !isnan(v);
      if (ok) {
        inf_seen |= isinf(v);
        carry[k] = v;
      }
      out[off + e] = carry[k];
      if (mask) mask[off + e] = ok ? 1 : 0;
    }
  }
  flag_warp(err, inf_seen, CV_FLAG_NONFINITE);
}

template <typename TIn>
static void launch_stats(const void *src, int64_t n, int64_t T, int64_t inner, int C,
                         int fill_mode, int seg_len, void *ws, float *seg_last, uint32_t *err,
                         cudaStream_t st) {
  using Acc = typename AccT<TIn>::type;
  const int NT = threads_for_channels(C);
  const int64_t nseg = (T + seg_len - 1) / seg_len;
  if constexpr (std::is_same<TIn, float>::value || std::is_same<TIn, uint16_t>::value) {
    constexpr int KV = CVB_STATS_KV;
    if (inner % 4 == 0 && (((uintptr_t)src | (uintptr_t)seg_last) & 15) == 0) {
      const int64_t nchunk = (inner + (int64_t)NT * 4 * KV - 1) / ((int64_t)NT * 4 * KV);
      dim3 grid((unsigned)nchunk, (unsigned)nseg, (unsigned)n);
      const size_t sm = (size_t)NT * 4 * 16;
      if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_stats_vec<TIn, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_stats_vec<TIn, KV><<<grid, NT, sm, st>>>((const TIn *)src, T, inner, C, fill_mode, seg_len,
                                                   (StatsEntry *)ws, seg_last, err);
      return;
    }
  }
  const int64_t nchunk = (inner + (int64_t)NT * kStatsK - 1) / ((int64_t)NT * kStatsK);
  dim3 grid((unsigned)nchunk, (unsigned)nseg, (unsigned)n);
  size_t sm = (size_t)NT * (2 * sizeof(Acc) + 2 * sizeof(unsigned));
  k_stats<TIn, kStatsK><<<grid, NT, sm, st>>>((const TIn *)src, T, inner, C, fill_mode, seg_len,
                                               (StatsEntry *)ws, seg_last, err);
}

}  // namespace cvb

using namespace cvb;

extern "C" {

size_t cv_stats_ws_bytes(int64_t n_cubes, int32_t C) {
  return (size_t)(n_cubes * C) * sizeof(StatsEntry);
}

int64_t cv_num_segments(int64_t T, int32_t seg_len) {
  if (seg_len <= 0) return -1;
  return (T + seg_len - 1) / seg_len;
}

int cv_stats_reset(void *stats_ws, int64_t n_cubes, int32_t C, void *stream) {
  if (!stats_ws || n_cubes < 0 || C <= 0) return fail(CV_ERR_ARG, "cv_stats_reset: bad arguments");
  const int64_t n = n_cubes * C;
  if (n == 0) return CV_OK;
  k_stats_reset<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (StatsEntry *)stats_ws, n);
  return check_launch("cv_stats_reset");
}

int cv_stats(const void *src, int32_t dtype, int64_t n_cubes, int64_t T, int64_t inner, int32_t C,
             int32_t fill_mode, int32_t seg_len, void *stats_ws, float *seg_last,
             uint32_t *err_word, void *stream) {
  if (!src || !stats_ws) return fail(CV_ERR_ARG, "cv_stats: null pointer");
  if (C <= 0 || C > kMaxC)
    return fail(CV_ERR_UNSUPPORTED, "cv_stats: %d channels (supported 1..%d)", C, kMaxC);
  if (n_cubes < 0 || T < 0 || inner < 0 || inner % C != 0)
    return fail(CV_ERR_SHAPE, "cv_stats: inner=%lld is not a multiple of C=%d", (long long)inner, C);
  if (seg_len <= 0) return fail(CV_ERR_ARG, "cv_stats: seg_len must be positive");
  if (n_cubes > 65535 || cv_num_segments(T, seg_len) > 65535)
    return fail(CV_ERR_UNSUPPORTED, "cv_stats: grid too large (n_cubes or T/seg_len > 65535)");
  if (n_cubes == 0 || T == 0 || inner == 0) return CV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case CV_F32: launch_stats<float>(src, n_cubes, T, inner, C, fill_mode, seg_len, stats_ws, seg_last, err_word, st); break;
    case CV_F64: launch_stats<double>(src, n_cubes, T, inner, C, fill_mode, seg_len, stats_ws, nullptr, err_word, st); break;
    case CV_U16: launch_stats<uint16_t>(src, n_cubes, T, inner, C, 0, seg_len, stats_ws, nullptr, err_word, st); break;
    case CV_U8: launch_stats<uint8_t>(src, n_cubes, T, inner, C, 0, seg_len, stats_ws, nullptr, err_word, st); break;
    default: return fail(CV_ERR_ARG, "cv_stats: unknown dtype %d", dtype);
  }
  return check_launch("cv_stats");
}

int cv_stats_finalize(const void *stats_ws, int64_t n_cubes, int32_t C, int32_t fill_mode,
                      float fill_value, double *mins, double *maxs, int64_t *nan_counts,
                      void *stream) {
  if (!stats_ws || C <= 0 || n_cubes < 0) return fail(CV_ERR_ARG, "cv_stats_finalize: bad arguments");
  const int64_t n = n_cubes * C;
  if (n == 0) return CV_OK;
  k_stats_finalize<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const StatsEntry *)stats_ws, n, fill_mode, fill_value, mins, maxs, nan_counts);
  return check_launch("cv_stats_finalize");
}

int cv_stats_lead_flags(const void *stats_ws, int64_t n_cubes, int32_t C, int32_t *lead, void *stream) {
  if (!stats_ws || !lead || C <= 0 || n_cubes < 0) return fail(CV_ERR_ARG, "cv_stats_lead_flags: bad arguments");
  const int64_t n = n_cubes * C;
  if (n == 0) return CV_OK;
  k_stats_lead<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>((const StatsEntry *)stats_ws, n,
                                                                              lead);
  return check_launch("cv_stats_lead_flags");
}

int cv_forward_fill(const float *src, int64_t n_outer, int64_t T, int64_t inner, float fill_value,
                    int32_t seg_len, const float *seg_last, const float *carry_in, float *out,
                    uint8_t *mask, uint32_t *err_word, void *stream) {
  if (!src || !out || !seg_last) return fail(CV_ERR_ARG, "cv_forward_fill: null pointer");
  if (n_outer < 0 || T < 0 || inner < 0 || seg_len <= 0) return fail(CV_ERR_SHAPE, "cv_forward_fill: bad sizes");
  if (n_outer > 65535 || cv_num_segments(T, seg_len) > 65535)
    return fail(CV_ERR_UNSUPPORTED, "cv_forward_fill: grid too large");
  if (n_outer == 0 || T == 0 || inner == 0) return CV_OK;
  constexpr int K = 4;
  const int NT = 256;
  dim3 grid((unsigned)((inner + NT * K - 1) / (NT * K)), (unsigned)cv_num_segments(T, seg_len),
            (unsigned)n_outer);
  k_forward_fill<K><<<grid, NT, 0, (cudaStream_t)stream>>>(src, T, inner, fill_value, seg_len,
                                                            seg_last, carry_in, out, mask, err_word);
  return check_launch("cv_forward_fill");
}

}  // extern "C"
