// K2/K3 — band PCA: fp64 shifted Gram (+ band stats), projection (+ component
// stats) and inverse projection.
//
// Replaces, for the array path:
//   pca_fit (covariance)  /root/reference/pkg/src/cubevid/transform.py:172-179
//   pca_forward           /root/reference/pkg/src/cubevid/transform.py:191-199
//   fit_quant on the PCs  SPEC.md:229 (transform.py:61-70)
//   pca_inverse           /root/reference/pkg/src/cubevid/transform.py:202-210
// The eigendecomposition (transform.py:180-187) stays on the host (C x C).
#include "common.cuh"
#include "pca_params.cuh"

namespace cvb {

constexpr int kGramK = 4;   // elements per thread per chunk (projection)
#ifndef CVB_GRAM_K
#define CVB_GRAM_K 16
#endif
constexpr int kGramKG = CVB_GRAM_K;  // elements per thread per chunk (Gram): 4x the work per barrier

// Gram partial of one CTA over a grid-stride set of pixel chunks.
// Staging: thread-owns-elements (band tid % C) -> shifted f64 in smem;
// accumulation: 4x4 tiles of the upper block triangle, one tile per thread,
// pixels strided over the lanes sharing a tile.
template <typename TIn, int MAXT>
__global__ void __launch_bounds__(MAXT)
k_gram(const TIn *__restrict__ src, int64_t n_pix, int C, double *__restrict__ partials,
       StatsEntry *__restrict__ stats, uint32_t *err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = blockDim.x, tid = threadIdx.x;
  const int P = NT * kGramKG / C;
  const int CS = C + 1;  // padded row stride
  double *xs = reinterpret_cast<double *>(smem);  // [P][CS]
  const int nb = (C + 3) / 4;
  const int ntile = nb * (nb + 1) / 2;
  const int nlanes = NT / ntile;
  // tile of this thread
  const int my_tile = tid % ntile, my_lane = tid / ntile;
  int bi = 0, bj = 0;
  {
    int tt = my_tile;
    for (int i = 0; i < nb; ++i) {
      const int row = nb - i;
      if (tt < row) { bi = i; bj = i + tt; break; }
      tt -= row;
    }
  }
  const bool tile_active = my_lane < nlanes;
  const int c = tid % C;
  const double shift = (double)ldg(src + c);

  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[r][s] = 0.0;
  double bsum = 0.0;
  float mn = INFINITY, mx = -INFINITY;
  double mnd = INFINITY, mxd = -INFINITY;
  bool nonfinite = false, isn = false;

  const int64_t nchunks = (n_pix + P - 1) / P;
  const int64_t ne = n_pix * C;
  // register prefetch of the next chunk (the staging barrier no longer
  // exposes the full load latency per chunk)
  TIn nxt[kGramKG];
  auto fetch = [&](int64_t ch) {
#pragma unroll
    for (int k = 0; k < kGramKG; ++k) {
      const int64_t e = ch * P * C + tid + k * NT;
      nxt[k] = (ch < nchunks && e < ne) ? ldg(src + e) : TIn(0);
    }
  };
  fetch(blockIdx.x);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t pix0 = ch * P;
    const int64_t e0 = pix0 * C;
    TIn cur[kGramKG];
#pragma unroll
    for (int k = 0; k < kGramKG; ++k) cur[k] = nxt[k];
    fetch(ch + gridDim.x);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kGramKG; ++k) {
      const int el = tid + k * NT;
      const int64_t e = e0 + el;
      double d = 0.0;
      if (e < ne) {
        const TIn v = cur[k];
        const double vd = (double)v;
        if constexpr (is_float_t<TIn>::value) {
          if (isnan(v)) isn = true;
          else if (isinf(v)) nonfinite = true;
        }
        mnd = fmin(mnd, vd);
        mxd = fmax(mxd, vd);
        d = __dsub_rn(vd, shift);
        if (isfinite(d)) bsum = __dadd_rn(bsum, d);
      }
      xs[(el / C) * CS + (el % C)] = isfinite(d) ? d : 0.0;
    }
    __syncthreads();
    if (tile_active) {
      const int lim = (int)min((int64_t)P, n_pix - pix0);
      for (int p = my_lane; p < lim; p += nlanes) {
        double rv[4], cv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int ci = 4 * bi + r, cj = 4 * bj + r;
          rv[r] = ci < C ? xs[p * CS + ci] : 0.0;
          cv[r] = cj < C ? xs[p * CS + cj] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int s = 0; s < 4; ++s) acc[r][s] = __fma_rn(rv[r], cv[s], acc[r][s]);
      }
    }
  }
  flag_warp(err, nonfinite, CV_FLAG_NONFINITE);
  flag_warp(err, isn, CV_FLAG_NAN);
  (void)mn;
  (void)mx;

  // band stats
  if (stats) commit_band_stats<double>(mnd, mxd, 0u, false, C, stats, smem);

  // deterministic CTA reduction of the tiles: red[lane][tile][16]
  __syncthreads();
  double *red = reinterpret_cast<double *>(smem);
  if (tile_active) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int s = 0; s < 4; ++s) red[((size_t)my_lane * ntile + my_tile) * 16 + r * 4 + s] = acc[r][s];
  }
  __syncthreads();
  const int stride = C + C * C;
  double *part = partials + (size_t)blockIdx.x * stride;
  for (int idx = tid; idx < ntile * 16; idx += NT) {
    const int tl = idx / 16, rs = idx % 16;
    double sum = 0.0;
    for (int l = 0; l < nlanes; ++l) sum += red[((size_t)l * ntile + tl) * 16 + rs];
    int tbi = 0, tbj = 0, tt = tl;
    for (int i = 0; i < nb; ++i) {
      const int row = nb - i;
      if (tt < row) { tbi = i; tbj = i + tt; break; }
      tt -= row;
    }
    const int ci = 4 * tbi + rs / 4, cj = 4 * tbj + rs % 4;
    if (ci < C && cj < C) {
      part[C + ci * C + cj] = sum;
      part[C + cj * C + ci] = sum;
    }
  }
  __syncthreads();
  // band sums: threads sharing band c
  red[tid] = bsum;
  __syncthreads();
  if (tid < C) {
    double s = 0.0;
    for (int i = tid; i < NT; i += C) s += red[i];
    part[tid] = s;
  }
}

// Pixel-per-lane Gram for float32 cubes with C <= kGpxC (ERA5 / SimpleS2: 12).
// Chunks of kGpxP pixels stream through a kGpxS-stage cp.async ring (one CTA
// per SM, ~60 KB in flight). Warp pair (2g, 2g+1) takes pixels g*32 + lane (+128) of
// the chunk; warp parity H owns half of the C(C+1)/2 products (static register
// indices, no shared-memory tiles) and the band statistics of bands
// [H*kGpxC/2, (H+1)*kGpxC/2). Same shifted one-pass sums as k_gram (shift =
// the first pixel), deterministic fixed-order reductions.
constexpr int kGpxC = 12;
constexpr int kGpxR = 2;  // pixel rounds per chunk: a chunk is blockDim.x pixels
constexpr int kGpxS = 6;
constexpr int kGpxNP = kGpxC * (kGpxC + 1) / 2;  // 78 products
constexpr int kGpxHalf = kGpxNP / 2;              // 39 per warp parity

__device__ __forceinline__ void gram_cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

template <int H, bool EXACT, bool CHK>
__device__ __forceinline__ void gram_px_accumulate(const float *__restrict__ px, int C_, const float (&sh)[kGpxC],
                                                   double (&acc)[kGpxHalf], double (&bsum)[kGpxC / 2],
                                                   float (&mn)[kGpxC / 2], float (&mx)[kGpxC / 2], bool &isn,
                                                   bool &nonfinite) {
  const int C = EXACT ? kGpxC : C_;
  float x[kGpxC];
  if (C == kGpxC) {
#pragma unroll
    for (int q = 0; q < kGpxC / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4 *>(px + 4 * q);
      x[4 * q] = v.x, x[4 * q + 1] = v.y, x[4 * q + 2] = v.z, x[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int c = 0; c < kGpxC; ++c) x[c] = c < C ? px[c] : sh[c];
  }
  double d[kGpxC];
#pragma unroll
  for (int c = 0; c < kGpxC; ++c) {
    const double dd = __dsub_rn((double)x[c], (double)sh[c]);
    d[c] = (!CHK || isfinite(dd)) ? dd : 0.0;
  }
#pragma unroll
  for (int j = 0; j < kGpxC / 2; ++j) {
    const int c = H * (kGpxC / 2) + j;
    if (c < C) {
      const float v = x[c];
      if (CHK) {
        isn |= isnan(v);
        nonfinite |= isinf(v);
      }
      mn[j] = fminf(mn[j], v);
      mx[j] = fmaxf(mx[j], v);
      bsum[j] = __dadd_rn(bsum[j], d[c]);
    }
  }
  int k = 0;
#pragma unroll
  for (int i = 0; i < kGpxC; ++i)
#pragma unroll
    for (int j = i; j < kGpxC; ++j, ++k)
      if (k >= H * kGpxHalf && k < (H + 1) * kGpxHalf) acc[k - H * kGpxHalf] = __fma_rn(d[i], d[j], acc[k - H * kGpxHalf]);
}

// CHK = false (default): no per-element finite tests. A NaN anywhere makes the
// products / sums of its band NaN and an infinity surfaces in the band's
// min / max, so both flags are read off the per-thread results once at the end;
// the sums of such a cube are not finite, and every caller discards them (fill
// first, or raise).
template <int NT, bool CHK>
__global__ void __launch_bounds__(NT, NT <= 64 ? 5 : 1)
k_gram_px(const float *__restrict__ src, int64_t n_pix, int C, double *__restrict__ partials,
          StatsEntry *__restrict__ stats, uint32_t *err) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kGpxP = NT;  // pixels per chunk
  float *ring = reinterpret_cast<float *>(smem);  // [kGpxS][kGpxP * C]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = warp & 1, wg = warp >> 1;
  const int SE = kGpxP * C;
  const int nvec = SE / 4;
  const int64_t ne = n_pix * C;
  const int64_t nchunks = (n_pix + kGpxP - 1) / kGpxP;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t nit = b < nchunks ? (nchunks - b + G - 1) / G : 0;

  float sh[kGpxC];
#pragma unroll
  for (int c = 0; c < kGpxC; ++c) sh[c] = c < C ? ldg(src + c) : 0.f;

  auto issue = [&](int64_t it) {
    float *st = ring + (size_t)(it % kGpxS) * SE;
    const int64_t e0 = (b + it * G) * SE;
    for (int v = tid; v < nvec; v += NT) {
      const int64_t e = e0 + 4 * (int64_t)v;
      if (e + 4 <= ne) gram_cp_async16(st + 4 * v, src + e);
      else
        for (int j = 0; j < 4; ++j) st[4 * v + j] = e + j < ne ? src[e + j] : 0.f;
    }
  };
#pragma unroll
  for (int s = 0; s < kGpxS - 1; ++s) {
    if (s < nit) issue(s);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }

  double acc[kGpxHalf];
#pragma unroll
  for (int k = 0; k < kGpxHalf; ++k) acc[k] = 0.0;
  double bsum[kGpxC / 2];
  float mn[kGpxC / 2], mx[kGpxC / 2];
#pragma unroll
  for (int j = 0; j < kGpxC / 2; ++j) bsum[j] = 0.0, mn[j] = INFINITY, mx[j] = -INFINITY;
  bool isn = false, nonfinite = false;
  const int p = wg * 32 + lane;

  for (int64_t it = 0; it < nit; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kGpxS - 2) : "memory");
    __syncthreads();
    if (it + kGpxS - 1 < nit) issue(it + kGpxS - 1);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const float *st = ring + (size_t)(it % kGpxS) * SE;
#pragma unroll
    for (int r = 0; r < kGpxR; ++r) {
      const int pp = p + (NT / 2) * r;
      if ((b + it * G) * kGpxP + pp < n_pix) {
        if (C == kGpxC) {
          if (H == 0) gram_px_accumulate<0, true, CHK>(st + pp * C, C, sh, acc, bsum, mn, mx, isn, nonfinite);
          else gram_px_accumulate<1, true, CHK>(st + pp * C, C, sh, acc, bsum, mn, mx, isn, nonfinite);
        } else {
          if (H == 0) gram_px_accumulate<0, false, CHK>(st + pp * C, C, sh, acc, bsum, mn, mx, isn, nonfinite);
          else gram_px_accumulate<1, false, CHK>(st + pp * C, C, sh, acc, bsum, mn, mx, isn, nonfinite);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (!CHK) {
#pragma unroll
    for (int k = 0; k < kGpxHalf; ++k) isn |= isnan(acc[k]);
#pragma unroll
    for (int j = 0; j < kGpxC / 2; ++j) {
      isn |= isnan(bsum[j]);
      nonfinite |= isinf(mn[j]) && mn[j] <= mx[j];
      nonfinite |= isinf(mx[j]) && mn[j] <= mx[j];
    }
#pragma unroll
    for (int c = 0; c < kGpxC; ++c) isn |= isnan(sh[c]);
  }
  flag_warp(err, nonfinite, CV_FLAG_NONFINITE);
  flag_warp(err, isn, CV_FLAG_NAN);

  // warp butterflies (fixed order), then the 4 pixel groups summed in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < kGpxHalf; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
#pragma unroll
    for (int j = 0; j < kGpxC / 2; ++j) {
      bsum[j] += __shfl_xor_sync(0xffffffffu, bsum[j], o);
      mn[j] = fminf(mn[j], __shfl_xor_sync(0xffffffffu, mn[j], o));
      mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], o));
    }
  }
  __syncthreads();  // ring reused as the reduction buffer
  double *red = reinterpret_cast<double *>(smem);  // [4][kGpxNP + kGpxC]
  constexpr int RS = kGpxNP + kGpxC;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kGpxHalf; ++k) red[wg * RS + H * kGpxHalf + k] = acc[k];
#pragma unroll
    for (int j = 0; j < kGpxC / 2; ++j) {
      const int c = H * (kGpxC / 2) + j;
      red[wg * RS + kGpxNP + c] = bsum[j];
      if (stats && c < C && mn[j] <= mx[j]) {
        atomicMin(&stats[c].min_key, dkey((double)mn[j]));
        atomicMax(&stats[c].max_key, dkey((double)mx[j]));
      }
    }
  }
  __syncthreads();
  double *part = partials + (size_t)b * (C + C * C);
  constexpr int ngroups = NT / 64;
  for (int idx = tid; idx < RS; idx += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < ngroups; ++g) s += red[g * RS + idx];
    if (idx < kGpxNP) {
      int i = 0, rem = idx;
      while (rem >= kGpxC - i) rem -= kGpxC - i, ++i;
      const int j = i + rem;
      if (i < C && j < C) {
        part[C + i * C + j] = s;
        part[C + j * C + i] = s;
      }
    } else if (idx - kGpxNP < C) {
      part[idx - kGpxNP] = s;
    }
  }
}

// Float32 cubes with exactly 12 bands: convert once, multiply from shared
// float64 tiles. k_gram_px converts and shifts every pixel twice (once per
// warp parity: 42 F2F + 28 DADD per pixel, XU pipe 43 % busy, 0.7 eligible
// warps per scheduler at 162 registers). Here a CTA has two roles:
//   * 3 converter warps (96 threads): thread i owns the 16-byte vectors
//     i + 96 k of a 128-pixel chunk (always the same four bands 4 (i % 3) ..),
//     copied with cp.async into a private 4-stage ring (only the copying
//     thread reads them back: no CTA barrier), converts them to shifted float64
//     once, keeps the band sums / min / max, and writes the pixel-major float64
//     tile (stride 14 doubles: conflict-free 16-byte reads);
//   * 4 product warps = 2 pairs x parity: a pair takes 64 pixels of the tile
//     (two per lane), each parity half of the 78 products in registers.
// Four tiles are in flight, handed over with named barriers (arrive / sync).
// (Loading the vectors two chunks ahead into registers instead of the cp.async ring freed a
// quarter of the shared-memory traffic but measured 14.5 vs 10.9 ms: the ring keeps three
// chunks per CTA in flight without holding registers.)
// Same shifted sums as k_gram_px (shift = first pixel), fixed-order reductions.
constexpr int kG12C = 12;
constexpr int kG12Conv = 96;                 // converter threads
constexpr int kG12Prod = 128;                // product threads
constexpr int kG12Threads = kG12Conv + kG12Prod;
constexpr int kG12K = 4;                     // 16-byte vectors per converter thread per chunk
constexpr int kG12Px = kG12Conv * kG12K / 3; // 128 pixels per chunk
constexpr int kG12Stages = 4;
constexpr int kG12PxStride = 14;             // doubles per pixel in the tile
constexpr int kG12Ring = kG12Stages * kG12Conv * kG12K * 16;         // bytes
constexpr int kG12Tile = kG12Px * kG12PxStride * 8;                  // bytes
constexpr int kG12Tiles = 4;  // float64 tiles in flight between the two roles (2 left both waiting on each other)
constexpr int kG12Smem = kG12Ring + kG12Tiles * kG12Tile;
// Tile hand-offs are named barriers (arrive / sync over the CTA's 224 threads); per-warp
// mbarriers measured slower here (11.3 vs 10.9 ms on config 5: the polls of seven warps
// compete with two resident CTAs' product warps).
constexpr int kG12BarFull = 1, kG12BarEmpty = 1 + kG12Tiles;

__device__ __forceinline__ void g12_bar_sync(int id) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(kG12Threads) : "memory");
}
__device__ __forceinline__ void g12_bar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "n"(kG12Threads) : "memory");
}

template <int H>
__device__ __forceinline__ void g12_products(const double *__restrict__ px, double (&acc)[kGpxHalf]) {
  double d[kG12C];
#pragma unroll
  for (int q = 0; q < kG12C / 2; ++q) {
    const double2 v = *reinterpret_cast<const double2 *>(px + 2 * q);
    d[2 * q] = v.x;
    d[2 * q + 1] = v.y;
  }
  int k = 0;
#pragma unroll
  for (int i = 0; i < kG12C; ++i)
#pragma unroll
    for (int j = i; j < kG12C; ++j, ++k)
      if (k >= H * kGpxHalf && k < (H + 1) * kGpxHalf) acc[k - H * kGpxHalf] = __fma_rn(d[i], d[j], acc[k - H * kGpxHalf]);
}

__global__ void __launch_bounds__(kG12Threads, 2)
k_gram12(const float *__restrict__ src, int64_t n_pix, double *__restrict__ partials,
         StatsEntry *__restrict__ stats, uint32_t *err) {
  extern __shared__ __align__(16) unsigned char smem[];
  float4 *ring = reinterpret_cast<float4 *>(smem);
  double *tiles = reinterpret_cast<double *>(smem + kG12Ring);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nvec = n_pix * 3;  // 16-byte vectors in the cube
  const int64_t nchunks = (n_pix + kG12Px - 1) / kG12Px;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t nit = b < nchunks ? (nchunks - b + G - 1) / G : 0;
  bool isn = false, nonfinite = false;
  constexpr int RS = kGpxNP + kG12C;
  double *red = reinterpret_cast<double *>(smem);  // end of kernel: [2 pairs][RS] + converter stats

  if (warp < 3) {
    // ------------------------------------------------------------ converters
    const int i = tid, r = i % 3;
    double shd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) shd[j] = (double)ldg(src + 4 * r + j);
    float mn[4], mx[4];
    double bs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) mn[j] = INFINITY, mx[j] = -INFINITY, bs[j] = 0.0;
    auto issue = [&](int64_t it) {
      if (it < nit) {
        const int64_t v0 = (b + it * G) * (kG12Conv * kG12K) + i;
        float4 *st = ring + (size_t)(it % kG12Stages) * (kG12Conv * kG12K) + i;
        const float4 *g = reinterpret_cast<const float4 *>(src) + v0;
        if (v0 - i + kG12Conv * kG12K <= nvec) {  // whole chunk inside the cube
#pragma unroll
          for (int k = 0; k < kG12K; ++k) gram_cp_async16(st + kG12Conv * k, g + kG12Conv * k);
        } else {
#pragma unroll
          for (int k = 0; k < kG12K; ++k)
            if (v0 + kG12Conv * k < nvec) gram_cp_async16(st + kG12Conv * k, g + kG12Conv * k);
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int s0 = 0; s0 < kG12Stages - 1; ++s0) issue(s0);
    for (int64_t it = 0; it < nit; ++it) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kG12Stages - 2) : "memory");
      issue(it + kG12Stages - 1);  // refills the stage this thread read one iteration ago
      const int bf = (int)(it % kG12Tiles);
      if (it >= kG12Tiles) g12_bar_sync(kG12BarEmpty + bf);
      const int64_t v0 = (b + it * G) * (kG12Conv * kG12K) + i;
      const float4 *st = ring + (size_t)(it % kG12Stages) * (kG12Conv * kG12K) + i;
      double *tile = tiles + (size_t)bf * (kG12Px * kG12PxStride);
      if (v0 - i + kG12Conv * kG12K <= nvec) {
        // whole chunk inside the cube: four independent vectors, no branches
        float4 x[kG12K];
#pragma unroll
        for (int k = 0; k < kG12K; ++k) x[k] = st[kG12Conv * k];
#pragma unroll
        for (int k = 0; k < kG12K; ++k) {
          const int vl = i + kG12Conv * k;  // vector inside the chunk: pixel vl / 3, bands 4 r ..
          double *dst = tile + (vl / 3) * kG12PxStride + 4 * r;
          const float xv[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
          double d[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mn[j] = fminf(mn[j], xv[j]);
            mx[j] = fmaxf(mx[j], xv[j]);
            d[j] = __dsub_rn((double)xv[j], shd[j]);
            bs[j] = __dadd_rn(bs[j], d[j]);
          }
          *reinterpret_cast<double2 *>(dst) = make_double2(d[0], d[1]);
          *reinterpret_cast<double2 *>(dst + 2) = make_double2(d[2], d[3]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < kG12K; ++k) {
          const int vl = i + kG12Conv * k;
          double *dst = tile + (vl / 3) * kG12PxStride + 4 * r;
          double d[4] = {0.0, 0.0, 0.0, 0.0};
          if (v0 + kG12Conv * k < nvec) {
            const float4 x = st[kG12Conv * k];
            const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              mn[j] = fminf(mn[j], xv[j]);
              mx[j] = fmaxf(mx[j], xv[j]);
              d[j] = __dsub_rn((double)xv[j], shd[j]);
              bs[j] = __dadd_rn(bs[j], d[j]);
            }
          }
          *reinterpret_cast<double2 *>(dst) = make_double2(d[0], d[1]);
          *reinterpret_cast<double2 *>(dst + 2) = make_double2(d[2], d[3]);
        }
      }
      g12_bar_arrive(kG12BarFull + bf);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      isn |= isnan(bs[j]) || isnan(shd[j]);
      nonfinite |= mn[j] <= mx[j] && (isinf(mn[j]) || isinf(mx[j]));
    }
    flag_warp(err, nonfinite, CV_FLAG_NONFINITE);
    flag_warp(err, isn, CV_FLAG_NAN);
    __syncthreads();  // every tile / ring read is done: the shared memory becomes the reduction buffer
    // converter stats: [96][4] sums, mins, maxs behind the product partials
    double *cs = red + 2 * RS;
    float *cf = reinterpret_cast<float *>(cs + kG12Conv * 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cs[i * 4 + j] = bs[j];
      cf[i * 8 + j] = mn[j];
      cf[i * 8 + 4 + j] = mx[j];
    }
    __syncthreads();
  } else {
    // ------------------------------------------------------------ product warps
    const int pw = warp - 3, H = pw & 1, pair = pw >> 1;
    double acc[kGpxHalf];
#pragma unroll
    for (int k = 0; k < kGpxHalf; ++k) acc[k] = 0.0;
    for (int64_t it = 0; it < nit; ++it) {
      const int bf = (int)(it % kG12Tiles);
      g12_bar_sync(kG12BarFull + bf);
      const double *tile = tiles + (size_t)bf * (kG12Px * kG12PxStride) + (size_t)(64 * pair + lane) * kG12PxStride;
      if (H == 0) {
        g12_products<0>(tile, acc);
        g12_products<0>(tile + 32 * kG12PxStride, acc);
      } else {
        g12_products<1>(tile, acc);
        g12_products<1>(tile + 32 * kG12PxStride, acc);
      }
      if (it + kG12Tiles < nit) g12_bar_arrive(kG12BarEmpty + bf);
    }
#pragma unroll
    for (int k = 0; k < kGpxHalf; ++k) isn |= isnan(acc[k]);
    flag_warp(err, isn, CV_FLAG_NAN);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int k = 0; k < kGpxHalf; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < kGpxHalf; ++k) red[pair * RS + H * kGpxHalf + k] = acc[k];
    __syncthreads();
  }
  // fixed-order CTA reduction (all threads)
  double *part = partials + (size_t)b * (kG12C + kG12C * kG12C);
  const double *cs = red + 2 * RS;
  const float *cf = reinterpret_cast<const float *>(cs + kG12Conv * 4);
  for (int idx = tid; idx < RS; idx += kG12Threads) {
    if (idx < kGpxNP) {
      const double s2 = red[idx] + red[RS + idx];
      int i2 = 0, rem = idx;
      while (rem >= kG12C - i2) rem -= kG12C - i2, ++i2;
      const int j2 = i2 + rem;
      part[kG12C + i2 * kG12C + j2] = s2;
      part[kG12C + j2 * kG12C + i2] = s2;
    } else {
      const int c = idx - kGpxNP, r = c / 4, j = c % 4;
      double s1 = 0.0;
      float lo = INFINITY, hi = -INFINITY;
      for (int t = r; t < kG12Conv; t += 3) {
        s1 += cs[t * 4 + j];
        lo = fminf(lo, cf[t * 8 + j]);
        hi = fmaxf(hi, cf[t * 8 + 4 + j]);
      }
      part[c] = s1;
      if (stats && lo <= hi) {
        atomicMin(&stats[c].min_key, dkey((double)lo));
        atomicMax(&stats[c].max_key, dkey((double)hi));
      }
    }
  }
}

// one warp per output: lanes stride over the CTA partials, fixed butterfly
// (deterministic for a given grid)
__global__ void k_reduce_partials(const double *__restrict__ partials, int nparts, int stride,
                                  double *__restrict__ out) {
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (i >= stride) return;
  double s = 0.0;
  for (int p = lane; p < nparts; p += 32) s += partials[(size_t)p * stride + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}

// Projection: stage spectra (thread-owns-elements), then one thread per pixel
// computes the K components; per-component min/max kept in registers (KB >= K).
template <typename TIn, typename TO, int KB>
__global__ void __launch_bounds__(1024)
k_pca_project(const TIn *__restrict__ src, int64_t n_pix, TO *__restrict__ out,
              StatsEntry *__restrict__ stats, const PcaParams pca, uint32_t *err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int NT = blockDim.x, tid = threadIdx.x;
  const int C = pca.C, K = pca.K;
  const int P = NT * kGramK / C;
  const int CS = C + 1;
  double *xs = reinterpret_cast<double *>(smem);
  const int64_t a = blockIdx.y;
  const TIn *cube = src + a * n_pix * C;
  double mn[KB], mx[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    mn[j] = INFINITY;
    mx[j] = -INFINITY;
  }
  bool bad = false;
  const int64_t nchunks = (n_pix + P - 1) / P;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t pix0 = ch * P;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kGramK; ++k) {
      const int el = tid + k * NT;
      const int64_t e = pix0 * C + el;
      double v = 0.0;
      if (e < n_pix * C) {
        v = (double)ldg(cube + e);
        bad |= !isfinite(v);
      }
      xs[(el / C) * CS + (el % C)] = v;
    }
    __syncthreads();
    for (int p = tid; p < P; p += NT) {
      const int64_t pix = pix0 + p;
      if (pix >= n_pix) break;
      double d[kMaxC];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c)
        if (c < C) d[c] = __dsub_rn(xs[p * CS + c], pca.mean[c]);
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        if (j < K) {
          const double pc = project_one(d, pca, j);
          mn[j] = fmin(mn[j], pc);
          mx[j] = fmax(mx[j], pc);
          if (out) out[(a * n_pix + pix) * K + j] = (TO)pc;
        }
      }
    }
  }
  flag_warp(err, bad, CV_FLAG_NONFINITE);
  if (stats) {
    // reduce per component: warp shuffle then one atomic per warp and component
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      if (j < K) {
        double a_mn = mn[j], a_mx = mx[j];
        for (int o = 16; o > 0; o >>= 1) {
          a_mn = fmin(a_mn, __shfl_xor_sync(0xffffffffu, a_mn, o));
          a_mx = fmax(a_mx, __shfl_xor_sync(0xffffffffu, a_mx, o));
        }
        if ((tid & 31) == 0 && a_mn <= a_mx) {
          atomicMin(&stats[a * K + j].min_key, dkey(a_mn));
          atomicMax(&stats[a * K + j].max_key, dkey(a_mx));
        }
      }
    }
  }
}

// Projection for C <= CM: one thread per pixel, its C values loaded straight
// into registers (a warp reads 32*C contiguous values), the differences to
// the mean kept in registers (CM static) and the K <= KB components formed
// with constant-bank weights; per-component min/max in registers. Several
// pixels per thread are in flight (PPT) to cover the load latency.
template <typename TIn, typename TO, int KB, int CM, int PPT>
__global__ void __launch_bounds__(256, (CM <= 12 && KB <= 8) ? 2 : 1)
k_pca_project_px(const TIn *__restrict__ src, int64_t n_pix, TO *__restrict__ out,
                 StatsEntry *__restrict__ stats, const PcaParams pca, uint32_t *err, bool pca_px_noprefetch = false) {
  const int C = pca.C, K = pca.K;
  const int64_t a = blockIdx.y;
  const TIn *cube = src + a * n_pix * C;
  double mn[KB], mx[KB];
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    mn[j] = INFINITY;
    mx[j] = -INFINITY;
  }
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * PPT;
  bool done = false;
  if constexpr (std::is_same<TIn, float>::value && CM % 4 == 0 && PPT == 1) {
    if (C == CM && !pca_px_noprefetch) {
      // exact-width pixels, software-pipelined: the next pixel's CM/4 16-byte
      // loads are in flight while this one is projected
      auto load = [&](int64_t pix, float4 (&q)[CM / 4]) {
#pragma unroll
        for (int c4 = 0; c4 < CM / 4; ++c4)
          q[c4] = pix < n_pix ? __ldg(reinterpret_cast<const float4 *>(cube + pix * C) + c4)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      float4 nq[CM / 4];
      int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
      load(pix, nq);
      for (; pix < n_pix; pix += stride) {
        float xv[CM];
#pragma unroll
        for (int c4 = 0; c4 < CM / 4; ++c4) {
          xv[4 * c4] = nq[c4].x, xv[4 * c4 + 1] = nq[c4].y, xv[4 * c4 + 2] = nq[c4].z, xv[4 * c4 + 3] = nq[c4].w;
        }
        load(pix + stride, nq);
        double d[CM];
#pragma unroll
        for (int c = 0; c < CM; ++c) {
          const double x = (double)xv[c];
          bad |= !isfinite(x);
          d[c] = __dsub_rn(x, pca.mean[c]);
        }
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          if (j < K) {
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < CM; ++c) acc = __fma_rn(d[c], pca.W[j * kMaxC + c], acc);
            mn[j] = fmin(mn[j], acc);
            mx[j] = fmax(mx[j], acc);
            if (out) out[(a * n_pix + pix) * K + j] = (TO)acc;
          }
        }
      }
      done = true;
    }
  }
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x * PPT + threadIdx.x; !done && p0 < n_pix; p0 += stride) {
    TIn v[PPT][CM];
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const int64_t pix = p0 + (int64_t)u * blockDim.x;
      if constexpr (std::is_same<TIn, float>::value && CM % 4 == 0) {
        if (C == CM) {  // whole pixel as CM/4 16-byte loads (pixel rows are 16-byte aligned)
#pragma unroll
          for (int c4 = 0; c4 < CM / 4; ++c4) {
            const float4 q = pix < n_pix ? __ldg(reinterpret_cast<const float4 *>(cube + pix * C) + c4)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
            v[u][4 * c4] = q.x;
            v[u][4 * c4 + 1] = q.y;
            v[u][4 * c4 + 2] = q.z;
            v[u][4 * c4 + 3] = q.w;
          }
          continue;
        }
      }
#pragma unroll
      for (int c = 0; c < CM; ++c) v[u][c] = (c < C && pix < n_pix) ? ldg(cube + pix * C + c) : TIn(0);
    }
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
      const int64_t pix = p0 + (int64_t)u * blockDim.x;
      if (pix >= n_pix) break;
      double d[CM];
#pragma unroll
      for (int c = 0; c < CM; ++c) {
        const double x = (double)v[u][c];
        if (c < C) bad |= !isfinite(x);
        d[c] = c < C ? __dsub_rn(x, pca.mean[c]) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        if (j < K) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < CM; ++c)
            if (c < C) acc = __fma_rn(d[c], pca.W[j * kMaxC + c], acc);
          mn[j] = fmin(mn[j], acc);
          mx[j] = fmax(mx[j], acc);
          if (out) out[(a * n_pix + pix) * K + j] = (TO)acc;
        }
      }
    }
  }
  flag_warp(err, bad, CV_FLAG_NONFINITE);
  if (stats) {
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      if (j < K) {
        double a_mn = mn[j], a_mx = mx[j];
        for (int o = 16; o > 0; o >>= 1) {
          a_mn = fmin(a_mn, __shfl_xor_sync(0xffffffffu, a_mn, o));
          a_mx = fmax(a_mx, __shfl_xor_sync(0xffffffffu, a_mx, o));
        }
        if ((threadIdx.x & 31) == 0 && a_mn <= a_mx) {
          atomicMin(&stats[a * K + j].min_key, dkey(a_mn));
          atomicMax(&stats[a * K + j].max_key, dkey(a_mx));
        }
      }
    }
  }
}

// Projection of float32 cubes with exactly 12 bands (ERA5 / SimpleS2), K = KE
// components. The weights sit in shared memory as float64 [KE][12] and are read
// with one broadcast LDS.64 per weight that serves TWO pixels of the thread
// (passed by value they end up in uniform registers, which spill at 72
// weights: the k_pca_project_px capture shows R2UR / MOV.SPILL / STL traffic at
// 36 thread-instructions per element against 6 DFMA). The next iteration's six
// 16-byte loads are in flight during the projection. Bit-identical to
// project_one (same fma order). A non-finite input makes every component
// non-finite (NaN / inf propagate through the fma chain, also past zero
// weights), so one check on the first component replaces the per-band tests.
__device__ __forceinline__ double lds_f64_volatile(uint32_t a) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}

constexpr int kP12Threads = 256;

template <typename TO, int KE, bool OUT>
__global__ void __launch_bounds__(kP12Threads, 2)
k_pca_project12(const float *__restrict__ src, int64_t n_pix, TO *__restrict__ out,
                StatsEntry *__restrict__ stats, const PcaParams pca, uint32_t *err) {
  constexpr int C = 12;
  __shared__ double wsm[KE * C];
  __shared__ double msm[C];
  const int64_t a = blockIdx.y;
  const float *cube = src + a * n_pix * C;
  for (int i = threadIdx.x; i < KE * C; i += kP12Threads) wsm[i] = pca.W[(i / C) * kMaxC + i % C];
  if (threadIdx.x < C) msm[threadIdx.x] = pca.mean[threadIdx.x];
  __syncthreads();
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(wsm);
  const uint32_t mbase = (uint32_t)__cvta_generic_to_shared(msm);
  double mn[KE], mx[KE];
#pragma unroll
  for (int j = 0; j < KE; ++j) {
    mn[j] = INFINITY;
    mx[j] = -INFINITY;
  }
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * (2 * kP12Threads);
  auto load = [&](int64_t pix, float4 (&q)[3]) {
#pragma unroll
    for (int c4 = 0; c4 < 3; ++c4)
      q[c4] = pix < n_pix ? __ldg(reinterpret_cast<const float4 *>(cube + pix * C) + c4)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  float4 n0[3], n1[3];
  int64_t pix = (int64_t)blockIdx.x * (2 * kP12Threads) + threadIdx.x;
  load(pix, n0);
  load(pix + kP12Threads, n1);
  for (; pix < n_pix; pix += stride) {
    double d0[C], d1[C];
#pragma unroll
    for (int c4 = 0; c4 < 3; ++c4) {
      const double m0 = lds_f64_volatile(mbase + 8u * (4 * c4)), m1 = lds_f64_volatile(mbase + 8u * (4 * c4 + 1));
      const double m2 = lds_f64_volatile(mbase + 8u * (4 * c4 + 2)), m3 = lds_f64_volatile(mbase + 8u * (4 * c4 + 3));
      d0[4 * c4] = __dsub_rn((double)n0[c4].x, m0);
      d0[4 * c4 + 1] = __dsub_rn((double)n0[c4].y, m1);
      d0[4 * c4 + 2] = __dsub_rn((double)n0[c4].z, m2);
      d0[4 * c4 + 3] = __dsub_rn((double)n0[c4].w, m3);
      d1[4 * c4] = __dsub_rn((double)n1[c4].x, m0);
      d1[4 * c4 + 1] = __dsub_rn((double)n1[c4].y, m1);
      d1[4 * c4 + 2] = __dsub_rn((double)n1[c4].z, m2);
      d1[4 * c4 + 3] = __dsub_rn((double)n1[c4].w, m3);
    }
    const bool v1 = pix + kP12Threads < n_pix;
    load(pix + stride, n0);
    load(pix + stride + kP12Threads, n1);
#pragma unroll
    for (int j = 0; j < KE; ++j) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double w = lds_f64_volatile(wbase + 8u * (uint32_t)(j * C + c));
        a0 = __fma_rn(d0[c], w, a0);
        a1 = __fma_rn(d1[c], w, a1);
      }
      if (j == 0) bad |= !isfinite(a0) || (v1 && !isfinite(a1));
      // compare-select (a NaN never wins, like fmin / fmax, at a third of their instructions)
      mn[j] = a0 < mn[j] ? a0 : mn[j];
      mx[j] = a0 > mx[j] ? a0 : mx[j];
      if (v1) {
        mn[j] = a1 < mn[j] ? a1 : mn[j];
        mx[j] = a1 > mx[j] ? a1 : mx[j];
      }
      if constexpr (OUT) {  // OUT = false: the range-only pass of the pipeline (no store code, fewer registers)
        out[(a * n_pix + pix) * KE + j] = (TO)a0;
        if (v1) out[(a * n_pix + pix + kP12Threads) * KE + j] = (TO)a1;
      }
    }
  }
  flag_warp(err, bad, CV_FLAG_NONFINITE);
  if (stats) {
#pragma unroll
    for (int j = 0; j < KE; ++j) {
      double a_mn = mn[j], a_mx = mx[j];
      for (int o = 16; o > 0; o >>= 1) {
        a_mn = fmin(a_mn, __shfl_xor_sync(0xffffffffu, a_mn, o));
        a_mx = fmax(a_mx, __shfl_xor_sync(0xffffffffu, a_mx, o));
      }
      if ((threadIdx.x & 31) == 0 && a_mn <= a_mx) {
        atomicMin(&stats[a * KE + j].min_key, dkey(a_mn));
        atomicMax(&stats[a * KE + j].max_key, dkey(a_mx));
      }
    }
  }
}

// Inverse projection: one thread per pixel.
template <typename TIn, typename TO>
__global__ void __launch_bounds__(256)
k_pca_inverse(const TIn *__restrict__ pc, int64_t n_total_pix, TO *__restrict__ out,
              const PcaParams pca) {
  const int C = pca.C, K = pca.K;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < n_total_pix;
       pix += (int64_t)gridDim.x * blockDim.x) {
    double v[kMaxC];
#pragma unroll
    for (int j = 0; j < kMaxC; ++j)
      if (j < K) v[j] = (double)ldg(pc + pix * K + j);
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < kMaxC; ++j)
        if (j < K) acc = __fma_rn(v[j], pca.W[j * kMaxC + c], acc);
      out[pix * C + c] = (TO)__dadd_rn(acc, pca.mean[c]);
    }
  }
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int gram_blocks(int64_t n_pix, int C) {
  const int NT = threads_for_channels(C);
  const int P = NT * kGramKG / C;
  const int64_t nchunks = (n_pix + P - 1) / P;
  int64_t nb = 5 * (int64_t)num_sms();
  if (nb > nchunks) nb = nchunks;
  if (nb < 1) nb = 1;
  return (int)nb;
}

template <typename TIn>
static int launch_gram(const void *src, int64_t n_pix, int C, void *ws, double *out, void *stats,
                       uint32_t *err, cudaStream_t st) {
  if constexpr (std::is_same<TIn, float>::value) {
    if (C == kG12C && ((uintptr_t)src & 15) == 0 && !g_variants.gram_tiles && g_variants.gram12) {
      int64_t nblk = (n_pix + kG12Px - 1) / kG12Px;
      if (nblk > 2 * (int64_t)num_sms()) nblk = 2 * (int64_t)num_sms();
      const int64_t cap = gram_blocks(n_pix, C);  // the workspace holds this many partials
      if (nblk > cap) nblk = cap;
      cudaFuncSetAttribute(k_gram12, cudaFuncAttributeMaxDynamicSharedMemorySize, kG12Smem);
      k_gram12<<<(unsigned)nblk, kG12Threads, kG12Smem, st>>>((const float *)src, n_pix, (double *)ws, (StatsEntry *)stats, err);
      int s = check_launch("cv_pca_gram(12)");
      if (s != CV_OK) return s;
      const int stride = C + C * C;
      k_reduce_partials<<<(stride + 7) / 8, 256, 0, st>>>((const double *)ws, (int)nblk, stride, out);
      return check_launch("cv_pca_gram(reduce)");
    }
    if (C <= kGpxC && ((uintptr_t)src & 15) == 0 && !g_variants.gram_tiles) {
      int nblk = gram_blocks(n_pix, C);
      if (nblk > num_sms()) nblk = num_sms();
      const int NT = g_variants.gram_nt == 256 ? 256 : 64;
      if (NT == 64) nblk = (int)min((int64_t)gram_blocks(n_pix, C), (int64_t)5 * num_sms());
      size_t sm = (size_t)kGpxS * NT * C * sizeof(float);
      const size_t smr = (size_t)(NT / 64) * (kGpxNP + kGpxC) * sizeof(double);
      if (smr > sm) sm = smr;
      auto kern = g_variants.gram_checks ? (NT == 64 ? k_gram_px<64, true> : k_gram_px<256, true>)
                                         : (NT == 64 ? k_gram_px<64, false> : k_gram_px<256, false>);
      if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<nblk, NT == 64 ? 64 : 256, sm, st>>>((const float *)src, n_pix, C, (double *)ws, (StatsEntry *)stats, err);
      int s = check_launch("cv_pca_gram(px)");
      if (s != CV_OK) return s;
      const int stride = C + C * C;
      k_reduce_partials<<<(stride + 7) / 8, 256, 0, st>>>((const double *)ws, nblk, stride, out);
      return check_launch("cv_pca_gram(reduce)");
    }
  }
  const int NT = threads_for_channels(C);
  const int P = NT * kGramKG / C;
  const int nb = (C + 3) / 4, ntile = nb * (nb + 1) / 2;
  size_t sm = (size_t)P * (C + 1) * sizeof(double);
  size_t sm2 = (size_t)NT * 16 * sizeof(double);  // tile reduction (>= ntile*nlanes*16)
  (void)ntile;
  if (sm2 > sm) sm = sm2;
  const int nblk = gram_blocks(n_pix, C);
  auto kern = NT <= 512 ? k_gram<TIn, 512> : k_gram<TIn, 1024>;
  if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kern<<<nblk, NT, sm, st>>>((const TIn *)src, n_pix, C, (double *)ws, (StatsEntry *)stats, err);
  int s = check_launch("cv_pca_gram");
  if (s != CV_OK) return s;
  const int stride = C + C * C;
  k_reduce_partials<<<(stride + 7) / 8, 256, 0, st>>>((const double *)ws, nblk, stride, out);
  return check_launch("cv_pca_gram(reduce)");
}

template <typename TIn, typename TO>
static int launch_project(const void *src, int64_t n_cubes, int64_t n_pix, const PcaParams &p,
                          void *out, void *stats, uint32_t *err, cudaStream_t st) {
  if (p.C <= 16 && p.K <= 16) {
    constexpr int PPT = 2;
    const int NT = 256;
    int64_t nb = (n_pix + (int64_t)NT * PPT - 1) / ((int64_t)NT * PPT);
    const int64_t cap = 8 * (int64_t)num_sms() / (n_cubes > 0 ? n_cubes : 1) + 1;
    if (nb > cap) nb = cap;
    if (nb < 1) nb = 1;
    dim3 grid((unsigned)nb, (unsigned)n_cubes);
#define CV_PX(KB, CM) \
  k_pca_project_px<TIn, TO, KB, CM, PPT><<<grid, NT, 0, st>>>((const TIn *)src, n_pix, (TO *)out, (StatsEntry *)stats, p, err)
    const bool al = ((uintptr_t)src & 15) == 0;
    if constexpr (std::is_same<TIn, float>::value) {
      if (p.C == 12 && al && g_variants.proj12 && (p.K == 6 || p.K == 9)) {
        // shared-memory weights, two pixels per thread, two CTAs per SM
        int64_t nb2 = (n_pix + 2 * kP12Threads - 1) / (2 * kP12Threads);
        // exactly two resident CTAs per SM in total: one CTA more would run alone after the
        // first wave (the i2 capture showed fp64-pipe max 67 % vs avg 45 % over the SMs)
        int64_t cap2 = 2 * (int64_t)num_sms() / (n_cubes > 0 ? n_cubes : 1);
        if (cap2 < 1) cap2 = 1;
        if (nb2 > cap2) nb2 = cap2;
        dim3 grid2((unsigned)(nb2 < 1 ? 1 : nb2), (unsigned)n_cubes);
#define CV_P12(KK, OO) k_pca_project12<TO, KK, OO><<<grid2, kP12Threads, 0, st>>>((const float *)src, n_pix, (TO *)out, (StatsEntry *)stats, p, err)
        if (p.K == 6) { if (out) CV_P12(6, true); else CV_P12(6, false); }
        else { if (out) CV_P12(9, true); else CV_P12(9, false); }
#undef CV_P12
        return check_launch("cv_pca_project(12)");
      }
    }
    if (p.C == 12 && al) {  // e.g. ERA5 / SimpleS2: exact-width register arrays, 16-byte loads,
                            // one pixel per thread and two CTAs per SM
      int64_t nb1 = (n_pix + NT - 1) / NT;
      if (nb1 > 2 * cap) nb1 = 2 * cap;
      dim3 grid1((unsigned)(nb1 < 1 ? 1 : nb1), (unsigned)n_cubes);
      if (p.K <= 8)
        k_pca_project_px<TIn, TO, 8, 12, 1><<<grid1, NT, 0, st>>>((const TIn *)src, n_pix, (TO *)out, (StatsEntry *)stats, p, err, g_variants.proj_nopf != 0);
      else
        k_pca_project_px<TIn, TO, 12, 12, 1><<<grid1, NT, 0, st>>>((const TIn *)src, n_pix, (TO *)out, (StatsEntry *)stats, p, err, g_variants.proj_nopf != 0);
    } else if (p.C <= 8) {
      if (p.K <= 8) CV_PX(8, 8); else CV_PX(16, 8);
    } else {
      if (p.K <= 8) CV_PX(8, 16); else CV_PX(16, 16);
    }
#undef CV_PX
    return check_launch("cv_pca_project(px)");
  }
  const int NT = threads_for_channels(p.C);
  const int P = NT * kGramK / p.C;
  const size_t sm = (size_t)P * (p.C + 1) * sizeof(double);
  const int64_t nchunks = (n_pix + P - 1) / P;
  int64_t nb = 4 * (int64_t)num_sms() / (n_cubes > 0 ? n_cubes : 1);
  if (nb < 1) nb = 1;
  if (nb > nchunks) nb = nchunks;
  dim3 grid((unsigned)nb, (unsigned)n_cubes);
#define CV_PROJ(KB)                                                                               \
  do {                                                                                            \
    auto kern = k_pca_project<TIn, TO, KB>;                                                       \
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    kern<<<grid, NT, sm, st>>>((const TIn *)src, n_pix, (TO *)out, (StatsEntry *)stats, p, err);  \
  } while (0)
  if (p.K <= 4) CV_PROJ(4);
  else if (p.K <= 8) CV_PROJ(8);
  else if (p.K <= 16) CV_PROJ(16);
  else CV_PROJ(32);
#undef CV_PROJ
  return check_launch("cv_pca_project");
}

}  // namespace cvb

using namespace cvb;

extern "C" {

size_t cv_gram_ws_bytes(int64_t n_pix, int32_t C) {
  if (C <= 0) return 0;
  return (size_t)gram_blocks(n_pix, C) * (size_t)(C + C * C) * sizeof(double);
}

int cv_pca_gram(const void *src, int32_t dtype, int64_t n_pix, int32_t C, void *ws, double *out,
                void *stats_ws, uint32_t *err_word, void *stream) {
  if (!src || !ws || !out) return fail(CV_ERR_ARG, "cv_pca_gram: null pointer");
  if (C <= 0 || C > kMaxC) return fail(CV_ERR_UNSUPPORTED, "cv_pca_gram: %d channels (supported 1..%d)", C, kMaxC);
  if (n_pix <= 0) return fail(CV_ERR_SHAPE, "cv_pca_gram: no pixels");
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case CV_F32: return launch_gram<float>(src, n_pix, C, ws, out, stats_ws, err_word, st);
    case CV_F64: return launch_gram<double>(src, n_pix, C, ws, out, stats_ws, err_word, st);
    case CV_U16: return launch_gram<uint16_t>(src, n_pix, C, ws, out, stats_ws, err_word, st);
    case CV_U8: return launch_gram<uint8_t>(src, n_pix, C, ws, out, stats_ws, err_word, st);
    default: return fail(CV_ERR_ARG, "cv_pca_gram: unknown dtype %d", dtype);
  }
}

int cv_pca_project(const void *src, int32_t dtype, int64_t n_cubes, int64_t n_pix, int32_t C,
                   const double *mean, const double *comps, int32_t K, void *out, int32_t out_dtype,
                   void *stats_ws, uint32_t *err_word, void *stream) {
  if (!src) return fail(CV_ERR_ARG, "cv_pca_project: null source");
  PcaParams p;
  int s = make_pca_params(p, mean, comps, K, C);
  if (s != CV_OK) return s;
  if (n_cubes < 0 || n_pix < 0 || n_cubes > 65535) return fail(CV_ERR_SHAPE, "cv_pca_project: bad sizes");
  if (n_cubes == 0 || n_pix == 0) return CV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool f64 = out_dtype == CV_F64;
  if (out && out_dtype != CV_F32 && out_dtype != CV_F64) return fail(CV_ERR_ARG, "cv_pca_project: out must be f32/f64");
  switch (dtype) {
    case CV_F32: return f64 ? launch_project<float, double>(src, n_cubes, n_pix, p, out, stats_ws, err_word, st)
                            : launch_project<float, float>(src, n_cubes, n_pix, p, out, stats_ws, err_word, st);
    case CV_F64: return f64 ? launch_project<double, double>(src, n_cubes, n_pix, p, out, stats_ws, err_word, st)
                            : launch_project<double, float>(src, n_cubes, n_pix, p, out, stats_ws, err_word, st);
    case CV_U16: return f64 ? launch_project<uint16_t, double>(src, n_cubes, n_pix, p, out, stats_ws, err_word, st)
                            : launch_project<uint16_t, float>(src, n_cubes, n_pix, p, out, stats_ws, err_word, st);
    default: return fail(CV_ERR_ARG, "cv_pca_project: unsupported dtype %d", dtype);
  }
}

int cv_pca_inverse(const void *pc, int32_t dtype, int64_t n_cubes, int64_t n_pix, int32_t K,
                   const double *mean, const double *comps, int32_t C, void *out, int32_t out_dtype,
                   void *stream) {
  if (!pc || !out) return fail(CV_ERR_ARG, "cv_pca_inverse: null pointer");
  PcaParams p;
  int s = make_pca_params(p, mean, comps, K, C);
  if (s != CV_OK) return s;
  const int64_t n = n_cubes * n_pix;
  if (n <= 0) return CV_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nb = (n + 255) / 256;
  if (nb > 148 * 32) nb = 148 * 32;
#define CV_INV(TI, TO) k_pca_inverse<TI, TO><<<(unsigned)nb, 256, 0, st>>>((const TI *)pc, n, (TO *)out, p)
  if (dtype == CV_F32 && out_dtype == CV_F32) CV_INV(float, float);
  else if (dtype == CV_F32 && out_dtype == CV_F64) CV_INV(float, double);
  else if (dtype == CV_F64 && out_dtype == CV_F32) CV_INV(double, float);
  else if (dtype == CV_F64 && out_dtype == CV_F64) CV_INV(double, double);
  else return fail(CV_ERR_ARG, "cv_pca_inverse: dtypes must be f32/f64");
#undef CV_INV
  return check_launch("cv_pca_inverse");
}

}  // extern "C"
