// K5+K6 without SSIM (PSNR only), streaming variant: frames + float32/uint16
// original, no PCA, C <= 8, H*W % 4 == 0.
//
// The decode + SSE pass has no spatial window, so it is a pure stream: a CTA
// owns a contiguous pixel range of one frame t of one cube; each thread takes
// quads of 4 consecutive pixels, loads their 4*C original values as C 16-byte
// (f32) / 8-byte (u16) vectors, the 4 samples of every band's plane as one
// 4-byte (u8) / 8-byte (u16) vector, dequantises in float64 (shared table for
// 8 bits, exact division-free formula otherwise), accumulates the
// per-band float64 SSE and writes the 4*C recon values as C float4 stores.
// Two quads per thread are in flight per iteration (the row-walking k_eval
// kept only one element per thread in flight and was latency bound).
#pragma once
#include "eval_kernel.cuh"

namespace cvb {

constexpr int kPsMaxC = 8;
constexpr int kPsThreads = 256;
constexpr int kPsLut = 256;  // 8-bit table (static shared memory)

// CC: the band count (compile time, so every per-element index is static)
template <typename TO, int RS, bool LUT, int CC>
__global__ void __launch_bounds__(kPsThreads, 2)
k_eval_psnr(const EvalArgs args) {
  using R = typename RawT<RS>::type;
  using OV = typename std::conditional<std::is_same<TO, float>::value, float4, ushort4>::type;
  using FV = typename std::conditional<RS == RS_FRAMES_U8, uchar4, ushort4>::type;
  __shared__ double lut[LUT ? CC : 1][LUT ? kPsLut : 1];
  __shared__ double red[kPsThreads / 32][CC];
  constexpr int C = CC;
  const int64_t T = args.T, HW = args.H * args.W;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int nchunk = gridDim.x;
  const int64_t nquad = HW / 4;
  const int64_t q0 = nquad * blockIdx.x / nchunk, q1 = nquad * (blockIdx.x + 1) / nchunk;
  const double L = args.L, rL = args.rL;

  double m[CC], sp[CC], sse[CC];
#pragma unroll
  for (int c = 0; c < CC; ++c) {
    m[c] = args.qmins[a * C + c];
    sp[c] = __dsub_rn(args.qmaxs[a * C + c], m[c]);
    sse[c] = 0.0;
  }
  if constexpr (LUT) {
    for (int i = threadIdx.x; i < C * kPsLut; i += blockDim.x) {
      const int c = i / kPsLut, q = i % kPsLut;
      if (q <= (int)args.Li) {
        const double mc = args.qmins[a * C + c];
        lut[c][q] = dequantize_fast((uint32_t)q, mc, __dsub_rn(args.qmaxs[a * C + c], mc), L, rL);
      }
    }
    __syncthreads();
  }
  const TO *ob = reinterpret_cast<const TO *>(args.orig) + (a * T + t) * HW * C;
  float *rb = args.recon_out ? args.recon_out + (a * T + t) * HW * C : nullptr;
  const R *fb = reinterpret_cast<const R *>(args.frames) + ((a * args.G) * T + t) * 3 * HW;
  const int64_t pstride = 3 * T * HW;  // plane c -> plane c+3 (next video)
  uint32_t qmax = 0;

  auto quad = [&](int64_t q) {
    // original: 4 pixels x C bands = C vectors of 4
    TO o[4 * CC];
#pragma unroll
    for (int k = 0; k < CC; ++k) {
        const OV v = __ldg(reinterpret_cast<const OV *>(ob + q * 4 * C) + k);
        o[4 * k] = v.x;
        o[4 * k + 1] = v.y;
        o[4 * k + 2] = v.z;
        o[4 * k + 3] = v.w;
      }
    float r[4 * CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) {
        const FV f = __ldg(reinterpret_cast<const FV *>(fb + (c / 3) * pstride + (c % 3) * HW + q * 4));
        const uint32_t qs[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          qmax = max(qmax, qs[i]);
          double rm;
          if constexpr (LUT) rm = lut[c][min(qs[i], (uint32_t)(kPsLut - 1))];
          else rm = dequantize_fast(qs[i], m[c], sp[c], L, rL);
          const double diff = __dsub_rn((double)o[i * C + c], rm);
          sse[c] = __fma_rn(diff, diff, sse[c]);
          r[i * C + c] = (float)rm;
        }
      }
    if (rb) {
#pragma unroll
      for (int k = 0; k < CC; ++k)
          reinterpret_cast<float4 *>(rb + q * 4 * C)[k] =
              make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
    }
  };
  int64_t q = q0 + threadIdx.x;
  for (; q + blockDim.x < q1; q += 2 * blockDim.x) {
    quad(q);
    quad(q + blockDim.x);
  }
  if (q < q1) quad(q);

  flag_warp(args.err, qmax > args.Li, CV_FLAG_INT_RANGE);
  // per-band CTA reduction (warp shuffles, then one row per warp)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < CC; ++c) {
    double v = sse[c];
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    if (lane == 0) red[wid][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < C) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w][threadIdx.x];
    // partials layout [n][T][nstrips][2C]: strip = chunk; SSIM sums zero
    double *p = args.part + ((a * T + t) * args.nstrips + blockIdx.x) * 2 * C;
    p[threadIdx.x] = v;
    p[C + threadIdx.x] = 0.0;
  }
  // strips beyond the chunk count (nstrips from the row-walking layout) stay
  // unused: the launcher sets nstrips = chunks
}

}  // namespace cvb
