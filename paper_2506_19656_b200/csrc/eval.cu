// K5+K6 — decode (drop padded planes, dequantise, optional inverse PCA) fused
// with the fidelity metrics: per-band SSE (PSNR) and 11x11 Gaussian SSIM.
//
// Replaces, for the array path:
//   _planar_bytes_to_frames  /root/reference/pkg/src/cubevid/codecs/bridge.py:163-174
//   drop padded planes       plan.py:106 (ChannelGroup.n_real)
//   dequantize               /root/reference/pkg/src/cubevid/transform.py:108-126
//   pca_inverse              /root/reference/pkg/src/cubevid/transform.py:202-210
//   psnr / ssim              SPEC.md:419-436 (module absent in the reference)
//
// Decomposition: one CTA per (cube, frame t, column strip of TX pixels); it
// walks all H rows of its strip top to bottom, prefetching row y+1 into
// registers while row y is processed. Thread (px, c) owns one output column.
// Per row the CTA converts the strip row (+5-pixel halos) into the four SSIM
// maps (s, d, s^2, d^2), s = x'+y', d = x-y (x' = x - c0 shifted original,
// y' recon), stored as float4 in shared memory; each thread runs the 11-tap
// horizontal Gaussian and scatters the result into an 11-slot register ring
// that accumulates the vertical 11-tap filter. All Gaussian weights are
// compile-time immediates (full-rate FFMA on sm_100a: 120 FMA/clk/SM measured,
// vs 77 for the register form). Every input row is read once per strip, the
// recon is scored from registers (never re-read from HBM) and written once.
#include "common.cuh"
#include "pca_params.cuh"

#include "eval_kernel.cuh"
#include "ssim_kernel.cuh"
#include "ssim7_kernel.cuh"
#include "ssim8_kernel.cuh"
#include "psnr_kernel.cuh"

#include <cstdlib>

namespace cvb {

// Deterministic reduction of the per-CTA partials: out[a][c] (sse, ssim).
__global__ void k_eval_finalize(const double *__restrict__ part, int64_t n, int64_t nper, int C,
                                double *__restrict__ sse, double *__restrict__ ssim) {
  // one warp per output value, fixed-order tree reduction
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n * 2 * C) return;
  const int64_t a = w / (2 * C);
  const int k = (int)(w % (2 * C));
  const double *p = part + a * nper * 2 * C + k;
  double s = 0.0;
  for (int64_t i = lane; i < nper; i += 32) s += p[i * 2 * C];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    if (k < C) {
      if (sse) sse[a * C + k] = s;
    } else if (ssim) {
      ssim[a * C + (k - C)] = s;
    }
  }
}

static size_t eval_smem(int C, int E, int TX, bool ssim, bool pca) {
  const int halo = ssim ? kSsimRadius : 0;
  const int NX = TX + 2 * halo;
  size_t off = ssim ? 2 * (size_t)NX * C * sizeof(float4) : 0;
  off += pca ? (size_t)NX * C * sizeof(double) : 0;
  off += pca ? 2 * (size_t)E * sizeof(double) : 0;
  const size_t red = 2 * (size_t)TX * C * sizeof(double);
  return off > red ? off : red;
}

template <typename TO, int RS>
static int launch_eval2(const EvalArgs &a, const PcaParams &inv, bool pca, bool ssim, int64_t n,
                        cudaStream_t st) {
  if (ssim) {
    const int ncg = (a.C + kSsimWarpsPerCta - 1) / kSsimWarpsPerCta;
    const int wpc = a.C < kSsimWarpsPerCta ? a.C : kSsimWarpsPerCta;
    dim3 grid((unsigned)(a.nstrips * ncg), (unsigned)a.T, (unsigned)n);
    if constexpr ((RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16) && std::is_same<TO, float>::value) {
      // k_eval_ssim8 (mbarrier-handed rings, 5-pair straight-line vertical loop) is the default
      // for every decode mode (config 5 eval 58.8 ms, config 2 23.4 vs 24.6 ms for k_eval_ssim7);
      // "eval_kernel" = 7 forces the older kernel for A/B runs
      const int ek = g_variants.eval_kernel;
      if (a.ssim7 && ek != 7) {
        constexpr int fsz = RS == RS_FRAMES_U8 ? 1 : 2;
        const int ngrp = (a.C + k8GB - 1) / k8GB;
        dim3 g8((unsigned)(ssim8_strips(a.W) * ngrp), (unsigned)a.T, (unsigned)n);
#define CV_S8(MODE, EP, EX, CQ)                                                                              \
  do {                                                                                                   \
    const Ssim8Geom g8m = ssim8_geom(a.C, MODE == K8_PCA ? a.E : k8GB, fsz, MODE == K8_LUT);              \
    if (g8m.ns < 2) return fail(CV_ERR_UNSUPPORTED, "cv_eval: %d channels do not fit the SSIM kernel's rings", a.C); \
    const size_t sm = (size_t)g8m.total;                                                                 \
    cudaFuncSetAttribute(k_eval_ssim8<RS, MODE, EP, EX, CQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_eval_ssim8<RS, MODE, EP, EX, CQ><<<g8, k8Threads, sm, st>>>(a, inv);                               \
  } while (0)
        // codes of a full-range depth (8-bit in u8, 16-bit in u16) cannot exceed L: no range test
        const bool full = a.Li == (fsz == 1 ? 0xFFu : 0xFFFFu);
        if (pca) {
          if (a.E == 6 && full) CV_S8(K8_PCA, 6, true, false);
          else if (a.E == 6) CV_S8(K8_PCA, 6, true, true);
          else if (a.E == 9 && full) CV_S8(K8_PCA, 9, true, false);
          else if (a.E == 9) CV_S8(K8_PCA, 9, true, true);
          else CV_S8(K8_PCA, k8PcaMax, false, true);
        } else if (a.bit_depth <= 10) {
          CV_S8(K8_LUT, 0, false, true);
        } else {
          CV_S8(K8_F64, 0, false, true);
        }
#undef CV_S8
        return check_launch("cv_eval(ssim8)");
      }
      if (a.ssim7) {
        constexpr int fsz = RS == RS_FRAMES_U8 ? 1 : 2;
        const int ngrp = (a.C + k7GB - 1) / k7GB;
        dim3 g7((unsigned)(ssim7_strips(a.W) * ngrp), (unsigned)a.T, (unsigned)n);
#define CV_S7(MODE, EP)                                                                                  \
  do {                                                                                                   \
    const size_t sm = (size_t)ssim7_geom(a.C, MODE == K7_PCA ? a.E : k7GB, fsz, MODE == K7_LUT).total;    \
    if (sm > 227 * 1024) return fail(CV_ERR_UNSUPPORTED, "cv_eval: %d channels do not fit k_eval_ssim7's rings", a.C); \
    cudaFuncSetAttribute(k_eval_ssim7<RS, MODE, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_eval_ssim7<RS, MODE, EP><<<g7, k7Threads, sm, st>>>(a, inv);                                       \
  } while (0)
        if (pca) {
          if (a.E == 6) CV_S7(K7_PCA, 6);
          else if (a.E == 9) CV_S7(K7_PCA, 9);
          else CV_S7(K7_PCA, k7PcaMax);
        } else if (a.bit_depth <= 10) {
          CV_S7(K7_LUT, 0);
        } else {
          CV_S7(K7_F64, 0);
        }
#undef CV_S7
        return check_launch("cv_eval(ssim7)");
      }
    }
    if constexpr (RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16) {
      if (pca) k_eval_ssim<TO, RS, true, false><<<grid, 32 * wpc, 0, st>>>(a, inv);
      else if (std::is_same<TO, float>::value && a.W % 4 == 0)
        k_eval_ssim<TO, RS, false, std::is_same<TO, float>::value><<<grid, 32 * wpc, 0, st>>>(a, inv);
      else k_eval_ssim<TO, RS, false, false><<<grid, 32 * wpc, 0, st>>>(a, inv);
    } else {
      k_eval_ssim<TO, RS, false, false><<<grid, 32 * wpc, 0, st>>>(a, inv);
    }
    return check_launch("cv_eval(ssim)");
  }
  if constexpr ((RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16) &&
                (std::is_same<TO, float>::value || std::is_same<TO, uint16_t>::value)) {
    if (a.psnr_vec) {
      dim3 gp((unsigned)a.nstrips, (unsigned)a.T, (unsigned)n);
#define CV_PS(CC)                                                                        \
  do {                                                                                   \
    if (a.bit_depth <= 8) k_eval_psnr<TO, RS, true, CC><<<gp, kPsThreads, 0, st>>>(a);  \
    else k_eval_psnr<TO, RS, false, CC><<<gp, kPsThreads, 0, st>>>(a);                   \
  } while (0)
      if (a.C == 4) CV_PS(4);
      else CV_PS(7);
#undef CV_PS
      return check_launch("cv_eval(psnr)");
    }
  }
  const int NT = a.TX * a.C;
  dim3 grid((unsigned)a.nstrips, (unsigned)a.T, (unsigned)n);
  const size_t sm = eval_smem(a.C, a.E, a.TX, ssim, pca);
#define CV_EV(P, S)                                                                      \
  do {                                                                                   \
    auto kern = k_eval<TO, RS, P, S>;                                                    \
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    kern<<<grid, NT, sm, st>>>(a, inv);                                                  \
  } while (0)
  if constexpr (RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16) {
    if (pca) { if (ssim) CV_EV(true, true); else CV_EV(true, false); }
    else { if (ssim) CV_EV(false, true); else CV_EV(false, false); }
  } else {
    if (ssim) CV_EV(false, true); else CV_EV(false, false);
  }
#undef CV_EV
  return check_launch("cv_eval");
}

template <typename TO>
static int launch_eval1(const EvalArgs &a, const PcaParams &inv, bool pca, bool ssim, int64_t n,
                        int rs, cudaStream_t st) {
  switch (rs) {
    case RS_FRAMES_U8: return launch_eval2<TO, RS_FRAMES_U8>(a, inv, pca, ssim, n, st);
    case RS_FRAMES_U16: return launch_eval2<TO, RS_FRAMES_U16>(a, inv, pca, ssim, n, st);
    case RS_RECON_F32: return launch_eval2<TO, RS_RECON_F32>(a, inv, false, ssim, n, st);
    default: return launch_eval2<TO, RS_RECON_F64>(a, inv, false, ssim, n, st);
  }
}

}  // namespace cvb

using namespace cvb;

extern "C" {

size_t cv_eval_ws_bytes(int64_t n_cubes, int64_t T, int64_t H, int64_t W, int32_t C,
                        int32_t want_ssim) {
  (void)H;
  if (C <= 0) return 0;
  const int TX = eval_tx(C, want_ssim != 0);
  int64_t nstrips = (W + TX - 1) / TX;
  if (want_ssim && W >= kSsimTaps && (int64_t)ssim7_strips(W) > nstrips) nstrips = ssim7_strips(W);
  return (size_t)(n_cubes * T * nstrips * 2 * C) * sizeof(double);
}

int cv_eval(const void *frames, int32_t fdtype, int32_t E, const double *qmins, const double *qmaxs,
            int32_t bit_depth, const double *inv_mean, const double *inv_comps, const void *recon_in,
            int32_t rdtype, const void *orig, int32_t odtype, int64_t n_cubes, int64_t T, int64_t H,
            int64_t W, int32_t C, const double *peaks, int32_t want_ssim, float *recon_out, void *ws,
            double *sse, double *ssim_sum, uint32_t *err_word, void *stream) {
  if (!orig || !ws) return fail(CV_ERR_ARG, "cv_eval: null pointer");
  if ((frames == nullptr) == (recon_in == nullptr))
    return fail(CV_ERR_ARG, "cv_eval: pass exactly one of frames / recon_in");
  if (C <= 0 || C > kMaxC) return fail(CV_ERR_UNSUPPORTED, "cv_eval: %d channels (supported 1..%d)", C, kMaxC);
  if (n_cubes < 0 || T < 0 || H < 0 || W < 0) return fail(CV_ERR_SHAPE, "cv_eval: negative size");
  if (n_cubes > 65535 || T > 65535) return fail(CV_ERR_UNSUPPORTED, "cv_eval: grid too large");
  if (want_ssim && (H < kSsimTaps || W < kSsimTaps))
    return fail(CV_ERR_SHAPE, "cv_eval: frames %lldx%lld smaller than the %d-px SSIM window",
                (long long)H, (long long)W, kSsimTaps);
  if (want_ssim && !peaks) return fail(CV_ERR_ARG, "cv_eval: SSIM needs per-band peaks");
  const bool pca = inv_comps != nullptr;
  PcaParams inv;
  memset(&inv, 0, sizeof inv);
  int rs;
  if (frames) {
    if (!qmins || !qmaxs) return fail(CV_ERR_ARG, "cv_eval: frames need qmins/qmaxs");
    if (!(bit_depth == 8 || bit_depth == 10 || bit_depth == 12 || bit_depth == 16))
      return fail(CV_ERR_ARG, "bit depth %d not in (8, 10, 12, 16)", bit_depth);
    if (fdtype == CV_U8) rs = RS_FRAMES_U8;
    else if (fdtype == CV_U16) rs = RS_FRAMES_U16;
    else return fail(CV_ERR_ARG, "cv_eval: frames must be u8/u16");
    if (pca) {
      int s = make_pca_params(inv, inv_mean, inv_comps, E, C);
      if (s != CV_OK) return s;
    } else if (E != C) {
      return fail(CV_ERR_SHAPE, "cv_eval: E=%d encoded channels but C=%d without PCA", E, C);
    }
  } else {
    if (rdtype == CV_F32) rs = RS_RECON_F32;
    else if (rdtype == CV_F64) rs = RS_RECON_F64;
    else return fail(CV_ERR_ARG, "cv_eval: recon_in must be f32/f64");
    E = C;
  }
  if (n_cubes == 0 || T == 0 || H == 0 || W == 0) return CV_OK;
  EvalArgs a;
  a.frames = frames;
  a.E = E;
  a.G = (E + 2) / 3;
  a.qmins = qmins;
  a.qmaxs = qmaxs;
  a.bit_depth = frames ? bit_depth : 8;
  a.Li = (1u << a.bit_depth) - 1u;
  a.L = (double)a.Li;
  a.rL = 1.0 / a.L;  // IEEE division on the host: RN(1/L)
  a.recon_in = recon_in;
  a.orig = orig;
  a.T = T;
  a.H = H;
  a.W = W;
  a.C = C;
  a.peaks = peaks;
  a.recon_out = recon_out;
  a.part = (double *)ws;
  a.err = err_word;
  const bool ssim = want_ssim != 0;
  a.TX = eval_tx(C, ssim);
  a.nstrips = (int)((W + a.TX - 1) / a.TX);
  // the SSIM kernel with bulk-copied rows: frames, float32 original, 16-byte
  // aligned rows (original W*C*4 and frame W*b bytes), <= 12 PCA planes
  const int fsz = fdtype == CV_U8 ? 1 : 2;
  a.ssim7 = ssim && frames && odtype == CV_F32 && (W * C) % 4 == 0 && (W * fsz) % 16 == 0 &&
            H * W * C < (int64_t)1 << 31 &&
            ((uintptr_t)orig % 16) == 0 && ((uintptr_t)frames % 16) == 0 && (!pca || E <= k7PcaMax);
  if (a.ssim7) a.nstrips = ssim7_strips(W);
  // streaming PSNR-only kernel: frames, f32/u16 original, no PCA, C in {4, 7},
  // 4-pixel quads; nstrips = pixel chunks per frame (<= the workspace's strips)
  a.psnr_vec = !ssim && frames && !pca && (odtype == CV_F32 || odtype == CV_U16) && (C == 4 || C == 7) &&
               (H * W) % 4 == 0;
  if (a.psnr_vec) {
    const int64_t want = (H * W + 32767) / 32768;  // ~32 K pixels per CTA
    a.nstrips = (int)(want < a.nstrips ? want : a.nstrips);
    if (a.nstrips < 1) a.nstrips = 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int s;
  switch (odtype) {
    case CV_F32: s = launch_eval1<float>(a, inv, pca, ssim, n_cubes, rs, st); break;
    case CV_F64: s = launch_eval1<double>(a, inv, pca, ssim, n_cubes, rs, st); break;
    case CV_U16: s = launch_eval1<uint16_t>(a, inv, pca, ssim, n_cubes, rs, st); break;
    default: return fail(CV_ERR_ARG, "cv_eval: original dtype %d unsupported (f32/f64/u16)", odtype);
  }
  if (s != CV_OK) return s;
  const int64_t nper = T * a.nstrips;
  const int64_t nwarps = n_cubes * 2 * C;
  k_eval_finalize<<<(unsigned)((nwarps * 32 + 255) / 256), 256, 0, st>>>((const double *)ws, n_cubes,
                                                                         nper, C, sse, ssim_sum);
  return check_launch("cv_eval(finalize)");
}

}  // extern "C"
