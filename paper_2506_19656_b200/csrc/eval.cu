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
// walks all H rows of its strip top to bottom. Thread (px, c) owns one output
// column. Per row the CTA converts the strip row (+5-pixel halos) into
// (s, d) = (x'+y', x-y) pairs in shared memory (x' = x - c0 shifted original,
// y' recon), each thread runs the 11-tap horizontal Gaussian on four maps
// (s, d, s^2, d^2) and scatters the result into an 11-slot register ring that
// accumulates the vertical 11-tap filter; a slot completes 5 rows later and is
// turned into the SSIM value of output row y-5. Every input row is read once
// per strip (no halo rows), recon values never round-trip through HBM before
// being scored, and the recon is written once (f32, channel-last).
#include "common.cuh"
#include "pca_params.cuh"

namespace cvb {

struct EvalArgs {
  const void *frames;
  int E, G;
  const double *qmins, *qmaxs;
  int bit_depth;
  const void *recon_in;
  const void *orig;
  int fill_mode;
  float fill;
  int seg_len;
  const float *seg_last;
  int64_t T, H, W;
  int C;
  const double *peaks;
  float *recon_out;
  double *part;  // [n][T][nstrips][2C]
  uint32_t *err;
  int TX, nstrips;
};

enum { RS_FRAMES_U8 = 0, RS_FRAMES_U16 = 1, RS_RECON_F32 = 2, RS_RECON_F64 = 3 };

__host__ __device__ inline int eval_tx(int C) {
  if (C <= 2) return 64;
  if (C <= 16) return 32;
  return 16;
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

// SSIM from the filtered maps of s = x'+y' and d = x-y (x' = x-c0, y' = y-c0):
//   mu_x = (ms+md)/2 + c0, mu_y = (ms-md)/2 + c0,
//   sigma_x^2+sigma_y^2 = (vs+vd)/2, 2 sigma_xy = (vs-vd)/2,
// written as l = 1 - md^2/den_l, cs = 1 - vd/den_c to keep float32 exact
// where the signal is in the small difference map.
__device__ __forceinline__ float ssim_px(float ms, float md, float ess, float edd, float c0,
                                         float C1, float C2) {
  const float mx = 0.5f * (ms + md) + c0;
  const float my = 0.5f * (ms - md) + c0;
  const float vs = ess - ms * ms;
  const float vd = edd - md * md;
  const float den_l = mx * mx + my * my + C1;
  const float den_c = 0.5f * (vs + vd) + C2;
  const float l = den_l > 0.f ? 1.f - (md * md) / den_l : 1.f;
  const float cs = den_c > 0.f ? 1.f - vd / den_c : 1.f;
  return l * cs;
}

// Vertical filter step for input row y with U = y mod 11: scatter the
// horizontal results into the 11-slot ring (static slot indices, so the ring
// stays in registers) and return the completed slot of output row y-5.
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
    r.s[slot] = fmaf(w, hs, r.s[slot]);
    r.d[slot] = fmaf(w, hd, r.d[slot]);
    r.ss[slot] = fmaf(w, hss, r.ss[slot]);
    r.dd[slot] = fmaf(w, hdd, r.dd[slot]);
  }
  constexpr int fs = (U + 6) % 11;
  os = r.s[fs];
  od = r.d[fs];
  oss = r.ss[fs];
  odd = r.dd[fs];
  r.s[fs] = r.d[fs] = r.ss[fs] = r.dd[fs] = 0.f;
}

template <typename TO, int RS, bool PCA, bool SSIM>
__global__ void __launch_bounds__(512)
k_eval(const EvalArgs args, const PcaParams inv) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int HALO = SSIM ? kSsimRadius : 0;
  const int NT = blockDim.x, tid = threadIdx.x;
  const int C = args.C, E = args.E, TX = args.TX;
  const int NX = TX + 2 * HALO;
  const int64_t T = args.T, H = args.H, W = args.W;
  const int64_t HW = H * W, inner = HW * C;
  const int64_t a = blockIdx.z, t = blockIdx.y;
  const int strip = blockIdx.x;
  const int64_t x0 = (int64_t)strip * TX;
  const int c = tid % C;
  const int px = tid / C;  // output column of this thread (compute phase)
  const bool fill = args.fill_mode != 0;

  // shared memory: srow [2][NX*C] float2 | rec [NX*C] double | qband [E] (m, span)
  float2 *srow = reinterpret_cast<float2 *>(smem);
  size_t off = SSIM ? 2 * (size_t)NX * C * sizeof(float2) : 0;
  off = (off + 15) & ~(size_t)15;
  double *rec = reinterpret_cast<double *>(smem + off);
  off += PCA ? (size_t)NX * C * sizeof(double) : 0;
  double *qm = reinterpret_cast<double *>(smem + off);
  double *qs = qm + (PCA ? E : 0);
  if constexpr (PCA) {
    for (int j = tid; j < E; j += NT) {
      qm[j] = args.qmins[a * E + j];
      qs[j] = __dsub_rn(args.qmaxs[a * E + j], qm[j]);
    }
    __syncthreads();
  }
  const double L = (double)((1u << args.bit_depth) - 1u);
  double my_m = 0.0, my_span = 0.0;
  if constexpr (!PCA && (RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16)) {
    my_m = args.qmins[a * E + c];
    my_span = __dsub_rn(args.qmaxs[a * E + c], my_m);
  }
  const double peak = args.peaks ? args.peaks[a * C + c] : 1.0;
  const float c0 = (float)peak;
  const float C1 = (float)((0.01 * peak) * (0.01 * peak));
  const float C2 = (float)((0.03 * peak) * (0.03 * peak));
  const bool col_valid = SSIM && (x0 + px >= HALO) && (x0 + px < W - HALO) && (px < TX);

  const TO *ocube = reinterpret_cast<const TO *>(args.orig) + a * T * inner;
  const TO *orow_t = ocube + t * inner;
  const float *sl_cube = args.seg_last ? args.seg_last + a * ((T + args.seg_len - 1) / args.seg_len) * inner : nullptr;

  double sse = 0.0, ssum = 0.0;
  bool nanbad = false, intbad = false;
  Ring ring;
#pragma unroll
  for (int i = 0; i < 11; ++i) ring.s[i] = ring.d[i] = ring.ss[i] = ring.dd[i] = 0.f;
  int buf = 0;

  {
    for (int64_t y = 0; y < H; ++y) {
      const int64_t rowpix = y * W;
      // ---- PCA: dequantise the strip row's components and invert (1 thread / pixel)
      if constexpr (PCA) {
        for (int p = tid; p < NX; p += NT) {
          const int64_t x = x0 - HALO + p;
          if (x < 0 || x >= W) continue;
          double pc[kMaxC];
#pragma unroll
          for (int j = 0; j < kMaxC; ++j) {
            if (j < E) {
              const int64_t fi = (((a * args.G + j / 3) * T + t) * 3 + j % 3) * HW + rowpix + x;
              uint32_t q;
              if constexpr (RS == RS_FRAMES_U8) q = ldg(reinterpret_cast<const uint8_t *>(args.frames) + fi);
              else q = ldg(reinterpret_cast<const uint16_t *>(args.frames) + fi);
              intbad |= (double)q > L;
              pc[j] = dequantize_value(q, qm[j], qs[j], L, qs[j] == 0.0);
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
      // ---- load/convert phase: element (px_in, c) of the strip row
      for (int el = tid; el < NX * C; el += NT) {
        const int pin = el / C;
        const int64_t x = x0 - HALO + pin;
        float2 sd = make_float2(0.f, 0.f);
        if (x >= 0 && x < W) {
          const int64_t e = (rowpix + x) * C + c;
          float o;
          if constexpr (sizeof(TO) == 8) {
            o = (float)ldg(orow_t + e);
          } else {
            o = (float)ldg(orow_t + e);
          }
          if (isnan(o)) {
            if (fill) o = fill_lookback<TO>(ocube, t, inner, e, args.seg_len, sl_cube, args.fill);
            else nanbad = true;
          }
          double r;
          if constexpr (PCA) {
            r = rec[pin * C + c];
          } else if constexpr (RS == RS_FRAMES_U8 || RS == RS_FRAMES_U16) {
            const int64_t fi = (((a * args.G + c / 3) * T + t) * 3 + c % 3) * HW + rowpix + x;
            uint32_t q;
            if constexpr (RS == RS_FRAMES_U8) q = ldg(reinterpret_cast<const uint8_t *>(args.frames) + fi);
            else q = ldg(reinterpret_cast<const uint16_t *>(args.frames) + fi);
            intbad |= (double)q > L;
            r = dequantize_value(q, my_m, my_span, L, my_span == 0.0);
          } else if constexpr (RS == RS_RECON_F32) {
            r = (double)ldg(reinterpret_cast<const float *>(args.recon_in) + t * inner + a * T * inner + e);
          } else {
            r = ldg(reinterpret_cast<const double *>(args.recon_in) + t * inner + a * T * inner + e);
          }
          const double od = (double)o;
          const double diff = __dsub_rn(od, r);
          if (pin >= HALO && pin < HALO + TX) {
            sse = __fma_rn(diff, diff, sse);
            if (args.recon_out) args.recon_out[(a * T + t) * inner + e] = (float)r;
          }
          if constexpr (SSIM) {
            const float xs = (float)__dsub_rn(od, (double)c0);
            const float ys = (float)__dsub_rn(r, (double)c0);
            sd = make_float2(xs + ys, (float)diff);
          }
        }
        if constexpr (SSIM) srow[(size_t)buf * NX * C + el] = sd;
      }
      if constexpr (SSIM) {
        __syncthreads();
        if (px < TX) {
          const float2 *sr = srow + (size_t)buf * NX * C + (size_t)px * C + c;
          float hs = 0.f, hd = 0.f, hss = 0.f, hdd = 0.f;
#pragma unroll
          for (int k = 0; k < kSsimTaps; ++k) {
            const float2 v = sr[k * C];
            const float w = gtap(k < kSsimRadius ? kSsimRadius - k : k - kSsimRadius);
            hs = fmaf(w, v.x, hs);
            hd = fmaf(w, v.y, hd);
            hss = fmaf(w, v.x * v.x, hss);
            hdd = fmaf(w, v.y * v.y, hdd);
          }
          // scatter into the vertical ring: this row feeds outputs y-5 .. y+5
          float os, od, oss, odd;
          switch ((int)(y % 11)) {
            case 0: ring_step<0>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 1: ring_step<1>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 2: ring_step<2>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 3: ring_step<3>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 4: ring_step<4>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 5: ring_step<5>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 6: ring_step<6>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 7: ring_step<7>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 8: ring_step<8>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            case 9: ring_step<9>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
            default: ring_step<10>(ring, hs, hd, hss, hdd, os, od, oss, odd); break;
          }
          if (y >= 2 * kSsimRadius && col_valid) ssum += (double)ssim_px(os, od, oss, odd, c0, C1, C2);
        }
        buf ^= 1;
      } else if constexpr (PCA) {
        __syncthreads();  // rec reused by the next row
      }
    }
  }
  flag_warp(args.err, nanbad, CV_FLAG_NAN);
  flag_warp(args.err, intbad, CV_FLAG_INT_RANGE);

  // per-band partials: threads c, c+C, ... share band c (NT multiple of C)
  __syncthreads();
  double *red = reinterpret_cast<double *>(smem);
  red[tid] = sse;
  red[NT + tid] = ssum;
  __syncthreads();
  if (tid < C) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = tid; i < NT; i += C) {
      s1 += red[i];
      s2 += red[NT + i];
    }
    double *p = args.part + (((a * T + t) * args.nstrips) + strip) * 2 * C;
    p[tid] = s1;
    p[C + tid] = s2;
  }
}

// Deterministic reduction of the per-CTA partials: out[a][c] (sse, ssim).
__global__ void k_eval_finalize(const double *__restrict__ part, int64_t n, int64_t nper, int C,
                                double *__restrict__ sse, double *__restrict__ ssim) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over n * 2C
  if (i >= n * 2 * C) return;
  const int64_t a = i / (2 * C);
  const int w = (int)(i % (2 * C));
  double s = 0.0;
  const double *p = part + a * nper * 2 * C + w;
  for (int64_t k = 0; k < nper; ++k) s += p[k * 2 * C];
  if (w < C) {
    if (sse) sse[a * C + w] = s;
  } else {
    if (ssim) ssim[a * C + (w - C)] = s;
  }
}

static size_t eval_smem(int C, int E, int TX, bool ssim, bool pca) {
  const int halo = ssim ? kSsimRadius : 0;
  const int NX = TX + 2 * halo;
  size_t off = ssim ? 2 * (size_t)NX * C * sizeof(float2) : 0;
  off = (off + 15) & ~(size_t)15;
  off += pca ? (size_t)NX * C * sizeof(double) : 0;
  off += pca ? 2 * (size_t)E * sizeof(double) : 0;
  const size_t red = 2 * (size_t)TX * C * sizeof(double);
  return off > red ? off : red;
}

template <typename TO, int RS>
static int launch_eval2(const EvalArgs &a, const PcaParams &inv, bool pca, bool ssim, int64_t n,
                        cudaStream_t st) {
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
  (void)want_ssim;
  if (C <= 0) return 0;
  const int TX = eval_tx(C);
  const int64_t nstrips = (W + TX - 1) / TX;
  return (size_t)(n_cubes * T * nstrips * 2 * C) * sizeof(double);
}

int cv_eval(const void *frames, int32_t fdtype, int32_t E, const double *qmins, const double *qmaxs,
            int32_t bit_depth, const double *inv_mean, const double *inv_comps, const void *recon_in,
            int32_t rdtype, const void *orig, int32_t odtype, int32_t fill_mode, float fill_value,
            int32_t seg_len, const float *seg_last, int64_t n_cubes, int64_t T, int64_t H, int64_t W,
            int32_t C, const double *peaks, int32_t want_ssim, float *recon_out, void *ws,
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
  if (fill_mode && (odtype != CV_F32 || !seg_last || seg_len <= 0))
    return fail(CV_ERR_ARG, "cv_eval: fill_mode needs f32 original and a seg_last map");
  if (n_cubes == 0 || T == 0 || H == 0 || W == 0) return CV_OK;
  EvalArgs a;
  a.frames = frames;
  a.E = E;
  a.G = (E + 2) / 3;
  a.qmins = qmins;
  a.qmaxs = qmaxs;
  a.bit_depth = frames ? bit_depth : 8;
  a.recon_in = recon_in;
  a.orig = orig;
  a.fill_mode = fill_mode;
  a.fill = fill_value;
  a.seg_len = seg_len > 0 ? seg_len : 1;
  a.seg_last = seg_last;
  a.T = T;
  a.H = H;
  a.W = W;
  a.C = C;
  a.peaks = peaks;
  a.recon_out = recon_out;
  a.part = (double *)ws;
  a.err = err_word;
  a.TX = eval_tx(C);
  a.nstrips = (int)((W + a.TX - 1) / a.TX);
  cudaStream_t st = (cudaStream_t)stream;
  const bool ssim = want_ssim != 0;
  int s;
  switch (odtype) {
    case CV_F32: s = launch_eval1<float>(a, inv, pca, ssim, n_cubes, rs, st); break;
    case CV_F64: s = launch_eval1<double>(a, inv, pca, ssim, n_cubes, rs, st); break;
    case CV_U16: s = launch_eval1<uint16_t>(a, inv, pca, ssim, n_cubes, rs, st); break;
    case CV_U8: s = launch_eval1<uint8_t>(a, inv, pca, ssim, n_cubes, rs, st); break;
    default: return fail(CV_ERR_ARG, "cv_eval: unknown original dtype %d", odtype);
  }
  if (s != CV_OK) return s;
  const int64_t nper = T * a.nstrips;
  const int64_t nout = n_cubes * 2 * C;
  k_eval_finalize<<<(unsigned)((nout + 127) / 128), 128, 0, st>>>((const double *)ws, n_cubes, nper, C,
                                                                  sse, ssim_sum);
  return check_launch("cv_eval(finalize)");
}

}  // extern "C"
