// Spectral angle, the third metric of the
// paper: per pixel theta = arccos(<o, r> / (|o| |r|)) over the channel vector,
// mean over pixels in degrees, zero-norm pixels skipped and counted.
// One thread per pixel, float64 dot products and arccos; per-CTA partials are
// reduced in a fixed order (deterministic).
#include "common.cuh"

namespace cvb {

template <typename TO, typename TR>
__global__ void __launch_bounds__(256)
k_spectral_angle(const TO *__restrict__ o, const TR *__restrict__ r, int64_t n_pix, int C,
                 double *__restrict__ part) {
  __shared__ double sh_sum[256];
  __shared__ unsigned long long sh_cnt[256];
  double sum = 0.0;
  unsigned long long cnt = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_pix;
       p += (int64_t)gridDim.x * blockDim.x) {
    const TO *op = o + p * C;
    const TR *rp = r + p * C;
    double dot = 0.0, no = 0.0, nr = 0.0;
    for (int c = 0; c < C; ++c) {
      const double a = (double)ldg(op + c), b = (double)ldg(rp + c);
      dot = __fma_rn(a, b, dot);
      no = __fma_rn(a, a, no);
      nr = __fma_rn(b, b, nr);
    }
    if (no > 0.0 && nr > 0.0) {
      double cs = dot / (sqrt(no) * sqrt(nr));
      cs = fmin(1.0, fmax(-1.0, cs));
      sum += acos(cs) * 57.29577951308232;  // degrees
      ++cnt;
    }
  }
  sh_sum[threadIdx.x] = sum;
  sh_cnt[threadIdx.x] = cnt;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh_sum[threadIdx.x] += sh_sum[threadIdx.x + s];
      sh_cnt[threadIdx.x] += sh_cnt[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sh_sum[0];
    part[2 * blockIdx.x + 1] = (double)sh_cnt[0];
  }
}

__global__ void k_angle_finalize(const double *__restrict__ part, int nparts, int64_t n_pix,
                                 double *__restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, n = 0.0;
  for (int i = 0; i < nparts; ++i) {
    s += part[2 * i];
    n += part[2 * i + 1];
  }
  out[0] = s;                  // sum of angles (degrees) over valid pixels
  out[1] = n;                  // valid pixels
  out[2] = (double)n_pix - n;  // skipped (zero-norm) pixels
}

constexpr int kAngleBlocks = 148 * 4;

}  // namespace cvb

using namespace cvb;

extern "C" {

size_t cv_angle_ws_bytes(void) { return (size_t)kAngleBlocks * 2 * sizeof(double); }

int cv_spectral_angle(const void *orig, int32_t odtype, const void *recon, int32_t rdtype,
                      int64_t n_pix, int32_t C, void *ws, double *out, void *stream) {
  if (!orig || !recon || !ws || !out) return fail(CV_ERR_ARG, "cv_spectral_angle: null pointer");
  if (C <= 0 || n_pix < 0) return fail(CV_ERR_SHAPE, "cv_spectral_angle: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nb = (n_pix + 255) / 256;
  if (nb > kAngleBlocks) nb = kAngleBlocks;
  if (nb < 1) nb = 1;
#define CV_ANG(TO, TR) \
  k_spectral_angle<TO, TR><<<(unsigned)nb, 256, 0, st>>>((const TO *)orig, (const TR *)recon, n_pix, C, (double *)ws)
  if (odtype == CV_F32 && rdtype == CV_F32) CV_ANG(float, float);
  else if (odtype == CV_F32 && rdtype == CV_F64) CV_ANG(float, double);
  else if (odtype == CV_F64 && rdtype == CV_F32) CV_ANG(double, float);
  else if (odtype == CV_F64 && rdtype == CV_F64) CV_ANG(double, double);
  else if (odtype == CV_U16 && rdtype == CV_F32) CV_ANG(uint16_t, float);
  else if (odtype == CV_U16 && rdtype == CV_F64) CV_ANG(uint16_t, double);
  else return fail(CV_ERR_ARG, "cv_spectral_angle: unsupported dtypes");
#undef CV_ANG
  int s = check_launch("cv_spectral_angle");
  if (s != CV_OK) return s;
  k_angle_finalize<<<1, 32, 0, st>>>((const double *)ws, (int)nb, n_pix, out);
  return check_launch("cv_spectral_angle(finalize)");
}

}  // extern "C"
