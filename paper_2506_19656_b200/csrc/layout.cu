// Layout kernels on either side of the hot path.
//
//   cv_select_stack  select_for_video  /root/reference/pkg/src/cubevid/cube.py:249-305
//                    (stack 3-D variables, or transpose one 4-D variable, into a
//                    contiguous channel-last [t, y, x, c] cube)
//   cv_planar_pack   _frames_to_planar_bytes  codecs/bridge.py:157-160
//                    ([t, y, x, c] integer frames -> planar [t, c, y, x] bytes)
//   cv_planar_unpack _planar_bytes_to_frames  codecs/bridge.py:163-174
//
// All three are pure data movement: a CTA takes one (t, y) row segment of 128
// pixels, gathers it channel by channel (coalesced when x is the variable's /
// plane's innermost axis) into a shared-memory tile laid out exactly like the
// channel-last destination, and writes the tile as one contiguous run (or the
// reverse for the unpack). Elements are moved as raw 1/2/4/8-byte words.
#include "common.cuh"

namespace cvb {

constexpr int kLayPx = 128;      // pixels per CTA tile
constexpr int kLayThreads = 256;

struct SelectArgs {
  const unsigned char *base[kMaxC];  // channel c starts here (device)
  int64_t st[kMaxC], sy[kMaxC], sx[kMaxC];  // element strides of the (t, y, x) roles
  int64_t T, H, W;
  int C;
};

template <typename U>
__global__ void __launch_bounds__(kLayThreads)
k_select_stack(const SelectArgs a, U *__restrict__ out) {
  __shared__ U tile[kLayPx * kMaxC];
  const int64_t t = blockIdx.z, y = blockIdx.y;
  const int64_t x0 = (int64_t)blockIdx.x * kLayPx;
  const int nx = (int)min((int64_t)kLayPx, a.W - x0);
  const int C = a.C;
  for (int i = threadIdx.x; i < kLayPx * C; i += kLayThreads) {
    const int c = i / kLayPx, x = i % kLayPx;
    if (x < nx) {
      const U *src = reinterpret_cast<const U *>(a.base[c]);
      tile[x * C + c] = src[t * a.st[c] + y * a.sy[c] + (x0 + x) * a.sx[c]];
    }
  }
  __syncthreads();
  U *dst = out + ((t * a.H + y) * a.W + x0) * C;
  for (int i = threadIdx.x; i < nx * C; i += kLayThreads) dst[i] = tile[i];
}

// PACK: q [T][HW][Cn] -> planes [T][Cn][HW]; !PACK: the inverse.
template <typename U, bool PACK>
__global__ void __launch_bounds__(kLayThreads)
k_planar(const U *__restrict__ in, U *__restrict__ out, int64_t HW, int Cn) {
  __shared__ U tile[kLayPx * kMaxC];
  const int64_t t = blockIdx.y;
  const int64_t p0 = (int64_t)blockIdx.x * kLayPx;
  const int np = (int)min((int64_t)kLayPx, HW - p0);
  if (PACK) {
    const U *src = in + (t * HW + p0) * Cn;
    for (int i = threadIdx.x; i < np * Cn; i += kLayThreads) tile[i] = src[i];
    __syncthreads();
    for (int i = threadIdx.x; i < kLayPx * Cn; i += kLayThreads) {
      const int c = i / kLayPx, p = i % kLayPx;
      if (p < np) out[(t * Cn + c) * HW + p0 + p] = tile[p * Cn + c];
    }
  } else {
    for (int i = threadIdx.x; i < kLayPx * Cn; i += kLayThreads) {
      const int c = i / kLayPx, p = i % kLayPx;
      if (p < np) tile[p * Cn + c] = in[(t * Cn + c) * HW + p0 + p];
    }
    __syncthreads();
    U *dst = out + (t * HW + p0) * Cn;
    for (int i = threadIdx.x; i < np * Cn; i += kLayThreads) dst[i] = tile[i];
  }
}

template <bool PACK>
static int launch_planar(const void *in, int32_t dtype, int64_t T, int64_t HW, int32_t Cn, void *out,
                         void *stream, const char *what) {
  if (!in || !out) return fail(CV_ERR_ARG, "%s: null pointer", what);
  if (dtype != CV_U8 && dtype != CV_U16) return fail(CV_ERR_ARG, "%s: frames must be u8/u16", what);
  if (Cn <= 0 || Cn > kMaxC) return fail(CV_ERR_UNSUPPORTED, "%s: %d planes (supported 1..%d)", what, Cn, kMaxC);
  if (T < 0 || HW < 0) return fail(CV_ERR_SHAPE, "%s: negative size", what);
  if (T > 65535) return fail(CV_ERR_UNSUPPORTED, "%s: grid too large", what);
  if (T == 0 || HW == 0) return CV_OK;
  dim3 grid((unsigned)((HW + kLayPx - 1) / kLayPx), (unsigned)T);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CV_U8) k_planar<uint8_t, PACK><<<grid, kLayThreads, 0, st>>>((const uint8_t *)in, (uint8_t *)out, HW, Cn);
  else k_planar<uint16_t, PACK><<<grid, kLayThreads, 0, st>>>((const uint16_t *)in, (uint16_t *)out, HW, Cn);
  return check_launch(what);
}

}  // namespace cvb

using namespace cvb;

extern "C" {

int cv_select_stack(const void *const *chan_ptrs, const int64_t *strides, int32_t C, int32_t elem_size,
                    int64_t T, int64_t H, int64_t W, void *out, void *stream) {
  if (!chan_ptrs || !strides || !out) return fail(CV_ERR_ARG, "cv_select_stack: null pointer");
  if (C <= 0 || C > kMaxC) return fail(CV_ERR_UNSUPPORTED, "cv_select_stack: %d channels (supported 1..%d)", C, kMaxC);
  if (T < 0 || H < 0 || W < 0) return fail(CV_ERR_SHAPE, "cv_select_stack: negative size");
  if (T > 65535 || H > 65535) return fail(CV_ERR_UNSUPPORTED, "cv_select_stack: grid too large");
  if (T == 0 || H == 0 || W == 0) return CV_OK;
  SelectArgs a;
  memset(&a, 0, sizeof a);
  for (int c = 0; c < C; ++c) {
    if (!chan_ptrs[c]) return fail(CV_ERR_ARG, "cv_select_stack: null channel pointer %d", c);
    a.base[c] = (const unsigned char *)chan_ptrs[c];
    a.st[c] = strides[3 * c];
    a.sy[c] = strides[3 * c + 1];
    a.sx[c] = strides[3 * c + 2];
  }
  a.T = T;
  a.H = H;
  a.W = W;
  a.C = C;
  dim3 grid((unsigned)((W + kLayPx - 1) / kLayPx), (unsigned)H, (unsigned)T);
  cudaStream_t st = (cudaStream_t)stream;
  switch (elem_size) {
    case 1: k_select_stack<uint8_t><<<grid, kLayThreads, 0, st>>>(a, (uint8_t *)out); break;
    case 2: k_select_stack<uint16_t><<<grid, kLayThreads, 0, st>>>(a, (uint16_t *)out); break;
    case 4: k_select_stack<uint32_t><<<grid, kLayThreads, 0, st>>>(a, (uint32_t *)out); break;
    case 8: k_select_stack<uint64_t><<<grid, kLayThreads, 0, st>>>(a, (uint64_t *)out); break;
    default: return fail(CV_ERR_ARG, "cv_select_stack: element size %d not in (1, 2, 4, 8)", elem_size);
  }
  return check_launch("cv_select_stack");
}

int cv_planar_pack(const void *q, int32_t dtype, int64_t T, int64_t HW, int32_t n_planes, void *out,
                   void *stream) {
  return launch_planar<true>(q, dtype, T, HW, n_planes, out, stream, "cv_planar_pack");
}

int cv_planar_unpack(const void *planes, int32_t dtype, int64_t T, int64_t HW, int32_t n_planes, void *out,
                     void *stream) {
  return launch_planar<false>(planes, dtype, T, HW, n_planes, out, stream, "cv_planar_unpack");
}

}  // extern "C"
