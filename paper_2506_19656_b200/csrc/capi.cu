// Host-side glue of the C ABI: status strings, last-error, launch checks.
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace cvb {

static thread_local std::string g_last_error;
Variants g_variants;
// kernels launched through this library (every launch site calls check_launch once)
static std::atomic<unsigned long long> g_launches{0};

void set_last_error(const std::string &msg) { g_last_error = msg; }

int fail(int status, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int check_launch(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return CV_OK;
}

}  // namespace cvb

extern "C" {

int cv_version(void) { return 100; /* 0.1.0 */ }

const char *cv_status_string(int status) {
  switch (status) {
    case CV_OK: return "ok";
    case CV_ERR_ARG: return "invalid argument";
    case CV_ERR_SHAPE: return "inconsistent shape";
    case CV_ERR_UNSUPPORTED: return "unsupported by the B200 path";
    case CV_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

const char *cv_last_error(void) { return cvb::g_last_error.c_str(); }

int cv_max_channels(void) { return cvb::kMaxC; }

int cv_set_variant(const char *name, int value) {
  if (!name) return cvb::fail(CV_ERR_ARG, "cv_set_variant: null name");
  const std::string n(name);
  cvb::Variants &v = cvb::g_variants;
  if (n == "gram_tiles") v.gram_tiles = value != 0;
  else if (n == "gram_nt") {
    if (value != 64 && value != 256) return cvb::fail(CV_ERR_ARG, "gram_nt must be 64 or 256, got %d", value);
    v.gram_nt = value;
  } else if (n == "proj_nopf") v.proj_nopf = value != 0;
  else if (n == "proj12") v.proj12 = value != 0;
  else if (n == "gram_checks") v.gram_checks = value != 0;
  else if (n == "gram12") v.gram12 = value != 0;
  else if (n == "qp_px1") v.qp_px1 = value != 0;
  else if (n == "qp_runtime_c") v.qp_runtime_c = value != 0;
  else if (n == "eval_kernel") {
    if (value != 0 && value != 7 && value != 8)
      return cvb::fail(CV_ERR_ARG, "eval_kernel must be 0, 7 or 8, got %d", value);
    v.eval_kernel = value;
  }
  else return cvb::fail(CV_ERR_ARG, "cv_set_variant: unknown variant '%s'", name);
  return CV_OK;
}

unsigned long long cv_launch_count(void) { return cvb::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
