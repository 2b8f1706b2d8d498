// Microbenchmark of the arithmetic pipes the eval kernel leans on (sm_100a):
// FFMA (immediate weight), FFMA (register weight), FFMA2 (__ffma2_rn), DFMA, DDIV.
// Prints achieved operations per SM per clock-ish (ops / s / n_SM).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_ffma_imm(float *out, float seed) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], 0.999f, 0.001f);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_ffma_reg(float *out, float seed, float w, float b) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
  float ws[8]; for (int i = 0; i < 8; ++i) ws[i] = w + i * 1e-7f;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], ws[i], b + ws[7 - i]);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_ffma2(float *out, float seed, float w, float b) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(seed + threadIdx.x * 1e-3f + i, seed - i);
  float2 ws[8], bs[8];
  for (int i = 0; i < 8; ++i) { ws[i] = make_float2(w + i * 1e-7f, w); bs[i] = make_float2(b, b + i); }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], ws[i], bs[i]);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) out[0] = s;
}
__global__ void k_dfma(double *out, double seed) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 4; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999, 0.001);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.) out[0] = s;
}
__global__ void k_ddiv(double *out, double seed) {
  double a[4];
  for (int i = 0; i < 4; ++i) a[i] = seed + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 32; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __ddiv_rn(1023.0 + a[i], 1023.0) ;
  double s = 0; for (int i = 0; i < 4; ++i) s += a[i];
  if (s == 12345.) out[0] = s;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *fo; double *dout; cudaMalloc(&fo, 64); cudaMalloc(&dout, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256;
  auto run = [&](const char *name, auto launch, double ops_per_thread) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = ops_per_thread * blocks * threads;
    double per_sm_clk = ops / (ms * 1e-3) / nsm / (clk * 1e3);
    printf("%-10s %8.3f ms  %10.2f Gop/s  %7.2f op/clk/SM (at %d MHz max)\n", name, ms, ops / ms / 1e6, per_sm_clk, clk / 1000);
  };
  run("ffma_imm", [&] { k_ffma_imm<<<blocks, threads>>>(fo, 1.f); }, 8.0 * ITERS);
  run("ffma_reg", [&] { k_ffma_reg<<<blocks, threads>>>(fo, 1.f, 0.999f, 0.001f); }, 8.0 * ITERS);
  run("ffma2", [&] { k_ffma2<<<blocks, threads>>>(fo, 1.f, 0.999f, 0.001f); }, 16.0 * ITERS);
  run("dfma", [&] { k_dfma<<<blocks, threads>>>(dout, 1.0); }, 8.0 * ITERS / 4);
  run("ddiv", [&] { k_ddiv<<<blocks, threads>>>(dout, 1.0); }, 4.0 * ITERS / 32);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
