// peaks.cu — microbenchmarks of the SIMT pipes the SF kernel is bound by (FP32 FFMA,
// packed FFMA2, FP64 DFMA, MUFU rsqrt), for the roofline denominators that
// MEASURED_PEAKS.json does not carry. Each thread runs 8 independent chains.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int CH = 8;

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, int iters, float a, float b) {
  float2 x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  const float2 aa = make_float2(a, a), bb = make_float2(b, b);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(x[c], aa, bb);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c].x + x[c].y;
  if (s == 12345.f) out[0] = s;
}

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_mufu(float* out, int iters) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = 1.0f + threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = rsqrtf(x[c]) + 1.0f;
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.f) out[0] = s;
}
}  // namespace

extern "C" {
// which: 0 FFMA (flop/s), 1 FFMA2 (flop/s), 2 DFMA (flop/s), 3 MUFU.RSQ (op/s). Returns ops/s.
double sfb_peak(int which, int blocks_per_sm, int iters) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256, blocks = sms * blocks_per_sm;
  void* buf = nullptr;
  cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    switch (which) {
      case 0: k_ffma<<<blocks, threads>>>((float*)buf, iters, 0.9999f, 1e-4f); break;
      case 1: k_ffma2<<<blocks, threads>>>((float*)buf, iters, 0.9999f, 1e-4f); break;
      case 2: k_dfma<<<blocks, threads>>>((double*)buf, iters, 0.9999, 1e-4); break;
      default: k_mufu<<<blocks, threads>>>((float*)buf, iters); break;
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = (which == 0 || which == 2) ? 2.0 : (which == 1 ? 4.0 : 1.0);
    const double ops = (double)blocks * threads * iters * CH * per;
    if (rep > 0) best = best > ops / (ms * 1e-3) ? best : ops / (ms * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
}
