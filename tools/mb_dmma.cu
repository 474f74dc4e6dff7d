#include <cstdio>
#include <cuda_runtime.h>
// FP64 tensor-core throughput: mma.sync.m8n8k4.f64 (256 FMA per warp-instruction) vs DFMA
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (MODE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
      } else {
        c[t][0] = fma(a, b, c[t][0]);
        c[t][1] = fma(a, b, c[t][1]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<sms * 2, 256>>>(o, iters); else k<1><<<sms * 2, 256>>>(o, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double warps = sms * 2.0 * 8, ops = warps * iters * 8;   // warp-instructions (mma) or 2x DFMA
      if (rep) {
        if (mode == 0) printf("DMMA m8n8k4: %.3f ms, %.2f TFLOP/s, %.2f SM-cycles per DMMA\n", ms,
                              ops * 256 * 2 / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 * sms / ops);
        else printf("DFMA: %.3f ms, %.2f TFLOP/s, %.3f SM-cycles per warp-DFMA\n", ms,
                    ops * 2 * 32 * 2 / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 * sms / (ops * 2));
      }
    }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
