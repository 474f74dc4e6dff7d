// Latency of a dependent chain of DMMA m8n8k4 (one warp) vs DFMA, in cycles per link.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4, c0 = 0, c1 = 0, f = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) f = fma(a, b, f);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  out[threadIdx.x] = c0 + c1 + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 16);
  const int iters = 4096;
  k<<<1, 32>>>(o, c, iters); k<<<1, 32>>>(o, c, iters);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("dependent DMMA: %.1f cycles/link, dependent DFMA: %.1f cycles/link\n", (double)h[0] / iters, (double)h[1] / iters);
}
