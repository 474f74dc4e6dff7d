#include <cstdio>
#include <cuda_runtime.h>
// check: A 8x4 row (lane: row lane>>2, col lane%4), B 4x8 col (row lane%4, col lane>>2),
// C 8x8 (row lane>>2, cols (lane%4)*2 + {0,1})
__global__ void k(double* out) {
  const int L = threadIdx.x;
  double A[8][4], B[4][8];
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 4; ++c) A[r][c] = 1.0 + r * 4 + c;
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 8; ++c) B[r][c] = 0.5 + r * 8 + c * 0.25;
  double a = A[L >> 2][L & 3], b = B[L & 3][L >> 2], c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  const int r = L >> 2, cc = (L & 3) * 2;
  double e0 = 0, e1 = 0;
  for (int t = 0; t < 4; ++t) { e0 += A[r][t] * B[t][cc]; e1 += A[r][t] * B[t][cc + 1]; }
  out[L] = fabs(c0 - e0) + fabs(c1 - e1);
}
int main() {
  double* d; cudaMalloc(&d, 32 * 8); k<<<1, 32>>>(d); double h[32];
  cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < 32; ++i) m = h[i] > m ? h[i] : m;
  printf("max layout error %g\n", m);
}
