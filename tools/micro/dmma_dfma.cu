// Do FP64 tensor-core MMAs (DMMA m8n8k4) and FP64 vector FMAs share a pipe?  Warps 0..W-1 run
// DMMA chains, the others DFMA chains (ILP 8); compare with each kind alone.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>  // 0: all DFMA, 1: all DMMA, 2: half warps DMMA / half DFMA
__global__ void k(double *x, int n) {
  const int w = threadIdx.x >> 5;
  const bool mma = MODE == 1 || (MODE == 2 && (w & 1));
  double acc[8], a = x[threadIdx.x] + 1e-3, b = x[threadIdx.x + 64] + 1e-3;
  for (int j = 0; j < 8; ++j) acc[j] = x[threadIdx.x + j];
  if (mma) {
    double d[4][2];
    for (int j = 0; j < 4; ++j) d[j][0] = d[j][1] = acc[j];
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    for (int j = 0; j < 4; ++j) acc[j] = d[j][0] + d[j][1];
  } else {
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fma(acc[j], a, b);
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 1.2345) x[0] = s;
}
int main() {
  double *x; cudaMalloc(&x, 1 << 20); cudaMemset(x, 0, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 20000, th = 512;
  const char *nm[] = {"DFMA only (16 warps x ILP 8)", "DMMA only (16 warps x 4 chains)", "half DMMA + half DFMA"};
  for (int m = 0; m < 3; ++m) {
    auto f = m == 0 ? k<0> : m == 1 ? k<1> : k<2>;
    f<<<148, th>>>(x, 100);
    cudaEventRecord(e0);
    f<<<148, th>>>(x, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = 148.0 * th / 32;
    double fma_dfma = 0, fma_dmma = 0;
    if (m == 0) fma_dfma = warps * 32 * 8.0 * n;
    if (m == 1) fma_dmma = warps * 4.0 * n * 256;
    if (m == 2) { fma_dfma = warps / 2 * 32 * 8.0 * n; fma_dmma = warps / 2 * 4.0 * n * 256; }
    printf("%-34s %.2f ms: DFMA %.1f T FMA/s + DMMA %.1f T FMA/s = %.1f T FMA/s\n", nm[m], ms, fma_dfma / ms / 1e9,
           fma_dmma / ms / 1e9, (fma_dfma + fma_dmma) / ms / 1e9);
  }
}
