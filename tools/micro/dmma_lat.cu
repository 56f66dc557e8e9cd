// DMMA m8n8k4 f64 throughput vs resident warps and independent chains per warp, and a
// concurrent DMMA + DFMA mix where both kinds run for the whole kernel (time-bounded loops).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_mma(double *x, int n) {
  double a = x[threadIdx.x] + 1e-3, b = x[threadIdx.x + 64] + 1e-3, d[CH][2];
  for (int j = 0; j < CH; ++j) d[j][0] = d[j][1] = x[j];
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int j = 0; j < CH; ++j) s += d[j][0] + d[j][1];
  if (s == 1.2345) x[0] = s;
}
// warps with (w % R) == 0 run DMMA (4 chains), the others DFMA (ILP 8); each warp counts its own
// iterations until a clock deadline, so both kinds run concurrently the whole time
__global__ void k_mix(double *x, unsigned long long *cnt, long long cycles, int R) {
  const int w = threadIdx.x >> 5;
  const bool mma = (w % R) == 0;
  double a = x[threadIdx.x] + 1e-3, b = x[threadIdx.x + 64] + 1e-3, acc[8];
  for (int j = 0; j < 8; ++j) acc[j] = x[j];
  const long long t0 = clock64();
  unsigned long long it = 0;
  if (mma) {
    while (clock64() - t0 < cycles) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[2 * j]), "+d"(acc[2 * j + 1]) : "d"(a), "d"(b));
      it += 32;  // DMMAs
    }
  } else {
    while (clock64() - t0 < cycles) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fma(acc[j], a, b);
      it += 64;  // DFMA warp instructions
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 1.2345) x[0] = s;
  if ((threadIdx.x & 31) == 0) atomicAdd(cnt + (mma ? 0 : 1), it);
}
template <int CH>
void run(double *x, int warps, cudaEvent_t e0, cudaEvent_t e1) {
  const int n = 4000;
  k_mma<CH><<<148, warps * 32>>>(x, 10);
  cudaEventRecord(e0);
  k_mma<CH><<<148, warps * 32>>>(x, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmma = 148.0 * warps * CH * n;
  printf("warps/SM %2d chains %d: %.2f T FMA/s, %.1f cycles per DMMA per SMSP\n", warps, CH, dmma * 256 / ms / 1e9,
         ms * 1e-3 * 1.92e9 / (dmma / 148 / 4));
}
int main() {
  double *x;
  unsigned long long *cnt;
  cudaMalloc(&x, 1 << 20);
  cudaMemset(x, 0, 1 << 20);
  cudaMalloc(&cnt, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w : {4, 8, 16, 32}) {
    run<1>(x, w, e0, e1);
    run<2>(x, w, e0, e1);
    run<4>(x, w, e0, e1);
    run<8>(x, w, e0, e1);
  }
  for (int R : {1, 2, 4, 8, 1000}) {
    cudaMemset(cnt, 0, 16);
    const long long cyc = 20000000;
    k_mix<<<148, 512>>>(x, cnt, cyc, R);
    cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, cnt, 16, cudaMemcpyDeviceToHost);
    const double sec = cyc / 1.92e9;  // approximate (SM clock)
    const double f1 = h[0] * 256.0 / sec / 1e12, f2 = h[1] * 32.0 / sec / 1e12;
    printf("mix 1/%d warps DMMA: DMMA %.1f T FMA/s (%.0f%% of 18.6) + DFMA %.1f T FMA/s (%.0f%% of 16.7) = %.0f%% pipe\n",
           R, f1, 100 * f1 / 18.6, f2, 100 * f2 / 16.7, 100 * (f1 / 18.6 + f2 / 16.7));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
