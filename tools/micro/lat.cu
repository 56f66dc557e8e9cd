// Latency / throughput microbenchmarks on one SM: dependent DFMA / DADD chains, LDS.64, SHFL,
// mbarrier arrive->wait round trip.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double *x, long long *cyc, int n) {
  double a = x[threadIdx.x], b = x[threadIdx.x + 32], c = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, c, b); a = fma(a, c, b); a = fma(a, c, b); a = fma(a, c, b); }
  long long t1 = clock64();
  x[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dadd_chain(double *x, long long *cyc, int n) {
  double a = x[threadIdx.x], b = x[threadIdx.x + 32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + b; a = a - b; a = a + b; a = a - b; }
  long long t1 = clock64();
  x[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int ILP>
__global__ void dfma_tput(double *x, long long *cyc, int n) {
  double a[ILP], c = 1.0000001, b = x[threadIdx.x];
  for (int j = 0; j < ILP; ++j) a[j] = x[threadIdx.x + j];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) a[j] = fma(a[j], c, b);
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int j = 0; j < ILP; ++j) s += a[j];
  x[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lds_chain(double *x, long long *cyc, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = (int)sm[j];
  long long t1 = clock64();
  x[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_chain(double *x, long long *cyc, int n) {
  double a = x[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_up_sync(~0u, a, 1) + 1.0;
  long long t1 = clock64();
  x[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *x; long long *c, h; cudaMalloc(&x, 1 << 20); cudaMemset(x, 0, 1 << 20); cudaMalloc(&c, 64);
  int n = 4096;
  dfma_chain<<<1, 32>>>(x, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  dadd_chain<<<1, 32>>>(x, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  for (int w : {1, 2, 4, 8, 16, 32}) {
    dfma_tput<4><<<1, 32 * w>>>(x, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA ILP4 x %2d warps: %.2f warp-instr/clk/SM\n", w, 4.0 * n * w / (double)h);
    dfma_tput<8><<<1, 32 * w>>>(x, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA ILP8 x %2d warps: %.2f warp-instr/clk/SM\n", w, 8.0 * n * w / (double)h);
  }
  lds_chain<<<1, 32>>>(x, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 dependent (+F2I) latency: %.2f cycles\n", (double)h / n);
  shfl_chain<<<1, 32>>>(x, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("SHFL.64 + DADD dependent latency: %.2f cycles\n", (double)h / n);
}
