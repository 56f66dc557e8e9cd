// microbench.cu -- B200 ceilings the roofline needs and the reference does not
// supply (SURVEY.md §8(d) "Prerequisite microbenchmarks"): sustained DFMA rate,
// DMMA (FP64 mma.sync m8n8k4) rate, shared-memory LDS.64 bandwidth, FP64
// global atomic (REDG) throughput and an HBM copy.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void k_dfma(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[2][2] = {{0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  if (c[0][0] + c[1][1] == 12345.678) out[0] = c[0][1];
}

__global__ void k_lds(double *out, int iters) {
  __shared__ double sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s += sm[(idx + j * 256) & 2047];
    idx = (idx + 32) & 2047;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_red(double *dst, long n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
      atomicAdd(dst + i, 1.0);
}

__global__ void k_copy(const double *__restrict__ a, double *__restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int lat_main();
int main(int argc, char **argv) {
  if (argc > 1) return lat_main();
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"mem_bytes\": %zu, \"clock_khz\": %d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor, p.totalGlobalMem, p.clockRate);
  double *buf;
  CK(cudaMalloc(&buf, 1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  float ms;
  // DFMA
  {
    const int iters = 20000, threads = 256, blocks = sms * 8;
    k_dfma<<<blocks, threads>>>(buf, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(buf, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 8;
    printf("{\"dfma_tflops\": %.3f, \"dfma_per_clk_per_sm_at_1965\": %.2f, \"ms\": %.3f}\n", 2 * fmas / ms / 1e9,
           fmas / (ms * 1e-3) / sms / 1.965e9, ms);
  }
  // DMMA
  {
    const int iters = 20000, threads = 256, blocks = sms * 8;
    k_dmma<<<blocks, threads>>>(buf, 100);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(buf, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * (threads / 32) * iters * 2 * (8 * 8 * 4 * 2);
    printf("{\"dmma_tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  // LDS.64
  {
    const int iters = 20000, threads = 256, blocks = sms * 8;
    k_lds<<<blocks, threads>>>(buf, 100);
    cudaEventRecord(e0);
    k_lds<<<blocks, threads>>>(buf, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)blocks * threads * iters * 8 * 8;
    printf("{\"lds64_tbps\": %.3f, \"bytes_per_clk_per_sm_at_1965\": %.1f}\n", bytes / ms / 1e9,
           bytes / (ms * 1e-3) / sms / 1.965e9);
  }
  // REDG f64 spread addresses
  {
    long n = 1 << 24;
    double *d;
    CK(cudaMalloc(&d, n * 8));
    cudaMemset(d, 0, n * 8);
    k_red<<<sms * 16, 256>>>(d, n, 1);
    cudaEventRecord(e0);
    k_red<<<sms * 16, 256>>>(d, n, 4);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"redg_f64_gops\": %.2f, \"n\": %ld}\n", 4.0 * n / ms / 1e6, n);
    cudaFree(d);
  }
  // HBM copy
  {
    long n = 1l << 28;  // 2 GiB per buffer
    double *a, *b;
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8));
    cudaMemset(a, 0, n * 8);
    k_copy<<<sms * 16, 256>>>(a, b, n);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      k_copy<<<sms * 16, 256>>>(a, b, n);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"copy_gbps\": %.1f}\n", 16.0 * n / best / 1e6);
  }
  return 0;
}

// ---- DFMA latency / ILP sweep: one warp per SM, `chains` independent dependent chains
template <int CH>
__global__ void k_dfma_lat(double *out, int iters, long long *cyc) {
  double x[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) x[j] = threadIdx.x * 1e-3 + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) x[j] = fma(x[j], 1.0000001, 1e-9);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int lat_main() {
  double *buf;
  long long *cyc, h;
  cudaMalloc(&buf, 1024);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
#define LAT(CH, W)                                                                                   \
  k_dfma_lat<CH><<<148, 32 * W>>>(buf, iters, cyc);                                                 \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                                    \
  printf("{\"dfma_chains\": %d, \"warps_per_sm\": %d, \"cycles_per_dfma_per_warp\": %.2f}\n", CH, W, \
         (double)h / iters / CH);
  LAT(1, 1) LAT(2, 1) LAT(4, 1) LAT(8, 1) LAT(1, 4) LAT(2, 4) LAT(4, 4) LAT(8, 4) LAT(2, 8) LAT(4, 8)
  return 0;
}
