// Cost of partial-sector writes on HBM: full zero vs the "column face" zero pattern of the Q6
// grid (every row y % 6 == 0 entirely, else every 6th double) vs storing 5 of every 6 doubles.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_full(double *x, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) x[i] = 0.0;
}
// rows of nx doubles; row r = i / nx
__global__ void k_faces(double *x, long nrows, long nx) {
  const long per = (nx + 5) / 6;  // face elements of a strided row
  for (long r = blockIdx.x; r < nrows; r += gridDim.x) {
    double *row = x + r * nx;
    if (r % 6 == 0) {
      for (long i = threadIdx.x; i < nx; i += blockDim.x) row[i] = 0.0;
    } else {
      for (long j = threadIdx.x; j < per; j += blockDim.x) row[6 * j] = 0.0;
    }
  }
}
__global__ void k_interior(double *x, long n) {  // 5 of every 6
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    if (i % 6) x[i] = 1.0;
}
int main() {
  const long nx = 1537, nrows = 1537L * 1537;  // one Q6 256^3 vector: 3.63 G doubles
  const long n = nx * nrows;
  double *x;
  if (cudaMalloc(&x, n * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); k_full<<<148 * 8, 512>>>(x, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("full zero      %.2f ms (%.2f TB/s)\n", ms, n * 8 / ms / 1e9);
    cudaEventRecord(a); k_faces<<<148 * 16, 256>>>(x, nrows, nx); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("face pattern   %.2f ms\n", ms);
    cudaEventRecord(a); k_interior<<<148 * 8, 512>>>(x, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("5 of 6 stores  %.2f ms\n", ms);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
