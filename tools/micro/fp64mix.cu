// FP64 instruction throughput per op (DFMA / DADD / DMUL / DFMA with a uniform-register
// operand), 16 warps per SM x 148 SMs, ILP 8.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double *x, double c, int n) {
  double a[8], b = x[threadIdx.x];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = x[threadIdx.x + j];
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = fma(a[j], b, 1e-9);
      if (OP == 1) a[j] = a[j] + b;
      if (OP == 2) a[j] = a[j] * b;
      if (OP == 3) a[j] = fma(a[j], c, b);
    }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0) x[0] = s;
}
int main() {
  double *x; cudaMalloc(&x, 1 << 20); cudaMemset(x, 0, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *nm[] = {"DFMA R,R,imm", "DADD", "DMUL", "DFMA R,UR(param),R"};
  int n = 20000;
  for (int op = 0; op < 4; ++op) {
    auto f = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
    f<<<148, 512>>>(x, 1.0000001, 100);
    cudaEventRecord(e0);
    f<<<148, 512>>>(x, 1.0000001, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * 512 * 8 * n;
    printf("%-20s %.2f T thread-ops/s = %.1f per clk per SM at 1.965 GHz\n", nm[op], ops / ms / 1e9, ops / ms / 1e9 * 1e12 / 148 / 1.965e9 / 1e12 * 1e12 / 1e12);
  }
}
