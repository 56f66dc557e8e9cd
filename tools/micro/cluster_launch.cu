// Per-CTA start / end times (globaltimer) of a grid with and without thread-block clusters:
// does a cluster launch stagger the CTAs?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void k(unsigned long long *t, long long spin_ns) {
  extern __shared__ double sm[];
  unsigned long long a, b;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  sm[threadIdx.x] = threadIdx.x;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b)); } while ((long long)(b - a) < spin_ns);
  __syncthreads();
  if (threadIdx.x == 0) { int id = blockIdx.x + gridDim.x * blockIdx.y; t[2 * id] = a; t[2 * id + 1] = b; }
}
int main() {
  int n = 128; size_t smem = 143 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long *d; cudaMalloc(&d, 2 * 8 * 1024);
  for (int clu : {0, 1, 2, 4, 8}) for (int thr : {256, 512}) for (int smk : {64, 143}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(clu ? clu : 2, n / (clu ? clu : 2)); cfg.blockDim = dim3(thr);
    cfg.dynamicSmemBytes = smk * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = clu; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = clu ? 1 : 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, 50000LL);
      cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); continue; }
    }
    std::vector<unsigned long long> h(2 * n); cudaMemcpy(h.data(), d, 16 * n, cudaMemcpyDeviceToHost);
    unsigned long long s0 = ~0ull, s1 = 0, e1 = 0;
    for (int i = 0; i < n; ++i) { s0 = std::min(s0, h[2*i]); s1 = std::max(s1, h[2*i]); e1 = std::max(e1, h[2*i+1]); }
    printf("cluster %d threads %d smem %dK: start spread %.1f us, total %.1f us (spin 50 us)\n", clu, thr, smk, (s1 - s0) / 1e3, (e1 - s0) / 1e3);
  }
}
