// Throughput of 8-byte-per-lane coalesced global->shared copies (cp.async LDGSTS) vs plain LDG
// (+ STS) vs LDG into registers, 16 warps/SM x 148 SMs, rows of 1 KB from a 512 MB buffer.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const double *__restrict__ src, double *out, long long n_rows, int iters) {
  __shared__ double st[13 * 256 * 2 - 1024];
  const int tid = threadIdx.x, t = tid & 255;
  double acc = 0;
  long long row = (long long)blockIdx.x * 13 + (tid >> 8) * 7;
  for (int it = 0; it < iters; ++it) {
    const double *s0 = src + ((row + (long long)it * 148 * 13) % (n_rows - 16)) * 256 + t;
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 13; ++i) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(&st[((i * 256 + t) * 2 + (tid >> 8)) % (13 * 512 - 1024)]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(s0 + i * 256) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 2;" ::: "memory");
      acc += st[t];
    } else if (MODE == 2) {  // 16 B per lane: lanes 0-15 row i, 16-31 row i+1 (two rows per instruction)
      const int l = tid & 31, wq = (tid >> 5) & 7;
#pragma unroll
      for (int i = 0; i < 13; i += 2) {
        const double *p = src + ((row + (long long)it * 148 * 13) % (n_rows - 16)) * 256 + (i + (l >> 4)) * 256 + wq * 32 + 2 * (l & 15);
        unsigned sa = (unsigned)__cvta_generic_to_shared(&st[((i * 256 + wq * 32 + 2 * (l & 15)) * 2) % (13 * 512 - 1024)]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa & ~15u), "l"(p) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 2;" ::: "memory");
      acc += st[t];
    } else if (MODE == 1) {
      double v[13];
#pragma unroll
      for (int i = 0; i < 13; ++i) v[i] = __ldg(s0 + i * 256);
#pragma unroll
      for (int i = 0; i < 13; ++i) acc += v[i];
    }
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  const long long n_rows = (512ll << 20) / 2048;
  double *src, *out; cudaMalloc(&src, n_rows * 2048); cudaMemset(src, 0, n_rows * 2048); cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    f<<<148, 512>>>(src, out, n_rows, 10);
    cudaEventRecord(a);
    int iters = 2000;
    f<<<148, 512>>>(src, out, n_rows, iters);
    cudaEventRecord(b); cudaEventSynchronize(b); printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = 148.0 * 512 * 13 * 8 * iters;
    double instr = 148.0 * 16 * (mode == 2 ? 7 : 13) * iters;
    if (mode == 2) bytes = 148.0 * 512 * 14 * 8 * iters;
    printf("%s: %.2f TB/s, %.1f cycles per warp-instruction per SM\n", mode == 0 ? "cp.async 8B " : mode == 1 ? "LDG 8B      " : "cp.async 16B",
           bytes / ms / 1e9, ms * 1e-3 * 1.965e9 / (instr / 148));
  }
}
