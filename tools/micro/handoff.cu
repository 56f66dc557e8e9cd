// Warp-to-warp hand-off round trip (ping-pong between warp 0 and warp 1 of one CTA) through
// an mbarrier (try_wait loop / test_wait loop / try_wait + nanosleep) and named barriers.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(unsigned a) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory"); }
template <int MODE>
__device__ __forceinline__ void wait(unsigned a, unsigned par) {
  if (MODE == 0) {
    asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" ::"r"(a), "r"(par) : "memory");
  } else if (MODE == 1) {
    asm volatile("{ .reg .pred p; W%=: mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" ::"r"(a), "r"(par) : "memory");
  } else {
    while (true) {
      unsigned ok;
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(a), "r"(par) : "memory");
      if (ok) break;
      __nanosleep(MODE == 2 ? 32 : 256);
    }
  }
}
template <int MODE>
__global__ void k(long long *out, int n) {
  __shared__ __align__(8) unsigned long long b[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&b[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&b[1])));
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (w == 0) {
      __syncwarp(); if (lane == 0) arrive(sa(&b[0]));
      wait<MODE>(sa(&b[1]), i & 1);
    } else if (w == 1) {
      wait<MODE>(sa(&b[0]), i & 1);
      __syncwarp(); if (lane == 0) arrive(sa(&b[1]));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void knamed(long long *out, int n) {
  const int w = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (w == 0) { asm volatile("bar.arrive 1, 64;" ::: "memory"); asm volatile("bar.sync 2, 64;" ::: "memory"); }
    else if (w == 1) { asm volatile("bar.sync 1, 64;" ::: "memory"); asm volatile("bar.arrive 2, 64;" ::: "memory"); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long *d, h; cudaMalloc(&d, 8); int n = 20000;
  const char *nm[] = {"try_wait loop", "test_wait loop", "try_wait+nanosleep(32)", "try_wait+nanosleep(256)"};
  for (int busy : {0, 14}) {
    int th = 64 + 32 * busy;
    k<0><<<1, th>>>(d, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%s (%d warps): %.0f cycles/round trip\n", nm[0], th / 32, (double)h / n);
    k<1><<<1, th>>>(d, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%s (%d warps): %.0f cycles/round trip\n", nm[1], th / 32, (double)h / n);
    k<2><<<1, th>>>(d, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%s (%d warps): %.0f cycles/round trip\n", nm[2], th / 32, (double)h / n);
    k<3><<<1, th>>>(d, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%s (%d warps): %.0f cycles/round trip\n", nm[3], th / 32, (double)h / n);
    knamed<<<1, th>>>(d, n); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("named bar.arrive/bar.sync (%d warps): %.0f cycles/round trip\n", th / 32, (double)h / n);
  }
}
