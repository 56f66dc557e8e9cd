// kernels_vec.cu -- vector kernels of the solver (§8(a) a10): fills, dot
// products (fixed block count + deterministic second pass), the CG and
// Chebyshev recurrences of S:500-508 / S:648-656, and the plane add of the
// halo exchange (§8(a) a8).  All FP64, grid-stride loops sized in multiples
// of the 148 SMs.
#include "internal.h"

namespace mf {

static unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

__global__ void k_zero(double *x, int64_t n) {
  // a dependent apply kernel may start its gather now (it waits for this grid before writing)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = 0.0;
}

cudaError_t launch_zero(double *x, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_zero<<<grid_for(n), 256, 0, s>>>(x, n);
  return cudaGetLastError();
}

// splitmix64 of (first_global + i + 2^40 seed) -> uniform [-1,1)  (R8; same
// counter generator as synth/, implemented here independently)
__global__ void k_splitmix(double *x, int64_t n, int64_t first, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)(first + i) + (seed << 40) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i] = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
  }
}

cudaError_t launch_splitmix(double *x, int64_t n, int64_t first_global, uint64_t seed, cudaStream_t s,
                            int64_t *launches) {
  ++*launches;
  k_splitmix<<<grid_for(n), 256, 0, s>>>(x, n, first_global, seed);
  return cudaGetLastError();
}

struct DotArgs {
  const double *a[3];
  const double *b[3];
};

// Dot products in ONE pass (fixed block count kDotBlocks, grid-stride): each block sums its
// products (per-thread FMA, then a warp / block tree), writes its partial, and the last block
// to finish (atomic ticket) adds the partials in block order and stores the result -- a
// deterministic order, no second launch.  The same tail finishes the fused update kernels.
template <int ND>
__device__ __forceinline__ void dot_finish(const double (&acc)[ND], double *partials, unsigned *ticket, double *out) {
  __shared__ double red[ND][8];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    double v = acc[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[j][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < ND) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[threadIdx.x][w];
    partials[threadIdx.x * kDotBlocks + blockIdx.x] = s;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (wid < ND) {
    double s = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(partials + wid * kDotBlocks + b);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[wid] = s;
  }
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch (stream order)
}

template <int ND>
__global__ void __launch_bounds__(256) k_dot(DotArgs args, int64_t n, double *partials, unsigned *ticket,
                                             double *out) {
  double acc[ND];
#pragma unroll
  for (int j = 0; j < ND; ++j) acc[j] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int j = 0; j < ND; ++j) acc[j] = fma(args.a[j][i], args.b[j][i], acc[j]);
  }
  dot_finish<ND>(acc, partials, ticket, out);
}

cudaError_t launch_dots(int nd, const double *const *a, const double *const *b, int64_t n, double *partials,
                        unsigned *ticket, double *out, cudaStream_t s, int64_t *launches) {
  DotArgs args{};
  for (int j = 0; j < nd; ++j) {
    args.a[j] = a[j];
    args.b[j] = b[j];
  }
  ++*launches;
  if (nd == 1) k_dot<1><<<kDotBlocks, 256, 0, s>>>(args, n, partials, ticket, out);
  else if (nd == 2) k_dot<2><<<kDotBlocks, 256, 0, s>>>(args, n, partials, ticket, out);
  else k_dot<3><<<kDotBlocks, 256, 0, s>>>(args, n, partials, ticket, out);
  return cudaGetLastError();
}

// CG update with the step length on the device: alpha = sc[rz] / sc[pv];
// x += alpha p, r -= alpha v, and rr = r.r over the owned prefix, in one pass
__global__ void __launch_bounds__(256) k_cg_xr_rr(const double *__restrict__ rz, const double *__restrict__ pv,
                                                  double *__restrict__ x, double *__restrict__ r,
                                                  const double *__restrict__ p, const double *__restrict__ v,
                                                  int64_t n, int64_t n_owned, double *partials, unsigned *ticket,
                                                  double *rr) {
  const double alpha = rz[0] / pv[0];
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, v[i], r[i]);
    r[i] = ri;
    if (i < n_owned) acc[0] = fma(ri, ri, acc[0]);
  }
  dot_finish<1>(acc, partials, ticket, rr);
}

cudaError_t launch_cg_xr_rr(const double *rz, const double *pv, double *x, double *r, const double *p,
                            const double *v, int64_t n, int64_t n_owned, double *partials, unsigned *ticket,
                            double *rr, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_cg_xr_rr<<<kDotBlocks, 256, 0, s>>>(rz, pv, x, r, p, v, n, n_owned, partials, ticket, rr);
  return cudaGetLastError();
}

// beta = rz_new / rz_old on the device; p = z + beta p
__global__ void k_cg_p_dev(const double *__restrict__ rz_new, const double *__restrict__ rz_old,
                           const double *__restrict__ z, double *__restrict__ p, int64_t n) {
  const double b = rz_new[0] / rz_old[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(b, p[i], z[i]);
}

cudaError_t launch_cg_p_dev(const double *rz_new, const double *rz_old, const double *z, double *p, int64_t n,
                            cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_cg_p_dev<<<grid_for(n), 256, 0, s>>>(rz_new, rz_old, z, p, n);
  return cudaGetLastError();
}

__global__ void k_axpby(double a, const double *__restrict__ x, double b, double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

cudaError_t launch_axpby(double a, const double *x, double b, double *y, int64_t n, cudaStream_t s,
                         int64_t *launches) {
  ++*launches;
  k_axpby<<<grid_for(n), 256, 0, s>>>(a, x, b, y, n);
  return cudaGetLastError();
}

// three-term form of the same Chebyshev step (S:648-656 with d_{k-1} = x_k - x_{k-1}):
// x_{k+1} = x_k + c1 (x_k - x_{k-1}) + c2 dinv (r - ax), written over x_{k-1} (xp; null: x_{k-1}
// = 0, the first step from x_0 = 0); no separate direction vector, 48 instead of 56 bytes per
// DoF.  With rz: r . x_{k+1} over the owned prefix (the CG's r.z, last step).
template <bool RZ>
__global__ void __launch_bounds__(256) k_cheb3(const double *__restrict__ r, const double *__restrict__ ax,
                                               const double *__restrict__ dinv, double c1, double c2,
                                               const double *__restrict__ x, double *xp, int64_t n, int64_t n_owned,
                                               bool first, double *partials, unsigned *ticket, double *rz) {
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i], xi = x[i];
    const double dk = first ? xi : xi - xp[i];
    const double xn = xi + (c1 * dk + c2 * (dinv[i] * (ri - ax[i])));
    xp[i] = xn;
    if (RZ && i < n_owned) acc[0] = fma(ri, xn, acc[0]);
  }
  if constexpr (RZ) dot_finish<1>(acc, partials, ticket, rz);
}

cudaError_t launch_cheb3(const double *r, const double *ax, const double *dinv, double c1, double c2,
                         const double *x, double *xp, bool first, int64_t n, int64_t n_owned, double *partials,
                         unsigned *ticket, double *rz, cudaStream_t s, int64_t *launches) {
  ++*launches;
  if (rz)
    k_cheb3<true><<<kDotBlocks, 256, 0, s>>>(r, ax, dinv, c1, c2, x, xp, n, n_owned, first, partials, ticket, rz);
  else
    k_cheb3<false><<<grid_for(n), 256, 0, s>>>(r, ax, dinv, c1, c2, x, xp, n, n_owned, first, nullptr, nullptr,
                                                nullptr);
  return cudaGetLastError();
}

// x = c0 dinv r (the Chebyshev start, x_0 = 0)
__global__ void k_cheb_init1(const double *__restrict__ r, const double *__restrict__ dinv, double c0,
                             double *__restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = r[i] * dinv[i] * c0;
}

cudaError_t launch_cheb_init1(const double *r, const double *dinv, double c0, double *x, int64_t n, cudaStream_t s,
                              int64_t *launches) {
  ++*launches;
  k_cheb_init1<<<grid_for(n), 256, 0, s>>>(r, dinv, c0, x, n);
  return cudaGetLastError();
}

__global__ void k_mul(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ out,
                      int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

cudaError_t launch_mul(const double *a, const double *b, double *out, int64_t n, cudaStream_t s,
                       int64_t *launches) {
  ++*launches;
  k_mul<<<grid_for(n), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}

__global__ void k_recip(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = 1.0 / x[i];
}

cudaError_t launch_recip(const double *x, double *y, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_recip<<<grid_for(n), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

__global__ void k_plane_add(double *__restrict__ dst, const double *__restrict__ recv, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = dst[i] + recv[i];
}

cudaError_t launch_plane_add(double *dst, const double *recv, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_plane_add<<<grid_for(n), 256, 0, s>>>(dst, recv, n);
  return cudaGetLastError();
}

// ---- FP32 vector kernels of the mixed-precision multigrid (§8(f) f2) ----------
__global__ void k_zero_f(float *x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = 0.f;
}
cudaError_t launch_zero_f(float *x, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_zero_f<<<grid_for(n), 256, 0, s>>>(x, n);
  return cudaGetLastError();
}

__global__ void k_d2f(const double *__restrict__ x, float *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}
__global__ void k_f2d(const float *__restrict__ x, double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (double)x[i];
}
cudaError_t launch_d2f(const double *x, float *y, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_d2f<<<grid_for(n), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}
cudaError_t launch_f2d(const float *x, double *y, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_f2d<<<grid_for(n), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

__global__ void k_cheb_init_f(const float *__restrict__ r, const float *__restrict__ dinv, float c0,
                              float *__restrict__ x, float *__restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = r[i] * dinv[i] * c0;
    x[i] = v;
    d[i] = v;
  }
}
cudaError_t launch_cheb_init_f(const float *r, const float *dinv, float c0, float *x, float *d, int64_t n,
                               cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_cheb_init_f<<<grid_for(n), 256, 0, s>>>(r, dinv, c0, x, d, n);
  return cudaGetLastError();
}

__global__ void k_cheb_step_f(const float *__restrict__ r, const float *__restrict__ ax, const float *__restrict__ dinv,
                              float c1, float c2, float *__restrict__ x, float *__restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float dn = c1 * d[i] + c2 * (dinv[i] * (r[i] - ax[i]));
    d[i] = dn;
    x[i] += dn;
  }
}
cudaError_t launch_cheb_step_f(const float *r, const float *ax, const float *dinv, float c1, float c2, float *x,
                               float *d, int64_t n, cudaStream_t s, int64_t *launches) {
  ++*launches;
  k_cheb_step_f<<<grid_for(n), 256, 0, s>>>(r, ax, dinv, c1, c2, x, d, n);
  return cudaGetLastError();
}

}  // namespace mf
