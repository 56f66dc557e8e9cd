// kernels_dg.cu -- symmetric interior penalty DG Laplacian on a brick (SURVEY §8(f)
// f4; §6.1; R16-R18), matrix-free.
//
// On axis-aligned cells every face integral factors into a 1D point term times the
// tangential mass (Gauss(k+1) is exact for both), so the operator is a Kronecker sum
// (the Kronecker-sum identity is one of the DG pins under tests/):
//     A = B_x (x) M_y (x) M_z + M_x (x) B_y (x) M_z + M_x (x) M_y (x) B_z,
// B_e the 1D SIP matrix along e (cell stiffness + interior point terms + Nitsche
// boundary points) and M_e the block-diagonal 1D DG mass.  Per cell K and direction
// e, B_e couples K only with its two neighbours along e:
//     (B_e u)_K = B_self(K) u_K + B_left u_{K-e} + B_right u_{K+e}
// (B_self differs on boundary cells; B_left, B_right are rank-2 face couplings), so a
// block of cells computes, for each e, the 1D SIP along e-pencils (neighbour pencils
// read from global memory; DG DoFs are cell-major, so a neighbour's pencil is one
// contiguous or strided run inside its cell block), then the two tangential masses,
// and accumulates.  Every DoF belongs to one cell: plain stores, no atomics.
#include <cmath>
#include <cstring>

#include "internal.h"

namespace mf {

namespace {

// the 1D blocks of direction e: [0] self, interior cell; [1] self, lower boundary;
// [2] self, upper boundary; [3] self, both; [4] coupling to the lower neighbour;
// [5] coupling to the upper neighbour; M = tangential mass h_e M_ref
struct DGParams {
  double B[3][6][kMaxN][kMaxN];
  double M[3][kMaxN][kMaxN];
  int64_t nc[3];
};

template <int N>
__device__ __forceinline__ void mv(const double (&A)[kMaxN][kMaxN], const double *x, double *y) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = A[i][0] * x[0];
#pragma unroll
    for (int j = 1; j < N; ++j) s = fma(A[i][j], x[j], s);
    y[i] = s;
  }
}
template <int N>
__device__ __forceinline__ void mv_acc(const double (&A)[kMaxN][kMaxN], const double *x, double *y) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = y[i];
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(A[i][j], x[j], s);
    y[i] = s;
  }
}

// lexicographic slot of entry i of pencil p along direction e (x fastest)
template <int N>
__device__ __forceinline__ int slot(int e, int p, int i) {
  if (e == 0) return N * p + i;                          // p = y + N z
  if (e == 1) return (p % N) + N * i + N * N * (p / N);  // p = x + N z
  return p + N * N * i;                                  // p = x + N y
}

template <int K>
__global__ void __launch_bounds__(256) k_apply_dg(const __grid_constant__ DGParams D, const double *__restrict__ src,
                                                  double *__restrict__ dst, int cpb) {
  constexpr int N = K + 1, NP = N * N, NV = NP * N;
  extern __shared__ double sm[];
  const int64_t ncells = D.nc[0] * D.nc[1] * D.nc[2];
  const int cl = threadIdx.x / NP, p = threadIdx.x - cl * NP;
  const bool active = cl < cpb;
  const int64_t cell = (int64_t)blockIdx.x * cpb + cl;
  const bool valid = active && cell < ncells;
  // shared memory: the contiguous cells [cell0 - 1, cell0 + cpb] (own cells and their
  // x-neighbours, one coalesced load), then T and W per cell
  const int64_t cell0 = (int64_t)blockIdx.x * cpb;
  double *Ux = sm, *U = Ux + (cl + 1) * NV;
  double *T = sm + (cpb + 2) * NV + (active ? cl : 0) * 2 * NV, *W = T + NV;
  int64_t c[3] = {0, 0, 0};
  if (valid) {
    c[0] = cell % D.nc[0];
    const int64_t r = cell / D.nc[0];
    c[1] = r % D.nc[1];
    c[2] = r / D.nc[1];
  }
  const int64_t stride[3] = {1, D.nc[0], D.nc[0] * D.nc[1]};
  const double *uK = src + cell * NV;
  double a[N], b[N];
  {
    const int64_t g0 = (cell0 - 1) * NV, gend = ncells * NV;
    for (int idx = threadIdx.x; idx < (cpb + 2) * NV; idx += blockDim.x) {
      const int64_t gi = g0 + idx;
      if (gi >= 0 && gi < gend) Ux[idx] = __ldg(src + gi);
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    // 1D SIP along e-pencils, neighbours' pencils from global memory
    if (valid) {
      const bool lo = c[e] == 0, hi = c[e] == D.nc[e] - 1;
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = U[slot<N>(e, p, i)];
      mv<N>(D.B[e][(lo ? 1 : 0) + (hi ? 2 : 0)], a, b);
      if (!lo) {  // x: the previous cell is in shared memory
        const double *un = uK - stride[e] * NV;
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] = e == 0 ? U[slot<N>(e, p, i) - NV] : __ldg(un + slot<N>(e, p, i));
        mv_acc<N>(D.B[e][4], a, b);
      }
      if (!hi) {
        const double *un = uK + stride[e] * NV;
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] = e == 0 ? U[slot<N>(e, p, i) + NV] : __ldg(un + slot<N>(e, p, i));
        mv_acc<N>(D.B[e][5], a, b);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) T[slot<N>(e, p, i)] = b[i];
    }
    __syncthreads();
    // tangential masses: first along t1 (in place), then along t2 into the accumulator
    const int t1 = e == 0 ? 1 : 0, t2 = e == 2 ? 1 : 2;
    if (valid) {
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = T[slot<N>(t1, p, i)];
      mv<N>(D.M[t1], a, b);
#pragma unroll
      for (int i = 0; i < N; ++i) T[slot<N>(t1, p, i)] = b[i];
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = T[slot<N>(t2, p, i)];
      mv<N>(D.M[t2], a, b);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int s = slot<N>(t2, p, i);
        W[s] = e == 0 ? b[i] : W[s] + b[i];
      }
    }
    __syncthreads();
  }
  if (valid) {
#pragma unroll
    for (int i = 0; i < N; ++i) dst[cell * NV + N * p + i] = W[N * p + i];
  }
}

__global__ void k_diag_dg(const __grid_constant__ DGParams D, int N, double *__restrict__ diag) {
  const int64_t NV = (int64_t)N * N * N, ncells = D.nc[0] * D.nc[1] * D.nc[2];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ncells * NV;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / NV;
    const int loc = (int)(g - cell * NV);
    const int ix[3] = {loc % N, (loc / N) % N, loc / (N * N)};
    int64_t c[3];
    c[0] = cell % D.nc[0];
    c[1] = (cell / D.nc[0]) % D.nc[1];
    c[2] = cell / (D.nc[0] * D.nc[1]);
    double s = 0.0;
    for (int e = 0; e < 3; ++e) {
      const int sb = (c[e] == 0 ? 1 : 0) + (c[e] == D.nc[e] - 1 ? 2 : 0);
      double t = D.B[e][sb][ix[e]][ix[e]];
      for (int f = 0; f < 3; ++f)
        if (f != e) t *= D.M[f][ix[f]][ix[f]];
      s += t;
    }
    diag[g] = s;
  }
}

// l_j and l_j' at x by the product formula on the GLL nodes
double lag(const double *x, int k, int j, double t) {
  double v = 1.0;
  for (int m = 0; m <= k; ++m)
    if (m != j) v *= (t - x[m]) / (x[j] - x[m]);
  return v;
}
double lag_d(const double *x, int k, int j, double t) {
  double s = 0.0;
  for (int q = 0; q <= k; ++q) {
    if (q == j) continue;
    double v = 1.0 / (x[j] - x[q]);
    for (int m = 0; m <= k; ++m)
      if (m != j && m != q) v *= (t - x[m]) / (x[j] - x[m]);
    s += v;
  }
  return s;
}

// R17: sigma = 2 (k+1)^2 / h; all terms times the constant coefficient
void build_dg(const Geo &g, const Tables &t, DGParams *D) {
  std::memset(D, 0, sizeof(*D));
  const int k = g.k, N = k + 1;
  double v0[kMaxN], v1[kMaxN], d0[kMaxN], d1[kMaxN];
  for (int i = 0; i < N; ++i) {
    v0[i] = lag(t.gll, k, i, 0.0);
    v1[i] = lag(t.gll, k, i, 1.0);
    d0[i] = lag_d(t.gll, k, i, 0.0);
    d1[i] = lag_d(t.gll, k, i, 1.0);
  }
  for (int e = 0; e < 3; ++e) {
    D->nc[e] = g.nc[e];
    const double h = g.h[e], c = g.coeff, sig = 2.0 * N * N / h;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        D->M[e][i][j] = h * t.Mr[i][j];
        const double kc = t.Kr[i][j] / h;
        // the upper face as the '-' side (J = v1, {d} = d1 / 2h) and the lower face as the '+' side
        const double up = -v1[i] * 0.5 * d1[j] / h - 0.5 * d1[i] / h * v1[j] + sig * v1[i] * v1[j];
        const double lo = 0.5 * v0[i] * d0[j] / h + 0.5 * d0[i] / h * v0[j] + sig * v0[i] * v0[j];
        // Nitsche boundary points: lower (outward -x: D = -d0/h), upper (D = d1/h)
        const double blo = v0[i] * d0[j] / h + d0[i] / h * v0[j] + sig * v0[i] * v0[j];
        const double bup = -v1[i] * d1[j] / h - d1[i] / h * v1[j] + sig * v1[i] * v1[j];
        D->B[e][0][i][j] = c * (kc + lo + up);
        D->B[e][1][i][j] = c * (kc + blo + up);
        D->B[e][2][i][j] = c * (kc + lo + bup);
        D->B[e][3][i][j] = c * (kc + blo + bup);
        // couplings (test i of this cell, trial j of the neighbour)
        D->B[e][4][i][j] = c * (0.5 * v0[i] * d1[j] / h - 0.5 * d0[i] / h * v1[j] - sig * v0[i] * v1[j]);
        D->B[e][5][i][j] = c * (-v1[i] * 0.5 * d0[j] / h + 0.5 * d1[i] / h * v0[j] - sig * v1[i] * v0[j]);
      }
  }
}

template <int K>
cudaError_t launch_dg_t(const DGParams &D, const double *src, double *dst, cudaStream_t s) {
  constexpr int N = K + 1, NP = N * N, NV = NP * N;
  int cpb = 256 / NP;
  while (cpb > 1 && (3 * cpb + 2) * NV * 8 > 96 * 1024) --cpb;
  if (cpb < 1) cpb = 1;
  const size_t smem = (size_t)(3 * cpb + 2) * NV * sizeof(double);  // own + x-neighbour cells, T, W
  static bool attr = (cudaFuncSetAttribute(k_apply_dg<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
                      true);
  (void)attr;
  const int64_t ncells = D.nc[0] * D.nc[1] * D.nc[2];
  const int64_t blocks = (ncells + cpb - 1) / cpb;
  if (blocks == 0) return cudaSuccess;
  k_apply_dg<K><<<(unsigned)blocks, ((cpb * NP + 31) / 32) * 32, smem, s>>>(D, src, dst, cpb);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_apply_dg(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                            int64_t *launches) {
  DGParams D;
  build_dg(g, t, &D);
  ++*launches;
  switch (g.k) {
    case 1: return launch_dg_t<1>(D, src, dst, s);
    case 2: return launch_dg_t<2>(D, src, dst, s);
    case 3: return launch_dg_t<3>(D, src, dst, s);
    case 4: return launch_dg_t<4>(D, src, dst, s);
    case 5: return launch_dg_t<5>(D, src, dst, s);
    case 6: return launch_dg_t<6>(D, src, dst, s);
    case 7: return launch_dg_t<7>(D, src, dst, s);
    case 8: return launch_dg_t<8>(D, src, dst, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_diagonal_dg(const Geo &g, const Tables &t, double *diag, cudaStream_t s, int64_t *launches) {
  DGParams D;
  build_dg(g, t, &D);
  ++*launches;
  k_diag_dg<<<148 * 8, 256, 0, s>>>(D, g.k + 1, diag);
  return cudaGetLastError();
}

}  // namespace mf
