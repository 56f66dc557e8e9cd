// tile_common.cuh -- pieces shared by the Cartesian tile kernels (kernels_tile.cu,
// kernels_plane.cu): even-odd 1D products, the kernel parameter block, the init
// kernel for shared planes / Dirichlet rows, cp.async helper and host set-up.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace mf {

constexpr int kMaxH = 5;  // (kMaxN + 1) / 2

template <class T>
struct EOMatT {
  T E[kMaxH][kMaxH];  // even part (rows i < h, cols j < h; col m = middle for odd n)
  T O[kMaxH][kMaxH];  // odd part (rows/cols < n/2)
};
using EOMat = EOMatT<double>;

// sm_100 DFMA takes no constant-bank operand: coefficients live in the 64-entry
// uniform register file, so only two EO matrices are kept -- M and K = f_x K_ref --
// and Ky' = ry K, Kz' = rz K are applied by scaling the data (ry = rz = 1 on
// cubes, where the ISO template skips the scaling).
struct TileParams {
  EOMat M, K;
  double ry, rz;
  EOMatT<float> Mf, Kf;  // the same in FP32 (mixed-precision multigrid, §8(f) f2)
  float ryf, rzf;
  int64_t Nx, Ny, Nz;  // local node counts
  int ncx, ncy, ncz;   // local cell counts
  int ntx, nty, nch, LZ;
  // z-split (multi-GPU overlap): chunk 0 = cell layer 0, chunk nch-1 = layer ncz-1, the
  // interior layers in chunks of LZ; pass 1 = the two boundary chunks, pass 2 = the rest
  // (pass 0 = every chunk).  Without zsplit chunk c = layers [c LZ, (c+1) LZ).
  int zsplit, pass;
  // pass 3 (layer range, the pipelined host apply): only cell layers [zr_lo, zr_hi), in
  // chunks of LZ; planes shared with the neighbouring ranges take atomics
  int zr_lo, zr_hi, lo_shared, hi_shared;
  uint32_t dirichlet;
  int skip_top_identity;
  unsigned long long *prof;  // debug counters [2][8] or null
};

// ---- even-odd 1D products --------------------------------------------------
template <int N>
struct EO {
  static constexpr int m = N / 2, h = (N + 1) / 2;
};

// the coefficient set of scalar type T
template <class T>
__device__ __forceinline__ const EOMatT<T> &tp_M(const TileParams &P);
template <>
__device__ __forceinline__ const EOMatT<double> &tp_M<double>(const TileParams &P) { return P.M; }
template <>
__device__ __forceinline__ const EOMatT<float> &tp_M<float>(const TileParams &P) { return P.Mf; }
template <class T>
__device__ __forceinline__ const EOMatT<T> &tp_K(const TileParams &P);
template <>
__device__ __forceinline__ const EOMatT<double> &tp_K<double>(const TileParams &P) { return P.K; }
template <>
__device__ __forceinline__ const EOMatT<float> &tp_K<float>(const TileParams &P) { return P.Kf; }

template <int N, class T>
__device__ __forceinline__ void eo_split(const T *u, T *e, T *o) {
  constexpr int m = N / 2;
#pragma unroll
  for (int j = 0; j < m; ++j) {
    e[j] = u[j] + u[N - 1 - j];
    o[j] = u[j] - u[N - 1 - j];
  }
  if (N & 1) e[m] = u[m];
}

// ve += E e, vo += O o
template <int N, class T>
__device__ __forceinline__ void eo_acc(const EOMatT<T> &A, const T *e, const T *o, T *ve, T *vo) {
  constexpr int m = N / 2, h = (N + 1) / 2;
#pragma unroll
  for (int i = 0; i < h; ++i)
#pragma unroll
    for (int j = 0; j < h; ++j) ve[i] = fma(A.E[i][j], e[j], ve[i]);
#pragma unroll
  for (int i = 0; i < m; ++i)
#pragma unroll
    for (int j = 0; j < m; ++j) vo[i] = fma(A.O[i][j], o[j], vo[i]);
}

template <int N, class T>
__device__ __forceinline__ void eo_first(const EOMatT<T> &A, const T *e, const T *o, T *ve, T *vo) {
  constexpr int m = N / 2, h = (N + 1) / 2;
#pragma unroll
  for (int i = 0; i < h; ++i) {
    ve[i] = A.E[i][0] * e[0];
#pragma unroll
    for (int j = 1; j < h; ++j) ve[i] = fma(A.E[i][j], e[j], ve[i]);
  }
#pragma unroll
  for (int i = 0; i < m; ++i) {
    vo[i] = A.O[i][0] * o[0];
#pragma unroll
    for (int j = 1; j < m; ++j) vo[i] = fma(A.O[i][j], o[j], vo[i]);
  }
}

template <int N, class T>
__device__ __forceinline__ void eo_combine(const T *ve, const T *vo, T *v) {
  constexpr int m = N / 2;
#pragma unroll
  for (int i = 0; i < m; ++i) {
    v[i] = ve[i] + vo[i];
    v[N - 1 - i] = ve[i] - vo[i];
  }
  if (N & 1) v[m] = ve[m];
}


// ---- init: shared-edge / chunk-plane nodes and Dirichlet rows ---------------
// dst = src on constrained nodes (except the top plane of a non-last slab),
// 0 on every other node that several blocks add into.  The planes are given as
// arithmetic families (axis, first coordinate, stride, count).
struct PlaneSet {
  int axis[12], count[12];
  int64_t c0[12], stride[12], lines[12];  // lines = count x lines per plane
  int64_t total_lines;
  int nfam;
  int gz_lo, gz_hi;  // the node planes the x- and y-plane families cover (a layer range)
};

template <class T>
static __global__ void __launch_bounds__(256) k_tile_init(const __grid_constant__ TileParams P,
                                                           const __grid_constant__ PlaneSet ps,
                                                           const T *__restrict__ src, T *__restrict__ dst) {
  // the apply kernel that follows may start now (programmatic dependent launch): it reads
  // src and builds its first faces, and waits for this grid before its first dst write
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // one warp per line of a plane (x-plane: line gz, nodes gy; y-plane: line gz,
  // nodes gx; z-plane: line gy, nodes gx), warps grid-stride over all lines
  const int Nx = (int)P.Nx, Ny = (int)P.Ny, Nz = (int)P.Nz;
  const uint32_t d = P.dirichlet;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int64_t L = warp; L < ps.total_lines; L += nwarps) {
    int f = 0;
    int64_t l = L;
    while (f < ps.nfam - 1 && l >= ps.lines[f]) l -= ps.lines[f++];
    const int axis = ps.axis[f];
    const int nlines = axis == 2 ? Ny : ps.gz_hi - ps.gz_lo + 1, nnodes = axis == 0 ? Ny : Nx;
    const int pl = (int)(l / nlines), line = (int)(l - (int64_t)pl * nlines) + (axis == 2 ? 0 : ps.gz_lo);
    const int c = (int)(ps.c0[f] + ps.stride[f] * pl);
    if (sizeof(T) == 8 && axis == 0 && c >= 4 && c + 4 < Nx && ((reinterpret_cast<uintptr_t>(dst) & 31) == 0)) {
      // strided x-plane nodes: write the whole aligned 32-byte sector around each
      // node instead of 8 bytes of it (no partial-sector writes).  The sector
      // stays inside the row, off the x faces (4 <= c < Nx - 4); its other nodes are
      // owned by one block, which overwrites them later, so they get the value every
      // writer agrees on (the identity on constrained nodes, else 0).  (Extending this
      // to the x faces themselves measured slower: 21.9 vs 18.3 us on cfg 3.)
      for (int a = lane; a < nnodes; a += 32) {
        const int64_t row = ((int64_t)line * Ny + a) * Nx;
        const int64_t g0 = (row + c) & ~(int64_t)3;
        const bool ycons = ((d & 4u) && a == 0) || ((d & 8u) && a == Ny - 1) || ((d & 16u) && line == 0) ||
                           ((d & 32u) && line == Nz - 1);
        const bool ident = ycons && !(P.skip_top_identity && line == Nz - 1);
        T v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = ident ? __ldg(src + g0 + q) : T(0);
        double2 *p = reinterpret_cast<double2 *>(dst + g0);
        p[0] = make_double2((double)v[0], (double)v[1]);
        p[1] = make_double2((double)v[2], (double)v[3]);
      }
      continue;
    }
    // 8 nodes per lane per round, all identity loads issued before the stores (a Dirichlet
    // line is a chain of dependent load -> store pairs otherwise)
    for (int a0 = lane; a0 < nnodes; a0 += 256) {
      T v[8];
      int64_t gis[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int a = a0 + 32 * j;
        const int gx = axis == 0 ? c : a, gy = axis == 0 ? a : (axis == 1 ? c : line), gz = axis == 2 ? c : line;
        const bool cons = ((d & 1u) && gx == 0) || ((d & 2u) && gx == Nx - 1) || ((d & 4u) && gy == 0) ||
                          ((d & 8u) && gy == Ny - 1) || ((d & 16u) && gz == 0) || ((d & 32u) && gz == Nz - 1);
        gis[j] = ((int64_t)gz * Ny + gy) * Nx + gx;
        const bool ident = a < nnodes && cons && !(P.skip_top_identity && gz == Nz - 1);
        v[j] = ident ? __ldg(src + gis[j]) : T(0);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (a0 + 32 * j < nnodes) dst[gis[j]] = v[j];
    }
  }
}

// 8-byte cp.async global -> shared; src_bytes = 0 writes zeros without reading
__device__ __forceinline__ void cp_async8z(double *smem, const double *gmem, unsigned src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes) : "memory");
}
// sizeof(T)-byte cp.async; `ok` false writes zeros without reading
template <class T>
__device__ __forceinline__ void cp_async_z(T *smem, const T *gmem, unsigned src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes ? 4u : 0u)
                 : "memory");
}
// predicated reduction (at != 0) or plain store, no divergent branch
__device__ __forceinline__ void red_or_st(double *p, double v, int at) {
  asm volatile(
      "{\n .reg .pred pa;\n setp.ne.s32 pa, %2, 0;\n"
      " @pa red.global.add.f64 [%0], %1;\n @!pa st.global.f64 [%0], %1;\n}\n" ::"l"(p),
      "d"(v), "r"(at)
      : "memory");
}
__device__ __forceinline__ void red_or_st(float *p, float v, int at) {
  asm volatile(
      "{\n .reg .pred pa;\n setp.ne.s32 pa, %2, 0;\n"
      " @pa red.global.add.f32 [%0], %1;\n @!pa st.global.f32 [%0], %1;\n}\n" ::"l"(p),
      "f"(v), "r"(at)
      : "memory");
}

// ---- host side -------------------------------------------------------------------
static inline void to_eo(int n, const double A[kMaxN][kMaxN], EOMat *out) {
  std::memset(out, 0, sizeof(EOMat));
  const int m = n / 2, h = (n + 1) / 2;
  for (int i = 0; i < h; ++i) {
    for (int j = 0; j < m; ++j) out->E[i][j] = 0.5 * (A[i][j] + A[i][n - 1 - j]);
    if (n & 1) out->E[i][m] = A[i][m];
  }
  // the middle row of an odd n: v[m] = sum_{j<m} A[m][j] e[j] + A[m][m] u[m] (e unhalved)
  if (n & 1)
    for (int j = 0; j < m; ++j) out->E[m][j] = A[m][j];
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) out->O[i][j] = 0.5 * (A[i][j] - A[i][n - 1 - j]);
}

// 1D reference mass M = S^T W S and stiffness K_ref = D^T W D from the tables
// (Gauss(k+1) integrates both exactly), then P.M = EO(M), P.K = EO(f_x K_ref),
// ry = f_y / f_x, rz = f_z / f_x, and the mesh sizes.
static inline void tile_params_common(const Geo &g, const Tables &t, int TX, int TY, TileParams *P) {
  const int N = g.k + 1;
  std::memset(P, 0, sizeof(*P));
  double M[kMaxN][kMaxN] = {}, Kx[kMaxN][kMaxN] = {};
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      long double mm = 0, kk = 0;
      for (int q = 0; q < N; ++q) {
        mm += (long double)t.w[q] * t.S[q][i] * t.S[q][j];
        kk += (long double)t.w[q] * t.D[q][i] * t.D[q][j];
      }
      M[i][j] = (double)mm;
      Kx[i][j] = (double)(g.fcart[0] * kk);
    }
  to_eo(N, M, &P->M);
  to_eo(N, Kx, &P->K);
  for (int i = 0; i < kMaxH; ++i)
    for (int j = 0; j < kMaxH; ++j) {
      P->Mf.E[i][j] = (float)P->M.E[i][j];
      P->Mf.O[i][j] = (float)P->M.O[i][j];
      P->Kf.E[i][j] = (float)P->K.E[i][j];
      P->Kf.O[i][j] = (float)P->K.O[i][j];
    }
  P->ry = g.fcart[1] / g.fcart[0];
  P->rz = g.fcart[2] / g.fcart[0];
  P->ryf = (float)P->ry;
  P->rzf = (float)P->rz;
  P->Nx = g.N[0];
  P->Ny = g.N[1];
  P->Nz = g.N[2];
  P->ncx = (int)g.nc[0];
  P->ncy = (int)g.nc[1];
  P->ncz = (int)g.nc[2];
  P->ntx = (P->ncx + TX - 1) / TX;
  P->nty = (P->ncy + TY - 1) / TY;
  P->dirichlet = g.dirichlet;
  P->skip_top_identity = g.skip_top_identity;
}

// z-chunk length balancing the (tile, chunk) items against the resident-block slots
static inline void tile_choose_chunks(TileParams *P, int slots, double per_chunk_overhead) {
  const int tiles = P->ntx * P->nty;
  int best_nch = 1;
  double best = 1e30;
  for (int nch = 1; nch <= P->ncz; ++nch) {
    const int LZ = (P->ncz + nch - 1) / nch;
    const int real_nch = (P->ncz + LZ - 1) / LZ;
    const double waves = std::ceil((double)tiles * real_nch / slots);
    const double cost = waves * (LZ + per_chunk_overhead);
    if (cost < best - 1e-9) {
      best = cost;
      best_nch = real_nch;
    }
  }
  P->LZ = (P->ncz + best_nch - 1) / best_nch;
  P->nch = (P->ncz + P->LZ - 1) / P->LZ;
}

// the z-split chunking: boundary layers alone, the ncz - 2 interior layers balanced
static inline void tile_choose_chunks_split(TileParams *P, int slots, double per_chunk_overhead) {
  P->zsplit = 1;
  if (P->ncz <= 2) {
    P->LZ = 1;
    P->nch = P->ncz;  // one or two boundary chunks, no interior
    return;
  }
  TileParams Q = *P;
  Q.ncz = P->ncz - 2;
  tile_choose_chunks(&Q, slots, per_chunk_overhead);
  P->LZ = Q.LZ;
  P->nch = Q.nch + 2;
}

// items (tile, chunk) of a pass, and the chunk's cell layers
__host__ __device__ inline int tile_pass_chunks(const TileParams &P) {
  if (P.pass == 0 || P.pass == 3) return P.nch;
  if (P.pass == 1) return P.nch >= 2 ? 2 : 1;
  return P.nch > 2 ? P.nch - 2 : 0;
}
__host__ __device__ inline int tile_pass_chunk(const TileParams &P, int j) {
  if (P.pass == 0 || P.pass == 3) return j;
  if (P.pass == 1) return j == 0 ? 0 : P.nch - 1;
  return 1 + j;
}
__host__ __device__ inline void tile_chunk_layers(const TileParams &P, int c, int &b, int &e) {
  if (P.pass == 3) {
    b = P.zr_lo + c * P.LZ;
    e = b + P.LZ < P.zr_hi ? b + P.LZ : P.zr_hi;
  } else if (!P.zsplit) {
    b = c * P.LZ;
    e = b + P.LZ < P.ncz ? b + P.LZ : P.ncz;
  } else if (c == 0) {
    b = 0;
    e = 1;
  } else if (c == P.nch - 1) {
    b = P.ncz - 1;
    e = P.ncz;
  } else {
    b = 1 + (c - 1) * P.LZ;
    e = b + P.LZ < P.ncz - 1 ? b + P.LZ : P.ncz - 1;
  }
}

// init kernel: planes shared between blocks (internal tile edges, chunk planes)
// get 0, Dirichlet faces get the identity value
template <class T>
static inline cudaError_t tile_launch_init(const TileParams &P, const Geo &g, int K, int TX, int TY,
                                           const T *src, T *dst, cudaStream_t s, int64_t *launches) {
  PlaneSet ps;
  std::memset(&ps, 0, sizeof(ps));
  // the node planes this launch owns: all, or for a layer range (pass 3) the planes of
  // its layers except the bottom one when the range below already initialised it
  const bool range = P.pass == 3;
  ps.gz_lo = range ? K * P.zr_lo + (P.lo_shared ? 1 : 0) : 0;
  ps.gz_hi = range ? K * P.zr_hi : (int)P.Nz - 1;
  const int nzl = ps.gz_hi - ps.gz_lo + 1;
  int total = 0;
  auto fam = [&](int axis, int64_t c0, int64_t stride, int count) {
    if (count <= 0) return;
    ps.axis[ps.nfam] = axis;
    ps.c0[ps.nfam] = c0;
    ps.stride[ps.nfam] = stride;
    ps.count[ps.nfam] = count;
    ps.lines[ps.nfam++] = (int64_t)count * (axis == 2 ? P.Ny : nzl);
    total += count;
  };
  fam(0, (int64_t)K * TX, (int64_t)K * TX, P.ntx - 1);
  fam(1, (int64_t)K * TY, (int64_t)K * TY, P.nty - 1);
  if (range) {  // chunk planes inside the range, and its top plane if a range above shares it
    fam(2, (int64_t)K * (P.zr_lo + P.LZ), (int64_t)K * P.LZ, P.nch - 1);
    if (P.hi_shared) fam(2, (int64_t)K * P.zr_hi, 1, 1);
  } else if (!P.zsplit) {
    fam(2, (int64_t)K * P.LZ, (int64_t)K * P.LZ, P.nch - 1);
  } else if (P.nch >= 2) {  // bottom planes of chunks 1 .. nch-1
    fam(2, (int64_t)K, (int64_t)K * P.LZ, P.nch - 2);
    fam(2, (int64_t)K * (P.ncz - 1), 1, 1);
  }
  if (g.dirichlet & 1u) fam(0, 0, 1, 1);
  if (g.dirichlet & 2u) fam(0, P.Nx - 1, 1, 1);
  if (g.dirichlet & 4u) fam(1, 0, 1, 1);
  if (g.dirichlet & 8u) fam(1, P.Ny - 1, 1, 1);
  if ((g.dirichlet & 16u) && (!range || P.zr_lo == 0)) fam(2, 0, 1, 1);
  if (((g.dirichlet & 32u) || g.skip_top_identity) && (!range || P.zr_hi == P.ncz)) fam(2, P.Nz - 1, 1, 1);
  if (total == 0) return cudaSuccess;
  ++*launches;
  for (int f = 0; f < ps.nfam; ++f) ps.total_lines += ps.lines[f];
  const int blocks = (int)std::min<int64_t>((ps.total_lines + 7) / 8, 148 * 8);
  k_tile_init<T><<<blocks, 256, 0, s>>>(P, ps, src, dst);
  return cudaGetLastError();
}

}  // namespace mf
