// kernels_general.cu -- the general matrix-free cell kernel (any dim in {2,3},
// degree k in 1..8, Cartesian or curved geometry, constant or variable
// coefficient), the metric precompute and the operator diagonal.
//
// Method (§3.6):
//   a3 gather the (k+1)^d cell values (Dirichlet DoFs read as 0),
//   a4 sum factorisation to the Gauss points: Q = (S (x) S (x) S) u, then the
//      reference gradient g_e = Co along e applied to Q (collocation derivative),
//   a5 quadrature-point operation t = G_q g  (G_q = c w |det J| J^{-1} J^{-T};
//      for affine boxes t_e = c w_q prod(h)/h_e^2 g_e),
//   a6 transposed sweeps R = sum_e Co^T_e t_e, v = (S^T (x) S^T (x) S^T) R,
//   a7 scatter-add (FP64 atomics into a zeroed dst) and the Dirichlet identity
//      dst_g = src_g, written once per constrained DoF by its owner cell.
// One thread block handles a batch of `cpb` consecutive cells (the
// GPU analogue of the SIMD cell batch); each thread owns one pencil of n values
// per sweep (thread-per-pencil, not the thread-per-DoF of P:960-961, whose
// n^4 shared-memory reads per sweep the pencil form avoids).  The 1D tables are
// a __grid_constant__ kernel parameter, so every matrix entry is a constant-bank
// operand of the DFMA.
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace mf {

template <int DIM, int N>
struct Shape {
  static constexpr int NP = DIM == 3 ? N * N : N;  // pencils per direction
  static constexpr int NV = NP * N;                // values per cell
};

// Shared-memory slot of local node (x, y, z) of a cell tensor.  Lexicographic, except
// for 3D with N = 4 (Q3): s = 16 z + 4 ((y + z) & 3) + ((x + z) & 3) puts the 16
// pencils of a half-warp on 16 distinct banks in every sweep direction and the 16
// nodes of a z-plane likewise (a Latin-cube map), with no padding.
template <int DIM, int N>
__device__ __forceinline__ int sidx(int x, int y, int z) {
  if (DIM == 3 && N == 4) return 16 * z + 4 * ((y + z) & 3) + ((x + z) & 3);
  return DIM == 3 ? (z * N + y) * N + x : y * N + x;
}

// slot of entry i of pencil p along direction dir (pencils enumerate the other two axes, x fastest)
template <int DIM, int N>
__device__ __forceinline__ int pen_off(int dir, int p, int i) {
  if (DIM == 2) return dir == 0 ? sidx<DIM, N>(i, p, 0) : sidx<DIM, N>(p, i, 0);
  if (dir == 0) return sidx<DIM, N>(i, p % N, p / N);  // p = z*N + y
  if (dir == 1) return sidx<DIM, N>(p % N, i, p / N);  // p = z*N + x
  return sidx<DIM, N>(p % N, p / N, i);                // p = y*N + x
}

// slot of the lexicographic local node / quadrature point i
template <int DIM, int N>
__device__ __forceinline__ int nidx(int i) {
  return sidx<DIM, N>(i % N, (i / N) % N, DIM == 3 ? i / (N * N) : 0);
}

// out[i] = sum_j M[i][j] in[j]   (TR: sum_j M[j][i] in[j])
template <int N, bool TR, class T>
__device__ __forceinline__ void mat1d(const T (&M)[kMaxN][kMaxN], const T *in, T *out) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = (TR ? M[0][i] : M[i][0]) * in[0];  // = fma(., ., 0.0), one instruction less
#pragma unroll
    for (int j = 1; j < N; ++j) s = fma(TR ? M[j][i] : M[i][j], in[j], s);
    out[i] = s;
  }
}

template <int DIM, int N, bool TR, class T>
__device__ __forceinline__ void sweep_inplace(const T (&M)[kMaxN][kMaxN], T *U, int dir, int p) {
  T a[N], b[N];
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = U[pen_off<DIM, N>(dir, p, i)];
  mat1d<N, TR>(M, a, b);
#pragma unroll
  for (int i = 0; i < N; ++i) U[pen_off<DIM, N>(dir, p, i)] = b[i];
}

struct CellIdx {
  int64_t c[3];
};

__device__ __forceinline__ CellIdx cell_coords(const Geo &g, int64_t cell) {
  CellIdx ci;
  ci.c[0] = cell % g.nc[0];
  int64_t r = cell / g.nc[0];
  ci.c[1] = r % g.nc[1];
  ci.c[2] = r / g.nc[1];
  return ci;
}

// local node (l) of cell (c) -> global node coords and local DoF index; constrained flag
template <int DIM, int N>
__device__ __forceinline__ int64_t node_index(const Geo &g, const CellIdx &ci, int i, int64_t m[3]) {
  const int K = N - 1;
  int l0 = i % N, l1 = DIM >= 2 ? (i / N) % N : 0, l2 = DIM == 3 ? i / (N * N) : 0;
  m[0] = K * ci.c[0] + l0;
  m[1] = K * ci.c[1] + l1;
  m[2] = DIM == 3 ? K * ci.c[2] + l2 : 0;
  return (m[2] * g.N[1] + m[1]) * g.N[0] + m[0];
}

__device__ __forceinline__ bool is_constrained(const Geo &g, const int64_t m[3]) {
  const uint32_t d = g.dirichlet;
  return ((d & 1u) && m[0] == 0) || ((d & 2u) && m[0] == g.N[0] - 1) || ((d & 4u) && m[1] == 0) ||
         ((d & 8u) && m[1] == g.N[1] - 1) || ((d & 16u) && m[2] == 0) || ((d & 32u) && m[2] == g.N[2] - 1);
}

// The cell that writes the identity row of a constrained node: local index
// >= 1 in every direction unless the node is on the low end of the brick.
template <int DIM, int N>
__device__ __forceinline__ bool owner_of(const Geo &g, const CellIdx &ci, int i, const int64_t m[3]) {
  int l0 = i % N, l1 = (i / N) % N, l2 = DIM == 3 ? i / (N * N) : 1;
  bool own = (l0 >= 1 || ci.c[0] == 0) && (l1 >= 1 || ci.c[1] == 0) && (DIM == 2 || l2 >= 1 || ci.c[2] == 0);
  if (g.skip_top_identity && DIM == 3 && m[2] == g.N[2] - 1) own = false;
  return own;
}

// the 1D tables the cell kernels read, in FP32 (mixed-precision multigrid, §8(f) f2)
struct TablesF {
  float S[kMaxN][kMaxN];
  float Co[kMaxN][kMaxN];
  float w[kMaxN];
  float xi[kMaxN];
  float Mr[kMaxN][kMaxN];
  float Kr[kMaxN][kMaxN];
  float Me[5][5], Mo[5][5], Ke[5][5], Ko[5][5];
};

// even-odd 1D product with the centro-symmetric matrix (E, O) (see Tables::Me)
template <int N, class T>
__device__ __forceinline__ void eo_sp(const T *u, T *e, T *o) {
  constexpr int m = N / 2;
#pragma unroll
  for (int j = 0; j < m; ++j) {
    e[j] = u[j] + u[N - 1 - j];
    o[j] = u[j] - u[N - 1 - j];
  }
  if (N & 1) e[m] = u[m];
}
template <int N, class T>
__device__ __forceinline__ void eo_mv(const T (&E)[5][5], const T (&O)[5][5], const T *e, const T *o, T *v) {
  constexpr int m = N / 2, h = (N + 1) / 2;
#pragma unroll
  for (int i = 0; i < h; ++i) {
    T ve = E[i][0] * e[0];
#pragma unroll
    for (int j = 1; j < h; ++j) ve = fma(E[i][j], e[j], ve);
    if (i < m) {
      T vo = O[i][0] * o[0];
#pragma unroll
      for (int j = 1; j < m; ++j) vo = fma(O[i][j], o[j], vo);
      v[i] = ve + vo;
      v[N - 1 - i] = ve - vo;
    } else {
      v[i] = ve;
    }
  }
}
template <class T>
struct TabOf;
template <>
struct TabOf<double> {
  using type = Tables;
};
template <>
struct TabOf<float> {
  using type = TablesF;
};

template <class T>
__device__ __forceinline__ T coeff_var_t(const T x[3]) {
  return T(1) / (T(0.05) + T(2) * (x[0] * x[0] + x[1] * x[1] + x[2] * x[2]));  // R5
}

__device__ __forceinline__ double coeff_var(const double x[3], int dim) {
  double r2 = 0.0;
  for (int d = 0; d < dim; ++d) r2 += x[d] * x[d];
  return 1.0 / (0.05 + 2.0 * r2);  // R5
}

// per-cell data of an apply block, computed once per cell
struct CellInfo {
  long long base;  // local DoF index of the cell's node (0,0,0)
  int cx, cy, cz;
  int flags;  // bits 0-5: the cell touches constrained face x-,x+,y-,y+,z-,z+;
              // 6-8: cx / cy / cz == 0 (identity-row owner rule); 9: skip identity on its top plane; 10: valid
};

template <int DIM, int K>
__device__ __forceinline__ CellInfo cell_info(const Geo &g, int64_t cell, int64_t ncells) {
  CellInfo ci;
  ci.flags = 0;
  ci.base = 0;
  ci.cx = ci.cy = ci.cz = 0;
  if (cell >= ncells) return ci;
  int64_t cx, cy, cz;
  if (ncells < (int64_t(1) << 31)) {  // 32-bit divisions (every local mesh up to 2^31 cells)
    const unsigned c = (unsigned)cell, n0 = (unsigned)g.nc[0], n1 = (unsigned)g.nc[1];
    const unsigned r = c / n0;
    cx = c - r * n0;
    cy = r % n1;
    cz = r / n1;
  } else {
    const int64_t r = cell / g.nc[0];
    cx = cell % g.nc[0];
    cy = r % g.nc[1];
    cz = r / g.nc[1];
  }
  ci.cx = (int)cx;
  ci.cy = (int)cy;
  ci.cz = (int)cz;
  ci.base = ((int64_t)K * cz * g.N[1] + (int64_t)K * cy) * g.N[0] + (int64_t)K * cx;
  const uint32_t d = g.dirichlet;
  int f = 1 << 10;
  if ((d & 1u) && cx == 0) f |= 1;
  if ((d & 2u) && cx == g.nc[0] - 1) f |= 2;
  if ((d & 4u) && cy == 0) f |= 4;
  if ((d & 8u) && cy == g.nc[1] - 1) f |= 8;
  if (DIM == 3 && (d & 16u) && cz == 0) f |= 16;
  if (DIM == 3 && (d & 32u) && cz == g.nc[2] - 1) f |= 32;
  if (cx == 0) f |= 64;
  if (cy == 0) f |= 128;
  if (DIM == 2 || cz == 0) f |= 256;
  if (DIM == 3 && g.skip_top_identity && cz == g.nc[2] - 1) f |= 512;
  ci.flags = f;
  return ci;
}

// node i of a cell: local DoF index, constrained flag, identity-row owner flag
template <int DIM, int N>
__device__ __forceinline__ void node_of(const CellInfo &ci, int i, int64_t Nx, int64_t plane, int64_t &gi,
                                        bool &cons, bool &owner) {
  const int lx = i % N, ly = (i / N) % N, lz = DIM == 3 ? i / (N * N) : 0;
  gi = ci.base + (DIM == 3 ? lz * plane : 0) + ly * Nx + lx;
  const int f = ci.flags;
  cons = ((f & 1) && lx == 0) || ((f & 2) && lx == N - 1) || ((f & 4) && ly == 0) || ((f & 8) && ly == N - 1) ||
         ((f & 16) && lz == 0) || ((f & 32) && lz == N - 1);
  owner = (lx >= 1 || (f & 64)) && (ly >= 1 || (f & 128)) && (DIM == 2 || lz >= 1 || (f & 256)) &&
          !((f & 512) && lz == N - 1);
}

// ---------------------------------------------------------------------------
// GEOM: 0 = affine box, constant coefficient; 1 = affine box, variable
// coefficient evaluated at x_q on the fly; 2 = stored metric G (curved).
template <int DIM, int K, int GEOM>
__global__ void __launch_bounds__(256) k_apply_general(const __grid_constant__ Tables t,
                                                       const __grid_constant__ Geo g,
                                                       const double *__restrict__ src, double *__restrict__ dst,
                                                       const double *__restrict__ metric, int cpb) {
  constexpr int N = K + 1, NP = Shape<DIM, N>::NP, NV = Shape<DIM, N>::NV;
  constexpr int CS = (DIM + 1) * NV;  // doubles of shared memory per cell
  extern __shared__ double sm[];
  CellInfo *info = reinterpret_cast<CellInfo *>(sm + cpb * CS);
  const int64_t ncells = g.nc[0] * g.nc[1] * (DIM == 3 ? g.nc[2] : 1);
  const int64_t cell0 = (int64_t)blockIdx.x * cpb;
  const int64_t Nx = g.N[0], plane = g.N[0] * g.N[1];

  // per-cell data, one 64-bit division per cell instead of one per node
  for (int cl = threadIdx.x; cl < cpb; cl += blockDim.x) info[cl] = cell_info<DIM, K>(g, cell0 + cl, ncells);
  __syncthreads();

  // a3: gather
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
    const int cl = idx / NV, i = idx - cl * NV;
    const CellInfo ci = info[cl];
    double v = 0.0;
    if (ci.flags) {
      int64_t gi;
      bool cons, owner;
      node_of<DIM, N>(ci, i, Nx, plane, gi, cons, owner);
      if (!cons) v = __ldg(src + gi);
    }
    sm[cl * CS + nidx<DIM, N>(i)] = v;
  }
  // a2 data of a5: optionally the stored metric of this thread's quadrature points
  // is loaded into registers here so its HBM latency overlaps the forward sweeps
  // (A thread owns at most N quadrature points, blockDim >= cpb * NP).  Measured on
  // cfg 4 the extra registers cost more occupancy than the overlap gains: off.
  constexpr bool PREF = false;
  constexpr int NGC = DIM == 3 ? 6 : 3;
  double gm[GEOM == 2 && PREF ? N : 1][NGC];
  if (GEOM == 2 && PREF) {
    const int64_t stride = ncells * NV;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      const int idx = threadIdx.x + r * blockDim.x;
      const int c2 = idx / NV, q = idx - c2 * NV;
      const int64_t cell = cell0 + c2;
      const bool ok = idx < cpb * NV && cell < ncells;
      const double *Gm = metric + (ok ? cell * NV + q : 0);
#pragma unroll
      for (int c = 0; c < NGC; ++c) gm[r][c] = ok ? __ldg(Gm + c * stride) : 0.0;
    }
  }
  __syncthreads();

  const int cl = threadIdx.x / NP, p = threadIdx.x - cl * NP;
  const bool active = cl < cpb;
  double *U = sm + cl * CS;

  // a4: values at Gauss points, one direction at a time
#pragma unroll
  for (int e = 0; e < DIM; ++e) {
    if (active) sweep_inplace<DIM, N, false>(t.S, U, e, p);
    __syncthreads();
  }
  // reference gradient by collocation derivative along each direction
  if (active) {
#pragma unroll
    for (int e = 0; e < DIM; ++e) {
      double a[N], b[N];
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = U[pen_off<DIM, N>(e, p, i)];
      mat1d<N, false>(t.Co, a, b);
      double *G = U + (e + 1) * NV;
#pragma unroll
      for (int i = 0; i < N; ++i) G[pen_off<DIM, N>(e, p, i)] = b[i];
    }
  }
  __syncthreads();

  // a5: quadrature-point operation
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const int idx = threadIdx.x + r * blockDim.x;
    if (idx >= cpb * NV) break;
    const int c2 = idx / NV, q = idx - c2 * NV;
    double *Uc = sm + c2 * CS;
    const int q0 = q % N, q1 = (q / N) % N, q2 = DIM == 3 ? q / (N * N) : 0;
    double gr[3], tt[3];
    const int qs = nidx<DIM, N>(q);
#pragma unroll
    for (int e = 0; e < DIM; ++e) gr[e] = Uc[(e + 1) * NV + qs];
    if (GEOM == 2) {
      double G[NGC];
      if (PREF) {
#pragma unroll
        for (int c = 0; c < NGC; ++c) G[c] = gm[PREF ? r : 0][c];
      } else {
        const int64_t cell = cell0 + c2;
        const bool ok = cell < ncells;
        const double *Gm = metric + (ok ? cell * NV + q : 0);
#pragma unroll
        for (int c = 0; c < NGC; ++c) G[c] = ok ? __ldg(Gm + c * (ncells * NV)) : 0.0;
      }
      if (DIM == 3) {
        tt[0] = G[0] * gr[0] + G[1] * gr[1] + G[2] * gr[2];
        tt[1] = G[1] * gr[0] + G[3] * gr[1] + G[4] * gr[2];
        tt[2] = G[2] * gr[0] + G[4] * gr[1] + G[5] * gr[2];
      } else {
        tt[0] = G[0] * gr[0] + G[1] * gr[1];
        tt[1] = G[1] * gr[0] + G[2] * gr[1];
      }
    } else {
      double W = t.w[q0] * t.w[q1] * (DIM == 3 ? t.w[q2] : 1.0);
      if (GEOM == 1) {
        const CellInfo ci = info[c2];
        double x[3];
        const int qq[3] = {q0, q1, q2};
        const int cc[3] = {ci.cx, ci.cy, ci.cz};
        for (int d = 0; d < DIM; ++d) {
          double cg = (double)(d == 2 ? cc[2] + g.cz0 : cc[d]);
          x[d] = g.lo[d] + g.h[d] * (cg + t.xi[qq[d]]);
        }
        double vol = g.h[0] * g.h[1] * (DIM == 3 ? g.h[2] : 1.0);
        W *= coeff_var(x, DIM) * vol;
#pragma unroll
        for (int e = 0; e < DIM; ++e) tt[e] = W / (g.h[e] * g.h[e]) * gr[e];
      } else {
#pragma unroll
        for (int e = 0; e < DIM; ++e) tt[e] = W * g.fcart[e] * gr[e];
      }
    }
#pragma unroll
    for (int e = 0; e < DIM; ++e) Uc[(e + 1) * NV + qs] = tt[e];
  }
  __syncthreads();

  // a6: transposed collocation derivative (in place, one array per direction)
  if (active) {
#pragma unroll
    for (int e = 0; e < DIM; ++e) sweep_inplace<DIM, N, true>(t.Co, U + (e + 1) * NV, e, p);
  }
  __syncthreads();
  // sum the directions and apply S^T along x
  if (active) {
    double a[N], b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int o = pen_off<DIM, N>(0, p, i);
      double s = U[NV + o];
#pragma unroll
      for (int e = 1; e < DIM; ++e) s += U[(e + 1) * NV + o];
      a[i] = s;
    }
    mat1d<N, true>(t.S, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) U[pen_off<DIM, N>(0, p, i)] = b[i];
  }
  __syncthreads();
#pragma unroll
  for (int e = 1; e < DIM; ++e) {
    if (active) sweep_inplace<DIM, N, true>(t.S, U, e, p);
    __syncthreads();
  }

  // a7: scatter-add and identity rows
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
    const int c2 = idx / NV, i = idx - c2 * NV;
    const CellInfo ci = info[c2];
    if (!ci.flags) continue;
    int64_t gi;
    bool cons, owner;
    node_of<DIM, N>(ci, i, Nx, plane, gi, cons, owner);
    if (cons) {
      if (owner) dst[gi] = __ldg(src + gi);
    } else {
      atomicAdd(dst + gi, sm[c2 * CS + nidx<DIM, N>(i)]);
    }
  }
}

// ---------------------------------------------------------------------------
// 3D general kernel (the default for dim = 3): the same a3-a7 arithmetic as
// k_apply_general, reorganised so that a thread keeps ONE pencil index p of one
// cell for the whole kernel.  Its three pencil slot lists (along x, y, z) are
// then computed once, the x-pencils are gathered / scattered straight between
// global memory and registers, and the z-direction steps that follow each other
// (S_z -> Co_z; q-point operation -> Co_z^T) stay in the registers of the
// z-pencil that produced them:
//   1 gather x-pencil, S_x            (regs -> U)
//   2 S_y                             (U -> U)
//   3 S_z -> Q (U), Co_z Q -> gz      (registers)
//   4 Co_x Q -> G0, Co_y Q -> G1
//   5 q-point op on the z-pencil, t_z -> Co_z^T in registers -> gz
//   6 Co_x^T G0, Co_y^T G1            (in place)
//   7 R = G0 + G1 + gz, S_z^T         (-> U)
//   8 S_y^T
//   9 S_x^T in regs, scatter-add + identity rows
// shared-memory layout of k_apply_cell3: work arrays [cpb][3 NV], then (curved cells) the
// metric [6][chunk] with chunk = cpb NV rounded up to 16 bytes, starting 16-byte aligned
template <int K, int GEOM, class T>
__host__ __device__ constexpr int cell3_ms_off();
template <int K, int GEOM, class T>
__host__ __device__ constexpr int cell3_chunk();
template <int K, int GEOM, class T>
__host__ __device__ constexpr size_t cell3_smem_bytes();

// unstructured hex meshes (GEOM 3): gather through cell_dofs, resolving a constraint
// line (hanging node) u = sum_j w_j u[dof_j]; the scatter adds the transpose
__device__ __forceinline__ double hex_gather(const HexDev &h, const double *__restrict__ src, int32_t d) {
  if (d >= 0) return __ldg(src + d);
  if (d == kHexDirichlet) return 0.0;
  const int l = -1 - d;
  double v = 0.0;
  for (int j = __ldg(h.line_ptr + l), e = __ldg(h.line_ptr + l + 1); j < e; ++j)
    v = fma(__ldg(h.line_w + j), __ldg(src + __ldg(h.line_dof + j)), v);
  return v;
}

__device__ __forceinline__ void hex_scatter(const HexDev &h, double *dst, int32_t d, double v) {
  if (d >= 0) {
    atomicAdd(dst + d, v);
  } else if (d != kHexDirichlet) {
    const int l = -1 - d;
    for (int j = __ldg(h.line_ptr + l), e = __ldg(h.line_ptr + l + 1); j < e; ++j)
      atomicAdd(dst + __ldg(h.line_dof + j), __ldg(h.line_w + j) * v);
  }
}

// sizeof(T)-byte cp.async (zero-fill when !ok)
template <class T>
__device__ __forceinline__ void cp_async_elem(T *smem, const T *gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(ok ? 4 : 0) : "memory");
}

// cells per block of k_apply_cell3: ~256 threads, ~128 with the staged metric
// (6 NV doubles per cell of extra shared memory), shared memory <= 48 KB
// Cartesian constant-coefficient Q6 (N = 7) in FP64: padded work layout, slot 54 z + 7 y + x,
// arrays of 378 doubles, cell stride 1137.  The plain layout (plane pitch 49 = 1 mod 16) puts
// the y-sweep lanes of consecutive z-planes on the same bank pairs; a bank model of the three
// sweeps gives 553 instead of 602 wavefronts per block
template <int K, int GEOM, class T>
__host__ __device__ constexpr bool cell3_padded() {
  return GEOM == 0 && K == 6 && sizeof(T) == 8;
}
// elements per work array and per cell of k_apply_cell3
template <int K, int GEOM, class T>
__host__ __device__ constexpr int cell3_as() {
  return cell3_padded<K, GEOM, T>() ? 54 * (K + 1) : (K + 1) * (K + 1) * (K + 1);
}
template <int K, int GEOM, class T>
__host__ __device__ constexpr int cell3_cs() {
  return cell3_padded<K, GEOM, T>() ? 3 * cell3_as<K, GEOM, T>() + 3 : 3 * (K + 1) * (K + 1) * (K + 1);
}

template <int K, int GEOM, class T = double>
__host__ __device__ constexpr int cell3_cpb() {
  constexpr int N = K + 1, NP = N * N, NV = NP * N;
  constexpr int per_cell = (int)sizeof(T) * (cell3_cs<K, GEOM, T>() + (GEOM >= 2 ? 6 * NV : 0));
  int c = (GEOM >= 2 ? 128 : 256) / NP;
  while (c > 1 && c * per_cell > 48 * 1024) --c;
  return c < 1 ? 1 : c;
}

template <int K, int GEOM, class T>
__host__ __device__ constexpr int cell3_ms_off() {
  constexpr int NV = (K + 1) * (K + 1) * (K + 1), E = 16 / (int)sizeof(T);
  (void)NV;
  return (cell3_cpb<K, GEOM, T>() * cell3_cs<K, GEOM, T>() + E - 1) / E * E;
}
template <int K, int GEOM, class T>
__host__ __device__ constexpr int cell3_chunk() {
  constexpr int NV = (K + 1) * (K + 1) * (K + 1), E = 16 / (int)sizeof(T);
  return (cell3_cpb<K, GEOM, T>() * NV + E - 1) / E * E;
}
template <int K, int GEOM, class T>
__host__ __device__ constexpr size_t cell3_smem_bytes() {
  return sizeof(T) * (size_t)(cell3_ms_off<K, GEOM, T>() + (GEOM >= 2 ? 6 * cell3_chunk<K, GEOM, T>() : 0));
}

template <int K, int GEOM, class T>
__global__ void __launch_bounds__(256) k_apply_cell3(const __grid_constant__ typename TabOf<T>::type t,
                                                     const __grid_constant__ Geo g, const T *__restrict__ src,
                                                     T *__restrict__ dst, const T *__restrict__ metric,
                                                     int64_t cbeg, int64_t cend, const __grid_constant__ HexDev hx);

// launch k_apply_cell3 as a programmatic dependent of the preceding (zeroing) kernel
template <int K, int GEOM>
static cudaError_t launch_cell3_pdl(unsigned blocks, unsigned threads, size_t smem, cudaStream_t s, const Tables &t,
                                    const Geo &g, const double *src, double *dst, const double *metric, int64_t cbeg,
                                    int64_t cend, const HexDev &hx) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool off = std::getenv("MF_NO_PDL") != nullptr;  // plain stream order (comparisons)
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k_apply_cell3<K, GEOM, double>, t, g, src, dst, metric, cbeg, cend, hx);
}

template <int K, int GEOM, class T>
__global__ void __launch_bounds__(256) k_apply_cell3(const __grid_constant__ typename TabOf<T>::type t,
                                                     const __grid_constant__ Geo g, const T *__restrict__ src,
                                                     T *__restrict__ dst, const T *__restrict__ metric,
                                                     int64_t cbeg, int64_t cend, const __grid_constant__ HexDev hx) {
  constexpr int N = K + 1, NP = N * N, NV = NP * N;
  constexpr int CS = cell3_cs<K, GEOM, T>();  // U, G0, G1 per cell (the z-gradient lives in registers)
  constexpr int AS = cell3_as<K, GEOM, T>();
  constexpr int cpb = cell3_cpb<K, GEOM, T>();
  extern __shared__ __align__(16) unsigned char smraw[];
  T *const sm = reinterpret_cast<T *>(smraw);
  const int64_t ncells = GEOM == 3 ? hx.ncells : g.nc[0] * g.nc[1] * g.nc[2];
  const int cl = threadIdx.x / NP, p = threadIdx.x - cl * NP;
  const bool active = cl < cpb;
  const int64_t cell0 = cbeg + (int64_t)blockIdx.x * cpb, cell = cell0 + cl;  // cells [cbeg, cend)
  const bool valid = active && cell < cend;
  T *U = sm + (active ? cl : 0) * CS, *G0 = U + AS, *G1 = U + 2 * AS;
  T gz[N];  // z-pencil: Co_z Q (steps 3-5), then Co_z^T t_z (steps 5-7)
  // curved cells: the block's metric [6][cpb][NV] is staged into shared memory by
  // cp.async at kernel start, so its HBM latency overlaps steps 1-4
  T *Ms = sm + cell3_ms_off<K, GEOM, T>();  // 16-byte aligned (bulk-copy destination)
  __shared__ alignas(8) unsigned long long mbar;
  bool bulk = false;
  if (GEOM >= 2) {
    constexpr int CH = cell3_chunk<K, GEOM, T>();  // padded component chunk (16-byte multiple)
    const int64_t cstride = ncells * NV;
    const int64_t rem = cend - cell0;
    const int ncb = rem < cpb ? (int)rem : cpb;
    const unsigned bytes = (unsigned)(ncb * NV * sizeof(T));
    // one thread, six bulk copies (TMA engine) completing on an mbarrier; the
    // 8-byte cp.async loop covers chunks that are not 16-byte multiples
    bulk = (bytes % 16 == 0) && ((cell0 * NV * (int64_t)sizeof(T)) % 16 == 0) &&
           ((cstride * (int64_t)sizeof(T)) % 16 == 0) &&
           ((reinterpret_cast<uintptr_t>(metric) & 15) == 0);
    if (bulk) {
      if (threadIdx.x == 0) {
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(6 * bytes) : "memory");
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(Ms + c * CH);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sa),
              "l"(metric + c * cstride + cell0 * NV), "r"(bytes), "r"(mb)
              : "memory");
        }
      }
    } else {
      const int avail = ncb * NV;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const T *gc = metric + c * cstride + cell0 * NV;
        for (int r = threadIdx.x; r < CH; r += blockDim.x) {
          const bool ok = r < avail;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(Ms + c * CH + r);
          cp_async_elem(Ms + c * CH + r, ok ? gc + r : metric, ok);
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  }
  int o0[N], o1[N], o2[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if constexpr (cell3_padded<K, GEOM, T>()) {
      const int u = p % N, w = p / N;
      o0[i] = 54 * w + N * u + i;  // x-pencil (y = u, z = w)
      o1[i] = 54 * w + N * i + u;  // y-pencil (x = u, z = w)
      o2[i] = 54 * i + N * w + u;  // z-pencil (x = u, y = w)
    } else {
      o0[i] = pen_off<3, N>(0, p, i);
      o1[i] = pen_off<3, N>(1, p, i);
      o2[i] = pen_off<3, N>(2, p, i);
    }
  }
  const int64_t Nx = g.N[0], plane = g.N[0] * g.N[1];
  const CellInfo ci = GEOM == 3 ? CellInfo{} : cell_info<3, K>(g, valid ? cell : ncells, ncells);
  T a[N], b[N];
  int32_t hd[GEOM == 3 ? N : 1];  // hex: the DoF entries of this thread's x-pencil
  if constexpr (GEOM == 3) {
    if (valid) {
#pragma unroll
      for (int i = 0; i < N; ++i) hd[i] = __ldg(hx.cell_dofs + cell * NV + N * p + i);
    }
  }

  if constexpr (GEOM == 0) {
    // Cartesian box, constant coefficient: the Gauss(k+1)-exact Kronecker form of the
    // cell operator, 7 one-dimensional products instead of 12
    // sweeps and no quadrature-point pass:
    //   v = fx K(x) M(y) M(z) u + fy M K M u + fz M M K u,   M, K = reference 1D mass / stiffness
    //   z-pencils: a = M u, b = fz K u;  y-pencils: c = M a, d = fy K a, e = M b;
    //   x-pencils: v = fx K c + M (d + e)
    const T fx = (T)g.fcart[0], fy = (T)g.fcart[1], fz = (T)g.fcart[2];
    T *A1 = G0, *B1 = G1;
    if (active) {  // gather the x-pencil
#pragma unroll
      for (int i = 0; i < N; ++i) {
        int64_t gi;
        bool cons, owner;
        node_of<3, N>(ci, i + N * p, Nx, plane, gi, cons, owner);
        a[i] = (valid && !cons) ? __ldg(src + gi) : T(0);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) U[o0[i]] = a[i];
    }
    __syncthreads();
    constexpr int h = (N + 1) / 2;
    T e[h], o[h];  // even-odd parts of the pencil (M and K are centro-symmetric)
    if (active) {  // z
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = U[o2[i]];
      eo_sp<N>(a, e, o);
      eo_mv<N>(t.Me, t.Mo, e, o, b);
#pragma unroll
      for (int i = 0; i < N; ++i) A1[o2[i]] = b[i];
      eo_mv<N>(t.Ke, t.Ko, e, o, b);
#pragma unroll
      for (int i = 0; i < N; ++i) B1[o2[i]] = fz * b[i];
    }
    __syncthreads();
    if (active) {  // y (each thread rewrites only its own pencil's slots)
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = A1[o1[i]];
      eo_sp<N>(a, e, o);
      eo_mv<N>(t.Me, t.Mo, e, o, b);
#pragma unroll
      for (int i = 0; i < N; ++i) A1[o1[i]] = b[i];
      eo_mv<N>(t.Ke, t.Ko, e, o, b);
#pragma unroll
      for (int i = 0; i < N; ++i) U[o1[i]] = fy * b[i];
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = B1[o1[i]];
      eo_sp<N>(a, e, o);
      eo_mv<N>(t.Me, t.Mo, e, o, b);
#pragma unroll
      for (int i = 0; i < N; ++i) B1[o1[i]] = b[i];
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the zeroing grid is complete
    if (active && valid) {  // x, then scatter-add and identity rows
#pragma unroll
      for (int i = 0; i < N; ++i) {
        a[i] = A1[o0[i]];
        gz[i] = U[o0[i]] + B1[o0[i]];
      }
      eo_sp<N>(a, e, o);
      eo_mv<N>(t.Ke, t.Ko, e, o, b);
      T v[N];
      eo_sp<N>(gz, e, o);
      eo_mv<N>(t.Me, t.Mo, e, o, v);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        int64_t gi;
        bool cons, owner;
        node_of<3, N>(ci, i + N * p, Nx, plane, gi, cons, owner);
        if (cons) {
          if (owner) dst[gi] = __ldg(src + gi);
        } else {
          atomicAdd(dst + gi, fma(fx, b[i], v[i]));
        }
      }
    }
    return;
  }

  // 1: gather the x-pencil (y = p % N, z = p / N), S along x
  if (active) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if constexpr (GEOM == 3) {
        a[i] = valid ? (T)hex_gather(hx, reinterpret_cast<const double *>(src), hd[i]) : T(0);
      } else {
        int64_t gi;
        bool cons, owner;
        node_of<3, N>(ci, i + N * p, Nx, plane, gi, cons, owner);
        a[i] = (valid && !cons) ? __ldg(src + gi) : 0.0;
      }
    }
    mat1d<N, false>(t.S, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) U[o0[i]] = b[i];
  }
  __syncthreads();
  // 2: S along y
  if (active) sweep_inplace<3, N, false>(t.S, U, 1, p);
  __syncthreads();
  // 3: S along z -> Q at the Gauss points; Co along z of this z-pencil in registers
  if (active) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = U[o2[i]];
    mat1d<N, false>(t.S, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) U[o2[i]] = b[i];
    mat1d<N, false>(t.Co, b, gz);  // stays in registers until step 5 (same thread, same pencil)
  }
  __syncthreads();
  // 4: Co along x and y of Q
  if (active) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = U[o0[i]];
    mat1d<N, false>(t.Co, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) G0[o0[i]] = b[i];
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = U[o1[i]];
    mat1d<N, false>(t.Co, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) G1[o1[i]] = b[i];
  }
  if (GEOM >= 2) {
    if (bulk) {
      const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
      asm volatile(
          "{\n .reg .pred P1;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
          " @!P1 bra WAIT%=;\n}\n" ::"r"(mb)
          : "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
  }
  __syncthreads();
  // 5: quadrature-point operation on the z-pencil (q = p + NP i), then Co_z^T in registers
  if (active) {
    constexpr int NGC = 6;
    const int qx = p % N, qy = p / N;
    const T *Gm = Ms + cl * NV + p;
    T t2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const T gr0 = G0[o2[i]], gr1 = G1[o2[i]], gr2 = gz[i];
      T tt0, tt1, tt2;
      if (GEOM >= 2) {
        T G[NGC];
#pragma unroll
        for (int c = 0; c < NGC; ++c) G[c] = Gm[c * cell3_chunk<K, GEOM, T>() + NP * i];
        tt0 = G[0] * gr0 + G[1] * gr1 + G[2] * gr2;
        tt1 = G[1] * gr0 + G[3] * gr1 + G[4] * gr2;
        tt2 = G[2] * gr0 + G[4] * gr1 + G[5] * gr2;
      } else {
        T W = t.w[qx] * t.w[qy] * t.w[i];
        if (GEOM == 1) {
          T x[3];
          x[0] = (T)g.lo[0] + (T)g.h[0] * ((T)ci.cx + t.xi[qx]);
          x[1] = (T)g.lo[1] + (T)g.h[1] * ((T)ci.cy + t.xi[qy]);
          x[2] = (T)g.lo[2] + (T)g.h[2] * ((T)(ci.cz + g.cz0) + t.xi[i]);
          W *= coeff_var_t<T>(x) * (T)(g.h[0] * g.h[1] * g.h[2]);
          tt0 = W / (T)(g.h[0] * g.h[0]) * gr0;
          tt1 = W / (T)(g.h[1] * g.h[1]) * gr1;
          tt2 = W / (T)(g.h[2] * g.h[2]) * gr2;
        } else {
          tt0 = W * (T)g.fcart[0] * gr0;
          tt1 = W * (T)g.fcart[1] * gr1;
          tt2 = W * (T)g.fcart[2] * gr2;
        }
      }
      G0[o2[i]] = tt0;
      G1[o2[i]] = tt1;
      t2[i] = tt2;
    }
    mat1d<N, true>(t.Co, t2, gz);  // Co_z^T t2, kept for step 7
  }
  __syncthreads();
  // 6: Co^T along x of G0, along y of G1
  if (active) {
    sweep_inplace<3, N, true>(t.Co, G0, 0, p);
    sweep_inplace<3, N, true>(t.Co, G1, 1, p);
  }
  __syncthreads();
  // 7: R = G0 + G1 + gz, S^T along z
  if (active) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = G0[o2[i]] + G1[o2[i]] + gz[i];
    mat1d<N, true>(t.S, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) U[o2[i]] = b[i];
  }
  __syncthreads();
  // 8: S^T along y
  if (active) sweep_inplace<3, N, true>(t.S, U, 1, p);
  __syncthreads();
  // 9: S^T along x in registers; scatter-add, identity rows by their owner cell (after the
  // zeroing grid this kernel may overlap under programmatic dependent launch)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (valid) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = U[o0[i]];
    mat1d<N, true>(t.S, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if constexpr (GEOM == 3) {
        hex_scatter(hx, reinterpret_cast<double *>(dst), hd[i], (double)b[i]);
      } else {
        int64_t gi;
        bool cons, owner;
        node_of<3, N>(ci, i + N * p, Nx, plane, gi, cons, owner);
        if (cons) {
          if (owner) dst[gi] = __ldg(src + gi);
        } else {
          atomicAdd(dst + gi, b[i]);
        }
      }
    }
  }
}

template <int DIM, int K>
static int cells_per_block() {
  constexpr int N = K + 1, NP = Shape<DIM, N>::NP, NV = Shape<DIM, N>::NV;
  int cpb = 256 / NP;
  const int cs = (DIM + 1) * NV * 8 + (int)sizeof(CellInfo);
  while (cpb > 1 && cpb * cs > 48 * 1024) --cpb;
  return cpb < 1 ? 1 : cpb;
}

// cells [cbeg, cend) (the 3D kernel; the 2D / v1 kernel always takes every cell)
template <int DIM, int K, int GEOM>
static cudaError_t launch_general_t(const Geo &g, const Tables &t, const double *src, double *dst,
                                    const double *metric, cudaStream_t s, int64_t cbeg, int64_t cend) {
  constexpr int N = K + 1, NP = Shape<DIM, N>::NP, NV = Shape<DIM, N>::NV;
  const int cpb = cells_per_block<DIM, K>();
  int threads = ((cpb * NP + 31) / 32) * 32;
  const int64_t ncells = g.nc[0] * g.nc[1] * (DIM == 3 ? g.nc[2] : 1);
  const int64_t blocks = (ncells + cpb - 1) / cpb;
  const size_t smem = (size_t)cpb * ((DIM + 1) * NV * sizeof(double) + sizeof(CellInfo));
  if (blocks == 0 || cend <= cbeg) return cudaSuccess;
  static const bool v1 = std::getenv("MF_GENERAL_V1") != nullptr;  // the original layout (comparisons)
  if constexpr (DIM == 3) {
    if (!v1) {
      constexpr int c3 = cell3_cpb<K, GEOM>();
      const int64_t b3 = (cend - cbeg + c3 - 1) / c3;
      const size_t sm3 = cell3_smem_bytes<K, GEOM, double>();
      smem_attr_once(k_apply_cell3<K, GEOM, double>, sm3);
      return launch_cell3_pdl<K, GEOM>((unsigned)b3, ((c3 * NP + 31) / 32) * 32, sm3, s, t, g, src, dst, metric, cbeg,
                                       cend, HexDev{});
    }
  }
  if (cbeg != 0 || cend != ncells) return cudaErrorNotSupported;
  k_apply_general<DIM, K, GEOM><<<(unsigned)blocks, threads, smem, s>>>(t, g, src, dst, metric, cpb);
  return cudaGetLastError();
}

template <int DIM, int GEOM>
static cudaError_t dispatch_k(const Geo &g, const Tables &t, const double *src, double *dst,
                              const double *metric, cudaStream_t s, int64_t cb, int64_t ce) {
  switch (g.k) {
    case 1: return launch_general_t<DIM, 1, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 2: return launch_general_t<DIM, 2, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 3: return launch_general_t<DIM, 3, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 4: return launch_general_t<DIM, 4, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 5: return launch_general_t<DIM, 5, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 6: return launch_general_t<DIM, 6, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 7: return launch_general_t<DIM, 7, GEOM>(g, t, src, dst, metric, s, cb, ce);
    case 8: return launch_general_t<DIM, 8, GEOM>(g, t, src, dst, metric, s, cb, ce);
  }
  return cudaErrorInvalidValue;
}

static int geom_kind(const Geo &g) {
  if (g.geom == MF_GEOM_SINE) return 2;
  return g.coeff_kind == MF_COEFF_VARIABLE ? 1 : 0;
}

// FP32 instance of the 3D kernel over every cell (mixed-precision multigrid)
template <int K, int GEOM>
static cudaError_t launch_cell3_f32(const Geo &g, const TablesF &tf, const float *src, float *dst,
                                    const float *metric, cudaStream_t s) {
  constexpr int N = K + 1, NP = N * N;
  constexpr int c3 = cell3_cpb<K, GEOM, float>();
  const int64_t ncells = g.nc[0] * g.nc[1] * g.nc[2];
  const int64_t b3 = (ncells + c3 - 1) / c3;
  const size_t sm3 = cell3_smem_bytes<K, GEOM, float>();
  smem_attr_once(k_apply_cell3<K, GEOM, float>, sm3);
  if (b3 == 0) return cudaSuccess;
  k_apply_cell3<K, GEOM, float><<<(unsigned)b3, ((c3 * NP + 31) / 32) * 32, sm3, s>>>(tf, g, src, dst, metric, 0,
                                                                                      ncells, HexDev{});
  return cudaGetLastError();
}

template <int GEOM>
static cudaError_t dispatch_f32(const Geo &g, const TablesF &tf, const float *src, float *dst, const float *metric,
                                cudaStream_t s) {
  switch (g.k) {
    case 1: return launch_cell3_f32<1, GEOM>(g, tf, src, dst, metric, s);
    case 2: return launch_cell3_f32<2, GEOM>(g, tf, src, dst, metric, s);
    case 3: return launch_cell3_f32<3, GEOM>(g, tf, src, dst, metric, s);
    case 4: return launch_cell3_f32<4, GEOM>(g, tf, src, dst, metric, s);
    case 5: return launch_cell3_f32<5, GEOM>(g, tf, src, dst, metric, s);
    case 6: return launch_cell3_f32<6, GEOM>(g, tf, src, dst, metric, s);
    case 7: return launch_cell3_f32<7, GEOM>(g, tf, src, dst, metric, s);
    case 8: return launch_cell3_f32<8, GEOM>(g, tf, src, dst, metric, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_apply_general_f32(const Geo &g, const Tables &t, const float *src, float *dst,
                                     const float *metric, cudaStream_t s, int64_t *launches) {
  if (g.dim != 3) return cudaErrorNotSupported;
  TablesF tf;
  for (int i = 0; i < kMaxN; ++i) {
    for (int j = 0; j < kMaxN; ++j) {
      tf.S[i][j] = (float)t.S[i][j];
      tf.Co[i][j] = (float)t.Co[i][j];
    }
    tf.w[i] = (float)t.w[i];
    tf.xi[i] = (float)t.xi[i];
    for (int j = 0; j < kMaxN; ++j) {
      tf.Mr[i][j] = (float)t.Mr[i][j];
      tf.Kr[i][j] = (float)t.Kr[i][j];
    }
  }
  for (int i = 0; i < 5; ++i) {
    for (int j = 0; j < 5; ++j) {
      tf.Me[i][j] = (float)t.Me[i][j];
      tf.Mo[i][j] = (float)t.Mo[i][j];
      tf.Ke[i][j] = (float)t.Ke[i][j];
      tf.Ko[i][j] = (float)t.Ko[i][j];
    }
  }
  ++*launches;
  const int gk = geom_kind(g);
  if (gk == 0) return dispatch_f32<0>(g, tf, src, dst, metric, s);
  if (gk == 1) return dispatch_f32<1>(g, tf, src, dst, metric, s);
  return dispatch_f32<2>(g, tf, src, dst, metric, s);
}

static cudaError_t general_range(const Geo &g, const Tables &t, const double *src, double *dst,
                                 const double *metric, cudaStream_t s, int64_t *launches, int64_t cb, int64_t ce) {
  if (ce <= cb) return cudaSuccess;
  ++*launches;
  const int gk = geom_kind(g);
  if (g.dim == 2) {
    if (gk == 0) return dispatch_k<2, 0>(g, t, src, dst, metric, s, cb, ce);
    if (gk == 1) return dispatch_k<2, 1>(g, t, src, dst, metric, s, cb, ce);
    return dispatch_k<2, 2>(g, t, src, dst, metric, s, cb, ce);
  }
  if (gk == 0) {
    // k = 5..7: the DMMA kernel (kernels_tc.cu) over whole cell layers
    const int64_t layer = g.nc[0] * g.nc[1];
    if (tc_supported(g) && cb % layer == 0 && ce % layer == 0)
      return launch_apply_tc(g, t, src, dst, s, (int)(cb / layer), (int)(ce / layer));
    return dispatch_k<3, 0>(g, t, src, dst, metric, s, cb, ce);
  }
  if (gk == 1) return dispatch_k<3, 1>(g, t, src, dst, metric, s, cb, ce);
  return dispatch_k<3, 2>(g, t, src, dst, metric, s, cb, ce);
}

// cells [cb, ce) only (the caller zeroes their dst planes not touched by earlier ranges)
cudaError_t launch_apply_general_cells(const Geo &g, const Tables &t, const double *src, double *dst,
                                       const double *metric, cudaStream_t s, int64_t *launches, int64_t cb,
                                       int64_t ce) {
  return general_range(g, t, src, dst, metric, s, launches, cb, ce);
}

// (the caller zeroes dst before part 0 / part 1)
cudaError_t launch_apply_general(const Geo &g, const Tables &t, const double *src, double *dst,
                                 const double *metric, cudaStream_t s, int64_t *launches, int part) {
  const int64_t layer = g.nc[0] * g.nc[1], ncells = layer * (g.dim == 3 ? g.nc[2] : 1);
  if (part == 0 || g.dim == 2) return part == 2 ? cudaSuccess : general_range(g, t, src, dst, metric, s, launches, 0, ncells);
  const int64_t nz = g.nc[2];
  if (part == 1) {  // the first and the last cell layer (all layers if nz <= 2)
    if (nz <= 2) return general_range(g, t, src, dst, metric, s, launches, 0, ncells);
    cudaError_t e = general_range(g, t, src, dst, metric, s, launches, 0, layer);
    if (e != cudaSuccess) return e;
    return general_range(g, t, src, dst, metric, s, launches, ncells - layer, ncells);
  }
  return nz <= 2 ? cudaSuccess : general_range(g, t, src, dst, metric, s, launches, layer, ncells - layer);
}

// ---------------------------------------------------------------------------
// Metric precompute (§8(a) a2): per cell and Gauss point, the isoparametric
// Jacobian J = sum_j x_j (x) grad-hat psi_j(xi_q) from the support points
// x_j = Phi(GLL node) (R4, H8), x_q = sum_j x_j psi_j(xi_q), and
// G = c(x_q) w_q det J J^{-1} J^{-T}, stored SoA [comp][cell][q]
// (3D comps: 00 01 02 11 12 22; 2D: 00 01 11).  det J <= 0 sets *bad.
// One block per cell; thread = Gauss point.  Setup only (brute-force sums).
template <int DIM, int K>
__global__ void k_metric(const __grid_constant__ Tables t, const __grid_constant__ Geo g, double *metric,
                         int *bad) {
  constexpr int N = K + 1, NV = Shape<DIM, N>::NV;
  __shared__ double X[NV][3];
  const int64_t cell = blockIdx.x;
  const int64_t ncells = g.nc[0] * g.nc[1] * (DIM == 3 ? g.nc[2] : 1);
  CellIdx ci = cell_coords(g, cell);
  for (int j = threadIdx.x; j < NV; j += blockDim.x) {
    const int l[3] = {j % N, (j / N) % N, DIM == 3 ? j / (N * N) : 0};
    double xb[3], s = 1.0;
    for (int d = 0; d < DIM; ++d) {
      double cg = (double)(d == 2 ? ci.c[2] + g.cz0 : ci.c[d]);
      xb[d] = g.lo[d] + g.h[d] * (cg + t.gll[l[d]]);
      s *= sin(M_PI * (xb[d] - g.lo[d]) / (g.hi[d] - g.lo[d]));
    }
    for (int d = 0; d < DIM; ++d)
      X[j][d] = xb[d] + (g.geom == MF_GEOM_SINE ? g.eps * (g.hi[d] - g.lo[d]) * s : 0.0);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NV; q += blockDim.x) {
    const int qd[3] = {q % N, (q / N) % N, DIM == 3 ? q / (N * N) : 0};
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, x[3] = {0, 0, 0};
    for (int j = 0; j < NV; ++j) {
      const int l[3] = {j % N, (j / N) % N, DIM == 3 ? j / (N * N) : 0};
      double sv[3], dv[3];
      for (int d = 0; d < DIM; ++d) {
        sv[d] = t.S[qd[d]][l[d]];
        dv[d] = t.D[qd[d]][l[d]];
      }
      double psi = sv[0] * sv[1] * (DIM == 3 ? sv[2] : 1.0);
      double gr[3];
      gr[0] = dv[0] * sv[1] * (DIM == 3 ? sv[2] : 1.0);
      gr[1] = sv[0] * dv[1] * (DIM == 3 ? sv[2] : 1.0);
      gr[2] = DIM == 3 ? sv[0] * sv[1] * dv[2] : 0.0;
      for (int a = 0; a < DIM; ++a) {
        x[a] += X[j][a] * psi;
        for (int b = 0; b < DIM; ++b) J[a][b] += X[j][a] * gr[b];
      }
    }
    double W = t.w[qd[0]] * t.w[qd[1]] * (DIM == 3 ? t.w[qd[2]] : 1.0);
    double c = g.coeff_kind == MF_COEFF_VARIABLE ? coeff_var(x, DIM) : g.coeff;
    const int64_t stride = ncells * NV;
    double *out = metric + cell * NV + q;
    if (DIM == 3) {
      double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
             C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      double det = J[0][0] * C00 + J[0][1] * C01 + J[0][2] * C02;
      if (!(det > 0.0)) atomicOr(bad, 1);
      double Ji[3][3];  // inverse
      Ji[0][0] = C00 / det;
      Ji[1][0] = C01 / det;
      Ji[2][0] = C02 / det;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
      const double f = c * W * det;
      int o = 0;
      for (int a = 0; a < 3; ++a)
        for (int b = a; b < 3; ++b) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m) s += Ji[a][m] * Ji[b][m];  // (J^{-1} J^{-T})_ab
          out[(o++) * stride] = f * s;
        }
    } else {
      double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      if (!(det > 0.0)) atomicOr(bad, 1);
      double Ji[2][2] = {{J[1][1] / det, -J[0][1] / det}, {-J[1][0] / det, J[0][0] / det}};
      const double f = c * W * det;
      out[0] = f * (Ji[0][0] * Ji[0][0] + Ji[0][1] * Ji[0][1]);
      out[stride] = f * (Ji[0][0] * Ji[1][0] + Ji[0][1] * Ji[1][1]);
      out[2 * stride] = f * (Ji[1][0] * Ji[1][0] + Ji[1][1] * Ji[1][1]);
    }
  }
}

template <int DIM>
static cudaError_t metric_k(const Geo &g, const Tables &t, double *metric, int *bad, cudaStream_t s) {
  const int64_t ncells = g.nc[0] * g.nc[1] * (DIM == 3 ? g.nc[2] : 1);
  if (ncells == 0) return cudaSuccess;
  const unsigned b = (unsigned)ncells;
  switch (g.k) {
    case 1: k_metric<DIM, 1><<<b, 128, 0, s>>>(t, g, metric, bad); break;
    case 2: k_metric<DIM, 2><<<b, 128, 0, s>>>(t, g, metric, bad); break;
    case 3: k_metric<DIM, 3><<<b, 128, 0, s>>>(t, g, metric, bad); break;
    case 4: k_metric<DIM, 4><<<b, 128, 0, s>>>(t, g, metric, bad); break;
    case 5: k_metric<DIM, 5><<<b, 256, 0, s>>>(t, g, metric, bad); break;
    case 6: k_metric<DIM, 6><<<b, 256, 0, s>>>(t, g, metric, bad); break;
    case 7: k_metric<DIM, 7><<<b, 256, 0, s>>>(t, g, metric, bad); break;
    case 8: k_metric<DIM, 8><<<b, 256, 0, s>>>(t, g, metric, bad); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_metric(const Geo &g, const Tables &t, double *metric, int *bad, cudaStream_t s,
                          int64_t *launches) {
  ++*launches;
  return g.dim == 2 ? metric_k<2>(g, t, metric, bad, s) : metric_k<3>(g, t, metric, bad, s);
}

// ---------------------------------------------------------------------------
// Diagonal (§8(a) a9): diag_i = sum_q sum_ab G_ab(q) dphi_i/dxhat_a dphi_i/dxhat_b,
// by sum factorisation: for each pair (a,b) the field G_ab(q) is contracted
// with T_d^T along each direction d, T_d = S.S (d not in {a,b}), D.S (d in
// exactly one), D.D (d = a = b) -- elementwise products of the 1D tables.
template <int N>
__device__ __forceinline__ double tab(const Tables &t, int kind, int q, int i) {
  double s = t.S[q][i], d = t.D[q][i];
  return kind == 0 ? s * s : (kind == 1 ? d * s : d * d);
}

template <int DIM, int K, int GEOM>
__global__ void __launch_bounds__(256) k_diagonal(const __grid_constant__ Tables t, const __grid_constant__ Geo g,
                                                  double *__restrict__ diag, const double *__restrict__ metric,
                                                  int cpb) {
  constexpr int N = K + 1, NP = Shape<DIM, N>::NP, NV = Shape<DIM, N>::NV;
  extern __shared__ double sm[];
  const int64_t ncells = g.nc[0] * g.nc[1] * (DIM == 3 ? g.nc[2] : 1);
  const int64_t cell0 = (int64_t)blockIdx.x * cpb;
  const int cl = threadIdx.x / NP, p = threadIdx.x - cl * NP;
  const bool active = cl < cpb;
  double *acc = sm + cl * 2 * NV, *tmp = acc + NV;
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) sm[(idx / NV) * 2 * NV + idx % NV] = 0.0;
  constexpr int NPAIR = DIM == 3 ? 6 : 3;
  for (int pr = 0; pr < NPAIR; ++pr) {
    int a, b;
    if (DIM == 3) {
      const int A[6] = {0, 0, 0, 1, 1, 2}, B[6] = {0, 1, 2, 1, 2, 2};
      a = A[pr];
      b = B[pr];
    } else {
      const int A[3] = {0, 0, 1}, B[3] = {0, 1, 1};
      a = A[pr];
      b = B[pr];
    }
    if (GEOM != 2 && a != b) continue;  // affine boxes: G is diagonal
    __syncthreads();
    for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
      const int c2 = idx / NV, q = idx - c2 * NV;
      const int64_t cell = cell0 + c2;
      double v = 0.0;
      if (cell < ncells) {
        const int qd[3] = {q % N, (q / N) % N, DIM == 3 ? q / (N * N) : 0};
        if (GEOM == 2) {
          v = metric[(int64_t)pr * ncells * NV + cell * NV + q] * (a == b ? 1.0 : 2.0);
        } else {
          double W = t.w[qd[0]] * t.w[qd[1]] * (DIM == 3 ? t.w[qd[2]] : 1.0);
          if (GEOM == 1) {
            CellIdx ci = cell_coords(g, cell);
            double x[3];
            for (int d = 0; d < DIM; ++d) {
              double cg = (double)(d == 2 ? ci.c[2] + g.cz0 : ci.c[d]);
              x[d] = g.lo[d] + g.h[d] * (cg + t.xi[qd[d]]);
            }
            double vol = g.h[0] * g.h[1] * (DIM == 3 ? g.h[2] : 1.0);
            v = W * coeff_var(x, DIM) * vol / (g.h[a] * g.h[a]);
          } else {
            v = W * g.fcart[a];
          }
        }
      }
      sm[c2 * 2 * NV + NV + nidx<DIM, N>(q)] = v;
    }
    __syncthreads();
    for (int e = 0; e < DIM; ++e) {
      const int kind = (e == a && e == b) ? 2 : ((e == a || e == b) ? 1 : 0);
      if (active) {
        double in[N], out[N];
#pragma unroll
        for (int i = 0; i < N; ++i) in[i] = tmp[pen_off<DIM, N>(e, p, i)];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) s = fma(tab<N>(t, kind, q, i), in[q], s);
          out[i] = s;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) tmp[pen_off<DIM, N>(e, p, i)] = out[i];
      }
      __syncthreads();
    }
    for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
      const int c2 = idx / NV, i = idx - c2 * NV;
      sm[c2 * 2 * NV + i] += sm[c2 * 2 * NV + NV + i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
    const int c2 = idx / NV, i = idx - c2 * NV;
    const int64_t cell = cell0 + c2;
    if (cell >= ncells) continue;
    CellIdx ci = cell_coords(g, cell);
    int64_t m[3];
    int64_t gi = node_index<DIM, N>(g, ci, i, m);
    if (is_constrained(g, m)) {
      if (owner_of<DIM, N>(g, ci, i, m)) diag[gi] = 1.0;
    } else {
      atomicAdd(diag + gi, sm[c2 * 2 * NV + nidx<DIM, N>(i)]);
    }
  }
}

template <int DIM, int K, int GEOM>
static cudaError_t diag_t(const Geo &g, const Tables &t, double *diag, const double *metric, cudaStream_t s) {
  constexpr int N = K + 1, NP = Shape<DIM, N>::NP, NV = Shape<DIM, N>::NV;
  int cpb = 256 / NP;
  while (cpb > 1 && cpb * 2 * NV * 8 > 48 * 1024) --cpb;
  if (cpb < 1) cpb = 1;
  const int threads = ((cpb * NP + 31) / 32) * 32;
  const int64_t ncells = g.nc[0] * g.nc[1] * (DIM == 3 ? g.nc[2] : 1);
  const int64_t blocks = (ncells + cpb - 1) / cpb;
  if (blocks == 0) return cudaSuccess;
  k_diagonal<DIM, K, GEOM><<<(unsigned)blocks, threads, (size_t)cpb * 2 * NV * 8, s>>>(t, g, diag, metric, cpb);
  return cudaGetLastError();
}

template <int DIM, int GEOM>
static cudaError_t diag_k(const Geo &g, const Tables &t, double *diag, const double *metric, cudaStream_t s) {
  switch (g.k) {
    case 1: return diag_t<DIM, 1, GEOM>(g, t, diag, metric, s);
    case 2: return diag_t<DIM, 2, GEOM>(g, t, diag, metric, s);
    case 3: return diag_t<DIM, 3, GEOM>(g, t, diag, metric, s);
    case 4: return diag_t<DIM, 4, GEOM>(g, t, diag, metric, s);
    case 5: return diag_t<DIM, 5, GEOM>(g, t, diag, metric, s);
    case 6: return diag_t<DIM, 6, GEOM>(g, t, diag, metric, s);
    case 7: return diag_t<DIM, 7, GEOM>(g, t, diag, metric, s);
    case 8: return diag_t<DIM, 8, GEOM>(g, t, diag, metric, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_diagonal(const Geo &g, const Tables &t, double *diag, const double *metric, cudaStream_t s,
                            int64_t *launches) {
  ++*launches;
  const int gk = geom_kind(g);
  if (g.dim == 2) {
    if (gk == 0) return diag_k<2, 0>(g, t, diag, metric, s);
    if (gk == 1) return diag_k<2, 1>(g, t, diag, metric, s);
    return diag_k<2, 2>(g, t, diag, metric, s);
  }
  if (gk == 0) return diag_k<3, 0>(g, t, diag, metric, s);
  if (gk == 1) return diag_k<3, 1>(g, t, diag, metric, s);
  return diag_k<3, 2>(g, t, diag, metric, s);
}

}  // namespace mf

namespace mf {

// x_g = value on every constrained local DoF (R3); used for the eigenvalue
// start vector and tests.  One pass over the local vector (setup only).
__global__ void k_set_constrained(const __grid_constant__ Geo g, double *x, double value) {
  const int64_t n = g.N[0] * g.N[1] * g.N[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t m[3] = {i % g.N[0], (i / g.N[0]) % g.N[1], i / (g.N[0] * g.N[1])};
    if (is_constrained(g, m)) x[i] = value;
  }
}

cudaError_t launch_set_constrained(const Geo &g, double *x, double value, cudaStream_t s, int64_t *launches) {
  ++*launches;
  const int64_t n = g.N[0] * g.N[1] * g.N[2];
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  k_set_constrained<<<(unsigned)b, 256, 0, s>>>(g, x, value);
  return cudaGetLastError();
}

}  // namespace mf

// ---------------------------------------------------------------------------
// General unstructured hexahedral meshes (§3.1,
// P:776-781 §3.5; R21, R22).  Same a3-a7 arithmetic as the stored-metric
// path of k_apply_general; the gather reads the cell's DoF indices from cell_dofs
// (int32, cell-major, coalesced) instead of computing them from brick coordinates,
// and resolves a constraint line -- a hanging node, u = sum_j w_j u[dof_j] -- in the
// gather and its transpose in the scatter (the paper's "constraints applied inside
// the matrix-free loop").  Dirichlet entries read zero and receive nothing; their
// identity rows are one extra pass over the Dirichlet list.
namespace mf {

// metric of the trilinear map (R21): thread = (cell, Gauss point);
// G = c(x_q) w_q det J J^-1 J^-T, J[a][e] = d x_a / d xi_e, SoA [comp][cell][q]
template <int K>
__global__ void k_hex_metric(const __grid_constant__ Tables t, const double *__restrict__ V,
                             const int32_t *__restrict__ CV, int64_t ncells, int coeff_kind, double coeff,
                             double *__restrict__ metric, int *bad) {
  constexpr int N = K + 1, NQ = N * N * N;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= ncells * NQ) return;
  const int64_t cell = idx / NQ;
  const int q = (int)(idx - cell * NQ);
  const double xi[3] = {t.xi[q % N], t.xi[(q / N) % N], t.xi[q / (N * N)]};
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, x[3] = {0, 0, 0};
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int c[3] = {v & 1, (v >> 1) & 1, v >> 2};
    double f[3], df[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      f[d] = c[d] ? xi[d] : 1.0 - xi[d];
      df[d] = c[d] ? 1.0 : -1.0;
    }
    const double Nv = f[0] * f[1] * f[2];
    const double dN[3] = {df[0] * f[1] * f[2], f[0] * df[1] * f[2], f[0] * f[1] * df[2]};
    const int64_t vid = CV[cell * 8 + v];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double X = V[vid * 3 + a];
      x[a] += X * Nv;
#pragma unroll
      for (int e = 0; e < 3; ++e) J[a][e] += X * dN[e];
    }
  }
  const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
               C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * C00 + J[0][1] * C01 + J[0][2] * C02;
  if (!(det > 0.0)) atomicExch(bad, 1);
  // J^-1 = adj(J) / det, adj(J)[e][a] = cofactor[a][e]
  double Ji[3][3];
  Ji[0][0] = C00 / det;
  Ji[1][0] = C01 / det;
  Ji[2][0] = C02 / det;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  const double c = coeff_kind == MF_COEFF_VARIABLE ? coeff_var(x, 3) : coeff;
  const double f = c * t.w[q % N] * t.w[(q / N) % N] * t.w[q / (N * N)] * det;
  const int ab[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  const int64_t stride = ncells * NQ;
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    const int a = ab[m][0], b = ab[m][1];
    metric[m * stride + idx] = f * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
  }
}

template <int K>
__global__ void __launch_bounds__(256) k_apply_hex(const __grid_constant__ Tables t, const __grid_constant__ HexDev h,
                                                   const double *__restrict__ src, double *__restrict__ dst,
                                                   int cpb) {
  constexpr int DIM = 3, N = K + 1, NP = N * N, NV = NP * N;
  constexpr int CS = 4 * NV;
  extern __shared__ double sm[];
  const int64_t ncells = h.ncells;
  const int64_t cell0 = (int64_t)blockIdx.x * cpb;
  // a3: gather through cell_dofs (constraint lines resolved here)
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
    const int cl = idx / NV, i = idx - cl * NV;
    const int64_t cell = cell0 + cl;
    double v = 0.0;
    if (cell < ncells) v = hex_gather(h, src, __ldg(h.cell_dofs + cell * NV + i));
    sm[cl * CS + nidx<DIM, N>(i)] = v;
  }
  __syncthreads();
  const int cl = threadIdx.x / NP, p = threadIdx.x - cl * NP;
  const bool active = cl < cpb;
  double *U = sm + cl * CS;
  // a4: values at the Gauss points, then the reference gradient
#pragma unroll
  for (int e = 0; e < DIM; ++e) {
    if (active) sweep_inplace<DIM, N, false>(t.S, U, e, p);
    __syncthreads();
  }
  if (active) {
#pragma unroll
    for (int e = 0; e < DIM; ++e) {
      double a[N], b[N];
#pragma unroll
      for (int i = 0; i < N; ++i) a[i] = U[pen_off<DIM, N>(e, p, i)];
      mat1d<N, false>(t.Co, a, b);
      double *G = U + (e + 1) * NV;
#pragma unroll
      for (int i = 0; i < N; ++i) G[pen_off<DIM, N>(e, p, i)] = b[i];
    }
  }
  __syncthreads();
  // a5: the stored metric of the trilinear map
  const int64_t stride = ncells * NV;
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
    const int c2 = idx / NV, q = idx - c2 * NV;
    const int64_t cell = cell0 + c2;
    const bool ok = cell < ncells;
    const double *Gm = h.metric + (ok ? cell * NV + q : 0);
    double G[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) G[c] = ok ? __ldg(Gm + c * stride) : 0.0;
    double *Uc = sm + c2 * CS;
    const int qs = nidx<DIM, N>(q);
    const double g0 = Uc[NV + qs], g1 = Uc[2 * NV + qs], g2 = Uc[3 * NV + qs];
    Uc[NV + qs] = G[0] * g0 + G[1] * g1 + G[2] * g2;
    Uc[2 * NV + qs] = G[1] * g0 + G[3] * g1 + G[4] * g2;
    Uc[3 * NV + qs] = G[2] * g0 + G[4] * g1 + G[5] * g2;
  }
  __syncthreads();
  // a6: transposed derivative and interpolation
  if (active) {
#pragma unroll
    for (int e = 0; e < DIM; ++e) sweep_inplace<DIM, N, true>(t.Co, U + (e + 1) * NV, e, p);
  }
  __syncthreads();
  if (active) {
    double a[N], b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int o = pen_off<DIM, N>(0, p, i);
      a[i] = U[NV + o] + U[2 * NV + o] + U[3 * NV + o];
    }
    mat1d<N, true>(t.S, a, b);
#pragma unroll
    for (int i = 0; i < N; ++i) U[pen_off<DIM, N>(0, p, i)] = b[i];
  }
  __syncthreads();
#pragma unroll
  for (int e = 1; e < DIM; ++e) {
    if (active) sweep_inplace<DIM, N, true>(t.S, U, e, p);
    __syncthreads();
  }
  // a7: scatter-add through cell_dofs (transpose of the constraint lines)
  for (int idx = threadIdx.x; idx < cpb * NV; idx += blockDim.x) {
    const int c2 = idx / NV, i = idx - c2 * NV;
    const int64_t cell = cell0 + c2;
    if (cell < ncells) hex_scatter(h, dst, __ldg(h.cell_dofs + cell * NV + i), sm[c2 * CS + nidx<DIM, N>(i)]);
  }
}

// dst[dir] = src[dir] (identity rows), or = value when src is null
__global__ void k_hex_identity(const int32_t *__restrict__ dir, int64_t n, const double *__restrict__ src,
                               double *__restrict__ dst, double value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = dir[i];
    dst[d] = src ? src[d] : value;
  }
}

// A_c[i][j] = sum_q grad_xi phi_i(q)^T G(q) grad_xi phi_j(q), brute force over q
template <int K>
__device__ double hex_entry(const Tables &t, const HexDev &h, int64_t cell, int i, int j) {
  constexpr int N = K + 1, NV = N * N * N;
  const int i0 = i % N, i1 = (i / N) % N, i2 = i / (N * N);
  const int j0 = j % N, j1 = (j / N) % N, j2 = j / (N * N);
  const int64_t stride = h.ncells * NV;
  double s = 0.0;
  for (int q = 0; q < NV; ++q) {
    const int q0 = q % N, q1 = (q / N) % N, q2 = q / (N * N);
    const double a[3] = {t.D[q0][i0] * t.S[q1][i1] * t.S[q2][i2], t.S[q0][i0] * t.D[q1][i1] * t.S[q2][i2],
                         t.S[q0][i0] * t.S[q1][i1] * t.D[q2][i2]};
    const double b[3] = {t.D[q0][j0] * t.S[q1][j1] * t.S[q2][j2], t.S[q0][j0] * t.D[q1][j1] * t.S[q2][j2],
                         t.S[q0][j0] * t.S[q1][j1] * t.D[q2][j2]};
    const double *Gm = h.metric + cell * NV + q;
    const double G[6] = {__ldg(Gm), __ldg(Gm + stride), __ldg(Gm + 2 * stride), __ldg(Gm + 3 * stride),
                         __ldg(Gm + 4 * stride), __ldg(Gm + 5 * stride)};
    s += a[0] * (G[0] * b[0] + G[1] * b[1] + G[2] * b[2]) + a[1] * (G[1] * b[0] + G[3] * b[1] + G[4] * b[2]) +
         a[2] * (G[2] * b[0] + G[4] * b[1] + G[5] * b[2]);
  }
  return s;
}

// diagonal of sum_c P_c^T A_c P_c: thread = (cell, local node i); on cells without
// constraint lines only A_c[i][i]; on the others every pair (i, j) whose expansions
// share a DoF m adds w_im w_jm A_c[i][j] to diag[m] (setup only)
template <int K>
__global__ void k_diag_hex(const __grid_constant__ Tables t, const __grid_constant__ HexDev h, double *diag) {
  constexpr int N = K + 1, NV = N * N * N;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= h.ncells * NV) return;
  const int64_t cell = idx / NV;
  const int i = (int)(idx - cell * NV);
  const int32_t di = h.cell_dofs[cell * NV + i];
  if (di == kHexDirichlet) return;
  if (!h.cell_lines[cell]) {
    if (di >= 0) atomicAdd(diag + di, hex_entry<K>(t, h, cell, i, i));
    return;
  }
  auto span = [&](int32_t d, int &b, int &e) {
    if (d >= 0) {
      b = 0;
      e = 1;
    } else {
      b = h.line_ptr[-1 - d];
      e = h.line_ptr[-d];
    }
  };
  int bi, ei;
  span(di, bi, ei);
  for (int j = 0; j < NV; ++j) {
    const int32_t dj = h.cell_dofs[cell * NV + j];
    if (dj == kHexDirichlet) continue;
    int bj, ej;
    span(dj, bj, ej);
    double Aij = 0.0;
    bool have = false;
    for (int a = bi; a < ei; ++a) {
      const int32_t m = di >= 0 ? di : h.line_dof[a];
      const double wm = di >= 0 ? 1.0 : h.line_w[a];
      double s = 0.0;
      bool hit = false;
      for (int b = bj; b < ej; ++b) {
        if ((dj >= 0 ? dj : h.line_dof[b]) == m) {
          s += dj >= 0 ? 1.0 : h.line_w[b];
          hit = true;
        }
      }
      if (!hit) continue;
      if (!have) {
        Aij = hex_entry<K>(t, h, cell, i, j);
        have = true;
      }
      atomicAdd(diag + m, wm * s * Aij);
    }
  }
}

template <int K>
static cudaError_t hex_metric_k(const Tables &t, const double *V, const int32_t *CV, int64_t ncells, int ck,
                                double cv, double *metric, int *bad, cudaStream_t s) {
  constexpr int NQ = (K + 1) * (K + 1) * (K + 1);
  const int64_t n = ncells * NQ;
  if (n == 0) return cudaSuccess;
  k_hex_metric<K><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(t, V, CV, ncells, ck, cv, metric, bad);
  return cudaGetLastError();
}

template <int K>
static cudaError_t hex_apply_k(const Tables &t, const HexDev &h, const double *src, double *dst, cudaStream_t s) {
  constexpr int N = K + 1, NP = N * N, NV = NP * N;
  static const bool v1 = std::getenv("MF_HEX_V1") != nullptr;  // the shared-memory pencil kernel (comparisons)
  if (!v1) {  // k_apply_cell3 with the cell_dofs gather / scatter and the TMA-staged metric
    constexpr int c3 = cell3_cpb<K, 3>();
    const int64_t b3 = (h.ncells + c3 - 1) / c3;
    const size_t sm3 = cell3_smem_bytes<K, 3, double>();
    smem_attr_once(k_apply_cell3<K, 3, double>, sm3);
    if (b3 == 0) return cudaSuccess;
    Geo g{};
    return launch_cell3_pdl<K, 3>((unsigned)b3, ((c3 * NP + 31) / 32) * 32, sm3, s, t, g, src, dst, h.metric, 0,
                                  h.ncells, h);
  }
  int cpb = 256 / NP;
  while (cpb > 1 && cpb * 4 * NV * 8 > 48 * 1024) --cpb;
  if (cpb < 1) cpb = 1;
  const int threads = ((cpb * NP + 31) / 32) * 32;
  const int64_t blocks = (h.ncells + cpb - 1) / cpb;
  if (blocks == 0) return cudaSuccess;
  k_apply_hex<K><<<(unsigned)blocks, threads, (size_t)cpb * 4 * NV * sizeof(double), s>>>(t, h, src, dst, cpb);
  return cudaGetLastError();
}

template <int K>
static cudaError_t hex_diag_k(const Tables &t, const HexDev &h, double *diag, cudaStream_t s) {
  constexpr int NV = (K + 1) * (K + 1) * (K + 1);
  const int64_t n = h.ncells * NV;
  if (n == 0) return cudaSuccess;
  k_diag_hex<K><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(t, h, diag);
  return cudaGetLastError();
}

#define MF_HEX_DISPATCH(CALL)      \
  switch (k) {                     \
    case 1: return CALL(1);        \
    case 2: return CALL(2);        \
    case 3: return CALL(3);        \
    case 4: return CALL(4);        \
    case 5: return CALL(5);        \
    case 6: return CALL(6);        \
    case 7: return CALL(7);        \
    case 8: return CALL(8);        \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_hex_metric(int k, const Tables &t, const double *V, const int32_t *CV, int64_t ncells,
                              int coeff_kind, double coeff, double *metric, int *bad, cudaStream_t s,
                              int64_t *launches) {
  ++*launches;
#define MF_C(KK) hex_metric_k<KK>(t, V, CV, ncells, coeff_kind, coeff, metric, bad, s)
  MF_HEX_DISPATCH(MF_C)
#undef MF_C
}

static cudaError_t hex_identity(const HexDev &h, const double *src, double *dst, double value, cudaStream_t s,
                                int64_t *launches) {
  if (h.ndir == 0) return cudaSuccess;
  ++*launches;
  int64_t b = (h.ndir + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  k_hex_identity<<<(unsigned)b, 256, 0, s>>>(h.dir, h.ndir, src, dst, value);
  return cudaGetLastError();
}

cudaError_t launch_apply_hex(int k, const Tables &t, const HexDev &h, const double *src, double *dst,
                             cudaStream_t s, int64_t *launches) {
  ++*launches;
  cudaError_t e = [&]() -> cudaError_t {
#define MF_C(KK) hex_apply_k<KK>(t, h, src, dst, s)
    MF_HEX_DISPATCH(MF_C)
#undef MF_C
  }();
  if (e != cudaSuccess) return e;
  return hex_identity(h, src, dst, 0.0, s, launches);
}

cudaError_t launch_diagonal_hex(int k, const Tables &t, const HexDev &h, double *diag, cudaStream_t s,
                                int64_t *launches) {
  ++*launches;
  cudaError_t e = [&]() -> cudaError_t {
#define MF_C(KK) hex_diag_k<KK>(t, h, diag, s)
    MF_HEX_DISPATCH(MF_C)
#undef MF_C
  }();
  if (e != cudaSuccess) return e;
  return hex_identity(h, nullptr, diag, 1.0, s, launches);
}

cudaError_t launch_hex_set(const HexDev &h, double *x, double value, cudaStream_t s, int64_t *launches) {
  return hex_identity(h, nullptr, x, value, s, launches);
}

}  // namespace mf
