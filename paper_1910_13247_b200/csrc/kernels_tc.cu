// kernels_tc.cu -- the Cartesian constant-coefficient cell operator for k = 5..7 on the FP64
// tensor cores (DMMA, mma.sync m8n8k4 f64).  §8(a) a3-a7 for cfg 5 Q6 (BASELINE configs[4]).
//
// The operation is the paper's matrix-free cell operator (§3, sum factorisation
// eq. (5)-(7)) in the exact Kronecker form of an affine box cell with constant coefficient
// (the same form as k_apply_cell3<k,0> and the halo kernel):
//   v_cell = fx Kx(x)My(x)Mz u + fy Mx(x)Ky(x)Mz u + fz Mx(x)My(x)Kz u
// with the reference 1D mass / stiffness M, K (Gauss(k+1) exact) and fd = c prod(h) / h_d^2.
//
// Design (B200-first, not the paper's): one warp per column of cells along z, no shared memory.
// Per z-slice w of a cell (the 8 x 8 padded (y, x) node plane, N = k + 1 <= 8 nodes):
//   1. y contraction on DMMA: a_w = M U_w, b_w = fy K U_w (A = the 8x8 matrix, two k-steps;
//      B = U_w[y][x] loaded straight from global memory into the B fragment, lane (k = y & 3,
//      n = x), constrained nodes and padding as 0);
//   2. x contraction on DMMA with the accumulator of step 1 as the A operand: the D fragment
//      holds D[y][2 (lane & 3) + i], which is the A fragment of k-step i when the contraction
//      index is permuted to x = 2 k + i (the B operand, a constant, is permuted the same way):
//      P_w = fx a_w K^T + b_w M^T,  Q_w = fz a_w M^T;
//   3. z contraction in scalar FP64 per lane: each lane holds P_w, Q_w at its two (y, x)
//      positions for every w, so v = M_z P + K_z Q is the even-odd product (M, K are
//      centro-symmetric) on registers.
// Consecutive cells of the column share the z-face slice: its P, Q (steps 1-2 depend only on
// the slice) and the output partial sums of that face stay in registers, so each further cell
// loads and contracts N - 1 slices and issues no atomics on its bottom face.  Output is
// scatter-add (dst zeroed by the preceding kernel, programmatic dependent launch) with the
// Dirichlet identity rows written by their owner cell (the rule of k_apply_cell3).
//
// Cost per cell (k = 6): 60 DMMA (16 SMSP cycles each) + ~136 DFMA-class lane instructions,
// ~12 loads and ~12 reductions per lane, vs ~1870 warp instructions of the collocation form.
// Registers bound the occupancy: the next cell's slices are prefetched one cell ahead (2 (N-1)
// doubles), P and Q of every slice are held for the z step (4 N), and for k = 5, 6 the matrix
// fragments are re-read from shared memory instead of being held (DESIGN.md §7.0b has the
// variants measured).  Cells off the Dirichlet faces take a branch-free scatter; boundary
// cells load their identity-row sources before storing (one latency instead of N).
#include <cstdint>
#include <cstdlib>

#include "internal.h"

namespace mf {

struct TcParams {
  double M[8][8], K[8][8];                           // reference 1D mass / stiffness, zero padded
  double Me[5][5], Mo[5][5], Ke[5][5], Ko[5][5];     // their even-odd parts (Tables::Me)
  double fx, fy, fz;
  int64_t Nx, plane;                                 // local node strides
  int64_t items;                                     // ncx * ncy * nchunks
  int ncx, ncy, ncz;                                 // local cells
  int cz_lo, cz_hi, lz;                              // cell layers [cz_lo, cz_hi) in chunks of lz
  uint32_t dirichlet;
  int skip_top_identity;
};

#ifdef MF_TC_STORE  // timing experiment only: plain stores instead of reductions (wrong results)
#define TC_RED(p, v) (*(p) = (v))
#else
#define TC_RED(p, v) atomicAdd((p), (v))
#endif

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// threads per block: 12 warps per SM for k = 5, 6 (<= 168 registers), 8 for k = 7 (~200)
#ifndef MF_TC_THREADS
#define MF_TC_THREADS 384
#endif
__host__ __device__ constexpr int tc_threads(int k) { return k == 7 ? 256 : MF_TC_THREADS; }

template <int K>
__global__ void __launch_bounds__(tc_threads(K), 1) k_apply_tc(const __grid_constant__ TcParams p,
                                                     const double *__restrict__ src, double *__restrict__ dst) {
  constexpr int N = K + 1, m = N / 2, h = (N + 1) / 2;
  static_assert(N <= 8, "one 8x8 DMMA tile per slice");
  const int lane = threadIdx.x & 31, r = lane >> 2, c4 = lane & 3;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // the lane constants: fragment values of the 1D matrices, step-1 A operands (row y' = r,
  // column y = 4 kk + c4) and step-2 B operands (B[k][n] = C[x' = r][x = 2 c4 + s] for k-step
  // s).  For k = 5, 6 they live in shared memory and are re-read per use (volatile: not
  // hoisted), so they do not hold 20 registers through the column walk (k = 6 then fits 12
  // warps per SM without spilling); k = 7 runs 8 warps and keeps them in registers.
  constexpr bool CSM = K != 7;
  __shared__ double cst[CSM ? 10 : 1][32];
  double creg[10];
  auto fill = [&](double *c, int stride) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      c[kk * stride] = p.M[r][4 * kk + c4];
      c[(2 + kk) * stride] = p.fy * p.K[r][4 * kk + c4];
      c[(4 + kk) * stride] = p.fx * p.K[r][2 * c4 + kk];
      c[(6 + kk) * stride] = p.M[r][2 * c4 + kk];
      c[(8 + kk) * stride] = p.fz * p.M[r][2 * c4 + kk];
    }
  };
  if constexpr (CSM) {
    if (threadIdx.x < 32) fill(&cst[0][lane], 32);
    __syncthreads();
  } else {
    fill(creg, 1);
  }
  const volatile double *cs = &cst[0][lane];
  auto C = [&](int i) -> double {
    if constexpr (CSM) {
      return cs[i * 32];
    } else {
      return creg[i];
    }
  };
  if (item >= p.items) return;
  const int cx = (int)(item % p.ncx);
  const int64_t t1 = item / p.ncx;
  const int cy = (int)(t1 % p.ncy), chunk = (int)(t1 / p.ncy);
  const int c0 = p.cz_lo + chunk * p.lz, c1 = min(c0 + p.lz, p.cz_hi);
  const uint32_t d = p.dirichlet;

  // the cell's x / y faces (fixed along the column)
  const bool fxm = (d & 1u) && cx == 0, fxp = (d & 2u) && cx == p.ncx - 1;
  const bool fym = (d & 4u) && cy == 0, fyp = (d & 8u) && cy == p.ncy - 1;
  // load positions (x = r, y = 4 kk + c4) and output positions (x = 2 c4 + i, y = r)
  bool lok[2];
  int lofs[2];
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const int x = r, y = 4 * kk + c4;
    const bool cons = (fxm && x == 0) || (fxp && x == N - 1) || (fym && y == 0) || (fyp && y == N - 1);
    lok[kk] = x < N && y < N && !cons;
    lofs[kk] = y * (int)p.Nx + x;
  }
  bool ook[2], ocons[2], oown[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int x = 2 * c4 + i, y = r;
    ook[i] = x < N && y < N;
    ocons[i] = (fxm && x == 0) || (fxp && x == N - 1) || (fym && y == 0) || (fyp && y == N - 1);
    oown[i] = (x >= 1 || cx == 0) && (y >= 1 || cy == 0);
  }
  const int oofs = r * (int)p.Nx + 2 * c4;
  const int64_t colbase = (int64_t)K * cy * p.Nx + (int64_t)K * cx;
  const bool xyface = fxm || fxp || fym || fyp;

  auto zcons = [&](int cz, int w) {
    return (w == 0 && (d & 16u) && cz == 0) || (w == N - 1 && (d & 32u) && cz == p.ncz - 1);
  };
  auto load_slice = [&](int cz, int w, double (&u)[2]) {
    const bool zc = zcons(cz, w);
    const double *ps = src + colbase + ((int64_t)K * cz + w) * p.plane;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) u[kk] = (lok[kk] && !zc) ? __ldg(ps + lofs[kk]) : 0.0;
  };

  double ub[N][2];
#pragma unroll
  for (int w = 0; w < N; ++w) load_slice(c0, w, ub[w]);
  double P[N][2], Q[N][2], carry[2] = {0.0, 0.0};
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // dst zeroing grid complete

  for (int cz = c0; cz < c1; ++cz) {
    const bool first = cz == c0, last = cz == c1 - 1;
#pragma unroll
    for (int w = 0; w < N; ++w) {
      if (w == 0 && !first) {  // the shared z-face slice: steps 1-2 of the cell below
        P[0][0] = P[N - 1][0];
        P[0][1] = P[N - 1][1];
        Q[0][0] = Q[N - 1][0];
        Q[0][1] = Q[N - 1][1];
        continue;
      }
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      dmma(a0, a1, C(0), ub[w][0]);
      dmma(b0, b1, C(2), ub[w][0]);
      dmma(a0, a1, C(1), ub[w][1]);
      dmma(b0, b1, C(3), ub[w][1]);
      if (w >= 1 && !last) load_slice(cz + 1, w, ub[w]);  // next cell, one cell ahead
      double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0, r0 = 0.0, r1 = 0.0;
      dmma(p0, p1, a0, C(4));
      dmma(r0, r1, b0, C(6));
      dmma(q0, q1, a0, C(8));
      dmma(p0, p1, a1, C(5));
      dmma(r0, r1, b1, C(7));
      dmma(q0, q1, a1, C(9));
      P[w][0] = p0 + r0;
      P[w][1] = p1 + r1;
      Q[w][0] = q0;
      Q[w][1] = q1;
    }
    // 3. z contraction (even-odd) and scatter, per output column i
    const int64_t cbase = colbase + (int64_t)K * cz * p.plane + oofs;
    const bool zm = (d & 16u) && cz == 0, zp = (d & 32u) && cz == p.ncz - 1;
    const bool skip = p.skip_top_identity && cz == p.ncz - 1;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      double pe[h], po[m > 0 ? m : 1], qe[h], qo[m > 0 ? m : 1], v[N];
#pragma unroll
      for (int j = 0; j < m; ++j) {
        pe[j] = P[j][i] + P[N - 1 - j][i];
        po[j] = P[j][i] - P[N - 1 - j][i];
        qe[j] = Q[j][i] + Q[N - 1 - j][i];
        qo[j] = Q[j][i] - Q[N - 1 - j][i];
      }
      if (N & 1) {
        pe[m] = P[m][i];
        qe[m] = Q[m][i];
      }
#pragma unroll
      for (int j = 0; j < h; ++j) {
        double ve = p.Me[j][0] * pe[0];
#pragma unroll
        for (int l = 1; l < h; ++l) ve = fma(p.Me[j][l], pe[l], ve);
#pragma unroll
        for (int l = 0; l < h; ++l) ve = fma(p.Ke[j][l], qe[l], ve);
        if (j < m) {
          double vo = p.Mo[j][0] * po[0];
#pragma unroll
          for (int l = 1; l < m; ++l) vo = fma(p.Mo[j][l], po[l], vo);
#pragma unroll
          for (int l = 0; l < m; ++l) vo = fma(p.Ko[j][l], qo[l], vo);
          v[j] = ve + vo;
          v[N - 1 - j] = ve - vo;
        } else {
          v[j] = ve;
        }
      }
      if (!ook[i]) continue;
      if (!xyface && !zm && !zp) {  // no constrained node in this cell column
        if (!first) v[0] += carry[i];
#pragma unroll
        for (int w = 0; w < N - 1; ++w) TC_RED(dst + cbase + (int64_t)w * p.plane + i, v[w]);
        if (last) {
          TC_RED(dst + cbase + (int64_t)(N - 1) * p.plane + i, v[N - 1]);
        } else {
          carry[i] = v[N - 1];
        }
        continue;
      }
      // identity rows: load every source value first (one latency, not N)
      double idv[N];
      bool idw[N];
#pragma unroll
      for (int w = 0; w < N; ++w) {
        const int64_t gi = cbase + (int64_t)w * p.plane + i;
        const bool cons = ocons[i] || (w == 0 && zm) || (w == N - 1 && zp);
        idw[w] = cons && oown[i] && (w >= 1 || cz == 0) && !(w == N - 1 && skip);
        idv[w] = idw[w] ? __ldg(src + gi) : 0.0;
      }
#pragma unroll
      for (int w = 0; w < N; ++w) {
        const int64_t gi = cbase + (int64_t)w * p.plane + i;
        const bool cons = ocons[i] || (w == 0 && zm) || (w == N - 1 && zp);
        if (cons) {
          if (idw[w]) dst[gi] = idv[w];
          continue;
        }
        double val = v[w];
        if (w == 0 && !first) val += carry[i];
        if (w == N - 1 && !last) {
          carry[i] = val;  // the top face: added by the cell above
        } else {
          TC_RED(dst + gi, val);
        }
      }
    }
  }
}

bool tc_supported(const Geo &g) {
  static const bool off = std::getenv("MF_NO_TC") != nullptr;  // the collocation kernel (comparisons)
  return !off && g.dim == 3 && g.k >= 5 && g.k <= 7 && g.geom == MF_GEOM_CARTESIAN &&
         g.coeff_kind == MF_COEFF_CONSTANT && g.nc[0] < (1 << 30) && g.nc[1] < (1 << 30) &&
         g.N[0] * (int64_t)8 < (int64_t(1) << 31);
}

template <int K>
static cudaError_t launch_tc_k(const TcParams &p, unsigned blocks, cudaStream_t s, const double *src, double *dst) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(tc_threads(K));
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool off = std::getenv("MF_NO_PDL") != nullptr;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k_apply_tc<K>, p, src, dst);
}

// the cell layers [cz_lo, cz_hi) (dst zeroed by the caller)
cudaError_t launch_apply_tc(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                            int cz_lo, int cz_hi) {
  if (!tc_supported(g)) return cudaErrorNotSupported;
  if (cz_hi <= cz_lo) return cudaSuccess;
  const int N = g.k + 1;
  TcParams p = {};
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) {
      p.M[i][j] = t.Mr[i][j];
      p.K[i][j] = t.Kr[i][j];
    }
  }
  for (int i = 0; i < 5; ++i) {
    for (int j = 0; j < 5; ++j) {
      p.Me[i][j] = t.Me[i][j];
      p.Mo[i][j] = t.Mo[i][j];
      p.Ke[i][j] = t.Ke[i][j];
      p.Ko[i][j] = t.Ko[i][j];
    }
  }
  p.fx = g.fcart[0];
  p.fy = g.fcart[1];
  p.fz = g.fcart[2];
  p.Nx = g.N[0];
  p.plane = g.N[0] * g.N[1];
  p.ncx = (int)g.nc[0];
  p.ncy = (int)g.nc[1];
  p.ncz = (int)g.nc[2];
  p.dirichlet = g.dirichlet;
  p.skip_top_identity = g.skip_top_identity;
  p.cz_lo = cz_lo;
  p.cz_hi = cz_hi;
  // z chunks: enough warps for ~8 per SM-slot wave, chunks of >= 4 cells
  const int64_t cols = g.nc[0] * g.nc[1], nz = cz_hi - cz_lo;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t want = (int64_t)sms * 12 * 8;  // ~8 waves of resident warps
  int64_t nch = (want + cols - 1) / cols;
  nch = nch < 1 ? 1 : nch;
  const int64_t maxch = nz >= 8 ? nz / 4 : 1;
  if (nch > maxch) nch = maxch;
  const int64_t lz = (nz + nch - 1) / nch;
  nch = (nz + lz - 1) / lz;
  p.lz = (int)lz;
  p.items = cols * nch;
  const int wpb = tc_threads(g.k) / 32;
  const int64_t blocks = (p.items + wpb - 1) / wpb;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  switch (g.k) {
    case 5: return launch_tc_k<5>(p, (unsigned)blocks, s, src, dst);
    case 6: return launch_tc_k<6>(p, (unsigned)blocks, s, src, dst);
    case 7: return launch_tc_k<7>(p, (unsigned)blocks, s, src, dst);
  }
  return cudaErrorNotSupported;
}

}  // namespace mf
