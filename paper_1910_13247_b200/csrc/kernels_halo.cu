// kernels_halo.cu -- Q4 Cartesian constant-coefficient apply in which every output node is
// written ONCE, with a plain coalesced store, by the one CTA that owns it: no init pass, no
// atomics (apply variant 6, the default for k = 4 where supported).
//
// Operator (§3.6 sum factorisation): on the Cartesian brick
// the cell operator is the Gauss(k+1)-exact Kronecker form, so the assembled operator is the
// Kronecker sum of assembled 1D matrices
//     A = Kx (x) My (x) Mz + Mx (x) Ky (x) Mz + Mx (x) My (x) Kz      (M = S^T W S, K_e = f_e D^T W D)
// evaluated per DoF plane and node column as
//     y step  a = My u,  b = Ky u                  (every node column of a plane)
//     x step  P = Kx a + Mx b,  Q = Mx a           (every node row of a plane)
//     z step  v = Mz P + Kz Q                      (every node column, across planes)
// with each 1D product the per-cell 5x5 matrix in even-odd form and the two cells sharing a
// vertex summed -- seven 1D products per DoF, about 35 FP64 instructions per DoF.
//
// Decomposition (CTA = 512 threads, one per SM): warps 0-7 consume (x and z steps, one node
// row each), warps 8-15 produce (y step); a/b pass through NB shared-memory buffers guarded by
// full / empty mbarriers, so the producers run ahead and their global loads are prefetched a
// step early.
//   tile    32 x 2 cells in x-y (128 x 8 owned node columns) marching a z-chunk of cell
//           layers, two DoF planes per step; the CTAs of one tile row in x form a
//           thread-block cluster (<= 8) that spans the whole x extent of the mesh
//   y step  thread per (node column, plane): 13 node rows from global memory (coalesced
//           across the warp), the 4 rows below the tile feeding only the top row of the cell
//           below (recomputed: a 5-term dot product per plane); a and b of the 8 owned rows go
//           to shared memory, and the CTA's column 0 to the left CTA's column-128 slots
//           (st.async into its shared memory, completing bytes on its mbarrier)
//   x step  warp per node row, lane per cell: P, Q on the cell's 5 nodes; node 4 to the next
//           lane by shuffle -- lane 31's to the right CTA's halo slots (st.async), so node 0 of
//           a lane (the vertex column shared with the left cell) is finished one step later
//   z step  the same lane, its 4 node columns: even-odd accumulation as the planes arrive
//           (pairs (1,3) then (2,4) with the carried plane 0); node 0 once its halo is in
//   store   through a per-warp shared row in the padded XS layout (conflict-free both ways)
//           to coalesced st.global; Dirichlet rows get the identity value (R3)
//   z halo  a chunk that starts above the local layer 0 first runs the layer below without
//           storing (its top plane's carry), so chunks are independent
// No cluster-wide barrier inside the loop: the DSMEM exchanges are producer -> consumer
// (st.async + complete_tx); their slot reuse is safe because each CTA's progress is bounded
// by its neighbours' data (DCOL / DHL slots, see the comment at their definition).
// Host-checked limits (cart_halo_supported): n_cells x <= 256; an x+ / y+ boundary row that
// no CTA computes (a full last tile) must be Dirichlet (identity only).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tile_common.cuh"

namespace mf {
namespace {

constexpr int HK = 4;
constexpr int HTX = 32, HTY = 2;           // cells per tile
constexpr int HROWS = HK * HTY;            // 8 owned node rows = consumer warps
constexpr int HCOLS = HK * HTX;            // 128 owned node columns per CTA
constexpr int HNT = 2 * 32 * HROWS;        // 512 threads: 8 consumer + 8 producer warps
constexpr int HYR = HROWS + HK + 1;        // 13 input rows of a y step
constexpr int HMAXCH = 64;                 // z-chunks per launch
constexpr int HMAXCLU = 8;                 // portable cluster size -> n_cells x <= 256
constexpr int NB = 3;                      // a/b buffers (producer lead)
constexpr int NS = 3;                      // producer input stages (cp.async ring: 2 steps of prefetch)
constexpr int PROD_REGS = 104, CONS_REGS = 152;  // per-role register budgets (setmaxnreg; sum 256 = 2 x 128)
// Column-128 slots (written by the right CTA's producers) and x-halo slots (written by the
// left CTA's consumers, one per layer).  The right CTA's producer reaches step t + DCOL only
// after its consumers finished step t + DCOL - NB, whose node-0 completion waited for this
// CTA's consumers up to step t + DCOL - NB - 3 >= t: slot t % DCOL is free.  The left CTA's
// consumer writes layer L + DHL only after this CTA's producers delivered that layer's
// column 0, i.e. after this CTA's consumers passed layer L + DHL - 2 > L + 1 (node 0 of L
// done).
constexpr int DCOL = 8, DHL = 4;

__host__ __device__ constexpr int hxs(int x) { return x + (x >> 4); }  // padded row slot
constexpr int HXP = hxs(HCOLS - 1) + 1;    // 135: row pitch
constexpr int AB_PL = HROWS * HXP;         // one plane of a (or b)
constexpr int AB_BUF = 2 * 2 * AB_PL;      // a and b of the step's two planes
constexpr int OXP = hxs(HCOLS) + 1;        // 137: output row pitch (column 128 = the x+ column)
constexpr int OUT_W = HK * OXP;            // per consumer warp: 4 output planes of its row
constexpr int COL_SLOT = 2 * 2 * HROWS;    // [plane j][a/b][row]
constexpr int HL_SLOT = (HK + 1) * HROWS * 2;  // [plane 0..4][row][P, Q]
constexpr int US_STAGE = HYR * 32 * HROWS;     // producer inputs of one step: [row][producer thread]
constexpr int C128_RING = 32;                  // column 128 of a full last CTA: [plane % 32][row 0..8]
constexpr int SMEM_D =
    NB * AB_BUF + HROWS * OUT_W + DCOL * COL_SLOT + DHL * HL_SLOT + NS * US_STAGE + C128_RING * (HROWS + 1);
constexpr int NBAR = 2 * NB + DCOL + DHL;
constexpr size_t HSMEM = sizeof(double) * SMEM_D + 8 * NBAR;

// even-odd form of a centro-symmetric 5x5 matrix A: e_j = u_j + u_{4-j}, o_j = u_j - u_{4-j}
// (e_2 = u_2); ve = E e, vo = O o; v_i = ve_i + vo_i, v_{4-i} = ve_i - vo_i, v_2 = ve_2
struct EO5 {
  double E[3][3];
  double O[2][2];
};

// coefficients: M and K = f_x K_ref only (52 uniform registers: DFMA takes its matrix operand
// from the uniform register file, so two matrices fit without reloads); Ky = ry K, Kz = rz K
// are applied by scaling data (ry = rz = 1 on cubic cells: the ISO instance skips that)
struct HaloParams {
  EO5 M, K;
  double ry, rz;
  int64_t Nx, Ny, Nz;    // local node counts
  int ncx, ncy, ncz;     // local cell counts
  int ntx, nty, nch;
  uint32_t dirichlet;
  int skip_top_identity;
  int cz[HMAXCH][2];     // z-chunks [begin, end) in cell layers
  unsigned long long *prof;  // debug timeline (MF_HALO_PROF): per CTA start / steps / end, or null
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// MF_CHECKED builds trap on any out-of-range global / shared / distributed-shared index (the
// compute-sanitizer substitute: it is closed on this GPU pool)
#ifdef MF_CHECKED
#define HCHECK(c)          \
  do {                     \
    if (!(c)) __trap();    \
  } while (0)
#else
#define HCHECK(c) \
  do {            \
  } while (0)
#endif

__device__ __forceinline__ void split5(const double *u, double *e, double *o) {
  e[0] = u[0] + u[4];
  e[1] = u[1] + u[3];
  e[2] = u[2];
  o[0] = u[0] - u[4];
  o[1] = u[1] - u[3];
}
__device__ __forceinline__ void mul5(const EO5 &A, const double *e, const double *o, double *ve, double *vo) {
#pragma unroll
  for (int i = 0; i < 3; ++i) ve[i] = fma(A.E[i][2], e[2], fma(A.E[i][1], e[1], A.E[i][0] * e[0]));
#pragma unroll
  for (int i = 0; i < 2; ++i) vo[i] = fma(A.O[i][1], o[1], A.O[i][0] * o[0]);
}
__device__ __forceinline__ void acc5(const EO5 &A, const double *e, const double *o, double *ve, double *vo) {
#pragma unroll
  for (int i = 0; i < 3; ++i) ve[i] = fma(A.E[i][2], e[2], fma(A.E[i][1], e[1], fma(A.E[i][0], e[0], ve[i])));
#pragma unroll
  for (int i = 0; i < 2; ++i) vo[i] = fma(A.O[i][1], o[1], fma(A.O[i][0], o[0], vo[i]));
}
__device__ __forceinline__ void comb5(const double *ve, const double *vo, double *v) {
  v[0] = ve[0] + vo[0];
  v[4] = ve[0] - vo[0];
  v[1] = ve[1] + vo[1];
  v[3] = ve[1] - vo[1];
  v[2] = ve[2];
}

// ---- cluster / mbarrier primitives (PTX) ----
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned map_rank(unsigned a, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void bar_init(unsigned a, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned a) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
// one arrival that also expects `bytes` of st.async data in the current phase
__device__ __forceinline__ void bar_expect(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool bar_try(unsigned a, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
// waiting warps back off (they would otherwise take issue slots from the working ones)
__device__ __forceinline__ void bar_wait(unsigned a, unsigned parity) {
#ifdef HALO_NOSYNC
  return;
#endif
  while (!bar_try(a, parity)) __nanosleep(64);
}
// wait for data that other CTAs of the cluster delivered with st.async
__device__ __forceinline__ void bar_wait_cluster(unsigned a, unsigned parity) {
#ifdef HALO_NOSYNC
  return;
#endif
  while (true) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(64);
  }
}
// two doubles into CTA `rank`'s shared memory at the offset of `local`, completing 16 bytes
// on that CTA's mbarrier at the offset of `bar`
__device__ __forceinline__ void st_async2(const double *local, unsigned bar, int rank, double a, double b) {
  const unsigned ra = map_rank(smem_u32(local), rank), rb = map_rank(bar, rank);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(ra),
               "d"(a), "d"(b), "r"(rb)
               : "memory");
}

template <bool ISO>
__global__ void __launch_bounds__(HNT, 1)
    k_apply_halo(const __grid_constant__ HaloParams P, const double *__restrict__ src, double *__restrict__ dst) {
  extern __shared__ __align__(16) double sm[];
  double *const AB = sm;                       // [NB][a/b][plane slot 2][row 8][HXP]
  double *const OUT = AB + NB * AB_BUF;        // [consumer warp][plane 4][OXP]
  double *const COL = OUT + HROWS * OUT_W;     // [DCOL][plane slot][a/b][row]: the right CTA's column 0
  double *const HL = COL + DCOL * COL_SLOT;    // [DHL][plane 0..4][row][P, Q]: x halo of node 0
  double *const US = HL + DHL * HL_SLOT;       // [NS][row][producer thread]: cp.async input stages
  // [plane % 32][row]: src of the x+ column (128) of a full last CTA, loaded by the producers with
  // their planes (cp.async) and copied to dst by the consumers (it is a Dirichlet column)
  double *const C128 = US + NS * US_STAGE;
  unsigned long long *const bars = reinterpret_cast<unsigned long long *>(C128 + C128_RING * (HROWS + 1));
  const unsigned b_full = smem_u32(bars), b_empty = b_full + 8 * NB, b_col = b_empty + 8 * NB,
                 b_hl = b_col + 8 * DCOL;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rank = blockIdx.x, ntx = P.ntx;
  const bool clu = ntx > 1;
  const int ty = blockIdx.y % P.nty, ch = blockIdx.y / P.nty;
  const int cz_b = P.cz[ch][0], cz_e = P.cz[ch][1];
  const int64_t Nx = P.Nx, Ny = P.Ny, Nz = P.Nz, plane = P.Nx * P.Ny;
  const uint32_t d = P.dirichlet;
  const double ry = P.ry, rz = P.rz;
  const int x0 = HCOLS * rank, y0 = HROWS * ty;
  const int nvx = min(HTX, P.ncx - HTX * rank), nvy = min(HTY, P.ncy - HTY * ty);
  const bool last_x = rank == ntx - 1, top = ty == P.nty - 1;
  const int Ls = cz_b > 0 ? cz_b - 1 : cz_b;     // first layer processed (z halo below the chunk)
  const int nsteps = 1 + 2 * (cz_e - Ls);        // init plane + two steps per layer
  auto col_bytes = [](int t) { return t == 0 ? 8u * 2 * HROWS : 8u * 4 * HROWS; };
  auto hl_bytes = [&](int L) { return 8u * 2 * HROWS * (HK + (L == Ls ? 1 : 0)); };
#ifdef HALO_PROF
  const int cta = blockIdx.x + gridDim.x * blockIdx.y;
#endif
  #ifdef HALO_PROF
  unsigned long long *const prof = P.prof ? P.prof + (size_t)cta * 640 : nullptr;
#else
  constexpr unsigned long long *prof = nullptr;
#endif
  if (prof && tid == 0) prof[0] = gtimer();

  // ---- init: zero the exchange slots (stay 0 where there is no neighbour), barriers, and the
  // expected bytes of the first uses of the exchange slots
  for (int i = tid; i < DCOL * COL_SLOT + DHL * HL_SLOT + NS * US_STAGE; i += HNT) COL[i] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      bar_init(b_full + 8 * b, HROWS);  // one elected arrival per warp
      bar_init(b_empty + 8 * b, HROWS);
    }
    for (int s = 0; s < DCOL; ++s) bar_init(b_col + 8 * s, 1);
    for (int s = 0; s < DHL; ++s) bar_init(b_hl + 8 * s, 1);

    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (!last_x)
      for (int s = 0; s < DCOL && s < nsteps; ++s) bar_expect(b_col + 8 * s, col_bytes(s));
    if (rank > 0)
      for (int s = 0; s < DHL && Ls + s < cz_e; ++s) bar_expect(b_hl + 8 * s, hl_bytes(Ls + s));
  }
  if (clu) cluster_barrier();
  else __syncthreads();

  if (w >= HROWS) {
    // ================= producer warps: y step =================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PROD_REGS));
    // (also the identity rows R3: dst = src on the Dirichlet nodes of the planes it loads,
    // with the values it loads anyway -- the consumers skip those nodes)
    const int yt = tid - 32 * HROWS, yc = yt & (HCOLS - 1), yj = yt >> 7;
    const int64_t gx = x0 + yc;
    const bool colin = gx < Nx, colc = ((d & 1u) && gx == 0) || ((d & 2u) && gx == Nx - 1);
    const int nrow = HK * nvy + (top ? 1 : 0);     // output node rows of the tile
    const int ncol = HK * nvx + (last_x ? 1 : 0);  // output node columns of the CTA
    uint32_t inmask = 0, consmask = 0;  // rows y0 - 4 + i inside the mesh / Dirichlet
#pragma unroll
    for (int i = 0; i < HYR; ++i) {
      const int64_t y = y0 - HK + i;
      if (colin && y >= 0 && y < Ny) inmask |= 1u << i;
      if (((d & 4u) && y == 0) || ((d & 8u) && y == Ny - 1)) consmask |= 1u << i;
    }
    const bool halo_y = ty > 0, cell1_y = nvy > 1;
    // the x+ column of a full last CTA (column 128, Dirichlet by the host check): identity
    // rows written by the two producers of column 127
    const bool col128 = ncol > HCOLS && yc == HCOLS - 1;
    const bool wslow = __any_sync(0xffffffffu, !colin || colc || consmask != 0 || col128);
    auto plane_of = [&](int t) {
      return t == 0 ? (int64_t)HK * Ls : (int64_t)HK * (Ls + (t - 1) / 2) + 1 + ((t - 1) & 1) + 2 * yj;
    };
    // step t's inputs -> stage t % NS (cp.async, one node per thread and row; rows outside the
    // mesh are never loaded: their stage slots stay 0 from the start)
    const bool allin = inmask == (1u << HYR) - 1;
    auto load = [&](int t) {
      if (t < nsteps && (t > 0 || yj == 0)) {
#ifndef HALO_NOLOAD
        const int64_t gz = plane_of(t);
        const double *s0 = src + gz * plane + (y0 - HK) * Nx + gx;
        double *st = US + (t % NS) * US_STAGE + yt;
#ifdef MF_CHECKED
        for (int i = 0; i < HYR; ++i)
          if ((inmask >> i) & 1u) HCHECK(s0 + i * Nx >= src && s0 + i * Nx < src + plane * Nz);
#endif
        if (allin) {
#pragma unroll
          for (int i = 0; i < HYR; ++i) cp_async_z<double>(st + i * 32 * HROWS, s0 + i * Nx, 8u);
        } else {
#pragma unroll
          for (int i = 0; i < HYR; ++i)
            if ((inmask >> i) & 1u) cp_async_z<double>(st + i * 32 * HROWS, s0 + i * Nx, 8u);
        }
        if (col128) {
          const double *s1 = src + gz * plane + y0 * Nx + gx + 1;
          double *c = C128 + (gz % C128_RING) * (HROWS + 1);
#pragma unroll
          for (int r = 0; r <= HROWS; ++r)
            if (r < nrow) {
              HCHECK(s1 + r * Nx >= src && s1 + r * Nx < src + plane * Nz);
              cp_async_z<double>(c + r, s1 + r * Nx, 8u);
            }
        }
#endif
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#ifdef HALO_ONLY_CONS  // (timing experiment: the producers only hand over buffers)
    for (int t = 0; t < nsteps; ++t) {
      if (t >= NB) bar_wait(b_empty + 8 * (t % NB), ((t / NB) - 1) & 1);
      __syncwarp();
      if (lane == 0) bar_arrive(b_full + 8 * (t % NB));
    }
    if (nsteps < 0)
#endif
    {
    for (int t = 0; t < NS - 1; ++t) load(t);
    for (int t = 0; t < nsteps; ++t) {
      load(t + NS - 1);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 1) : "memory");
      const int64_t gz = plane_of(t);
      const bool on = t > 0 || yj == 0;
      double u[HYR];
      {
        // rows outside the mesh are never copied (their stage rows stay 0 from the start)
        const int p0 = (int)((gz + (y0 - HK) + x0) & 1);  // Nx, plane odd: row i starts at parity p0 ^ (i & 1)
        const double *st = US + (t % NS) * US_STAGE + yt;
        (void)p0;
#pragma unroll
        for (int i = 0; i < HYR; ++i) u[i] = st[i * 32 * HROWS];
        const bool zc = ((d & 16u) && gz == 0) || ((d & 32u) && gz == Nz - 1);  // a Dirichlet z plane
        if (wslow || zc) {  // warp with columns outside the mesh, Dirichlet nodes or the x+ column
          const bool outp = gz >= (int64_t)HK * cz_b && (gz < (int64_t)HK * cz_e || (cz_e == P.ncz && gz == Nz - 1));
          if ((zc || colc || consmask) && on && outp && colin) {  // identity rows (R3) with the loaded values
            const bool skipid = P.skip_top_identity && gz == Nz - 1;
            double *d0 = dst + gz * plane + y0 * Nx + gx;
#pragma unroll
            for (int r = 0; r <= HROWS; ++r)
              if (r < nrow && yc < ncol && (zc || colc || ((consmask >> (r + HK)) & 1u))) {
                HCHECK(d0 + r * Nx >= dst && d0 + r * Nx < dst + plane * Nz);
                d0[r * Nx] = skipid ? 0.0 : u[r + HK];
              }
          }
          if (zc || colc || !colin) {
#pragma unroll
            for (int i = 0; i < HYR; ++i) u[i] = 0.0;
          } else if (consmask) {
#pragma unroll
            for (int i = 0; i < HYR; ++i)
              if ((consmask >> i) & 1u) u[i] = 0.0;
          }
        }
      }
      // y step into registers first (three independent chains: the top row of the cell below
      // from u rows 0..4, cell 0 from rows 4..8, cell 1 from rows 8..12), then the buffer
      double av[HROWS], bv[HROWS];
      {
        double e[3], o[2], f[3], g[3], ve[3], vo[2], a0[5], b0[5], a1[5], b1[5];
        double ha = 0.0, hb = 0.0;
        if (halo_y) {  // row 4 of the cell below = ve_0 - vo_0 of its even-odd product
          double he[3], ho[2];
          split5(u, he, ho);
          ha = fma(P.M.E[0][2], he[2], fma(P.M.E[0][1], he[1], P.M.E[0][0] * he[0])) -
               fma(P.M.O[0][1], ho[1], P.M.O[0][0] * ho[0]);
          hb = fma(P.K.E[0][2], he[2], fma(P.K.E[0][1], he[1], P.K.E[0][0] * he[0])) -
               fma(P.K.O[0][1], ho[1], P.K.O[0][0] * ho[0]);
          if (!ISO) hb *= ry;
        }
        split5(u + 4, e, o);
        split5(u + 8, f, g);
        mul5(P.M, e, o, ve, vo);
        comb5(ve, vo, a0);
        mul5(P.M, f, g, ve, vo);
        comb5(ve, vo, a1);
        mul5(P.K, e, o, ve, vo);
        comb5(ve, vo, b0);
        mul5(P.K, f, g, ve, vo);
        comb5(ve, vo, b1);
        if (!ISO) {
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            b0[i] *= ry;
            b1[i] *= ry;
          }
        }
        if (!cell1_y) {
#pragma unroll
          for (int i = 0; i < 5; ++i) a1[i] = b1[i] = 0.0;
        }
        av[0] = a0[0] + ha;
        bv[0] = b0[0] + hb;
#pragma unroll
        for (int r = 1; r < HK; ++r) {
          av[r] = a0[r];
          bv[r] = b0[r];
          av[HK + r] = a1[r];
          bv[HK + r] = b1[r];
        }
        av[HK] = a0[HK] + a1[0];
        bv[HK] = b0[HK] + b1[0];
      }
      const int b = t % NB;
#ifndef HALO_NOEMPTY
      if (t >= NB) bar_wait(b_empty + 8 * b, ((t / NB) - 1) & 1);
#endif
      if (prof && yt == 0 && t < 24) prof[100 + 2 * t] = gtimer();
      if (prof && lane == 0 && t >= 10 && t < 20) prof[160 + (w - HROWS) * 30 + (t - 10) * 3 + 1] = gtimer();
      if (on) {
        double *pa = AB + b * AB_BUF + yj * AB_PL + hxs(yc);
        double *pb = pa + 2 * AB_PL;
        HCHECK(pb + (HROWS - 1) * HXP < AB + NB * AB_BUF);
#pragma unroll
        for (int r = 0; r < HROWS; ++r) {
          pa[r * HXP] = av[r];
          pb[r * HXP] = bv[r];
        }
        if (yc == 0 && rank > 0) {  // column 0 -> the left CTA's column-128 slot of this step
          const int sc = t % DCOL;
          double *cs = COL + sc * COL_SLOT + yj * 2 * HROWS;
          HCHECK(cs + 2 * HROWS <= COL + DCOL * COL_SLOT);
#pragma unroll
          for (int r = 0; r < HROWS; r += 2) {
            st_async2(cs + r, b_col + 8 * sc, rank - 1, av[r], av[r + 1]);
            st_async2(cs + HROWS + r, b_col + 8 * sc, rank - 1, bv[r], bv[r + 1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(b_full + 8 * b);
      if (prof && yt == 0 && t < 24) prof[101 + 2 * t] = gtimer();
      if (prof && lane == 0 && t >= 10 && t < 20) prof[160 + (w - HROWS) * 30 + (t - 10) * 3 + 2] = gtimer();
    }
    }
  } else {
    // ================= consumer warps: x and z steps, stores =================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONS_REGS));
    const int nrow = HK * nvy + (top ? 1 : 0);     // output node rows (9: row 8 is Dirichlet, identity only)
    const int ncol = HK * nvx + (last_x ? 1 : 0);  // output node columns of this CTA
    const int xb = HK * lane + (lane >> 2);        // hxs(4 lane + i) = xb + i (i < 4)
    const int xb4 = hxs(HK * lane + HK);
    const bool partial_x = nvx < HTX, cell_ok = lane < nvx;
    double *const outw = OUT + w * OUT_W;
    const int oxl = lane + (lane >> 4);            // hxs(lane + 32 m) = oxl + 34 m
    uint32_t xcm = 0;                              // x-Dirichlet output columns of this lane
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const int64_t g = x0 + lane + 32 * m;
      if (((d & 1u) && g == 0) || ((d & 2u) && g == Nx - 1)) xcm |= 1u << m;
    }

    auto xstep = [&](int b, int j, int s, double *Pv, double *Qv) {
      const double *pa = AB + b * AB_BUF + j * AB_PL + w * HXP;
      const double *pb = pa + 2 * AB_PL;
      const double *c = COL + s * COL_SLOT + j * 2 * HROWS + w;
      double a[5], bb[5];
#pragma unroll
      for (int i = 0; i < HK; ++i) {
        a[i] = pa[xb + i];
        bb[i] = pb[xb + i];
      }
      const double *pa4 = lane == 31 ? c : pa + xb4, *pb4 = lane == 31 ? c + HROWS : pb + xb4;
      HCHECK(pb + xb < AB + NB * AB_BUF && ((lane == 31 && pb4 < COL + DCOL * COL_SLOT) ||
                                            (lane < 31 && pb4 < AB + NB * AB_BUF)));
      a[HK] = *pa4;
      bb[HK] = *pb4;
      double ea[3], oa[2], eb[3], ob[2], ve[3], vo[2];
      split5(a, ea, oa);
      split5(bb, eb, ob);
      mul5(P.K, ea, oa, ve, vo);
      acc5(P.M, eb, ob, ve, vo);
      comb5(ve, vo, Pv);
      mul5(P.M, ea, oa, ve, vo);
      comb5(ve, vo, Qv);
      if (partial_x && !cell_ok) {  // an absent cell (its inputs may hold the boundary column)
#pragma unroll
        for (int i = 0; i < 5; ++i) Pv[i] = Qv[i] = 0.0;
      }
    };
    // node 4 -> node 0 of the next lane; lane 31's -> the right CTA's x-halo slot of layer L, plane m
    auto xpass = [&](double *Pv, double *Qv, int L, int m) {
      const double p4 = __shfl_up_sync(0xffffffffu, Pv[HK], 1), q4 = __shfl_up_sync(0xffffffffu, Qv[HK], 1);
      if (lane > 0) {
        Pv[0] += p4;
        Qv[0] += q4;
      }
      if (lane == 31 && !last_x) {
        const int s = (L - Ls) % DHL;
        HCHECK(s >= 0 && (m * HROWS + w) * 2 + 1 < HL_SLOT);
        st_async2(HL + s * HL_SLOT + (m * HROWS + w) * 2, b_hl + 8 * s, rank + 1, Pv[HK], Qv[HK]);
      }
    };

    // OUT slots [0, np) of this warp's row -> dst planes gz0 .. gz0 + np - 1; Dirichlet nodes
    // are skipped (the producers write their identity values)
    const bool c128 = ncol > HCOLS && lane == 0;  // this lane writes the x+ column (Dirichlet)
    auto store = [&](int64_t gz0, int np) {
      __syncwarp();
      const int64_t y = y0 + w;
      const bool rc = ((d & 4u) && y == 0) || ((d & 8u) && y == Ny - 1);
      if (w < nrow) {
        for (int l = 0; l < np; ++l) {
          const int64_t gz = gz0 + l;
          double *const drow = dst + gz * plane + y * Nx + x0 + lane;
          HCHECK(gz >= 0 && gz < Nz && y < Ny);
          if (c128) {
            const double *c = C128 + (gz % C128_RING) * (HROWS + 1);
            const bool skipid = P.skip_top_identity && gz == Nz - 1;
            HCHECK(drow + HCOLS < dst + plane * Nz);
            drow[HCOLS] = skipid ? 0.0 : c[w];
            if (w == 0 && nrow > HROWS) drow[HROWS * Nx + HCOLS] = skipid ? 0.0 : c[HROWS];
          }
          if (rc || ((d & 16u) && gz == 0) || ((d & 32u) && gz == Nz - 1)) continue;
          const double *o = outw + l * OXP + oxl;
          if (ncol >= HCOLS && !(xcm & 15u)) {
#pragma unroll
            for (int m = 0; m < 4; ++m) drow[32 * m] = o[34 * m];
          } else {
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (lane + 32 * m < ncol && !((xcm >> m) & 1u)) drow[32 * m] = o[34 * m];
          }
        }
      }
      __syncwarp();
    };

    // z state of this lane's node columns n = 0..3 (x = 4 lane + n)
    double pc[HK] = {}, qc[HK] = {}, vc[HK] = {};  // P, Q of the layer's plane 0; v carried from below
    double ze[HK][3] = {}, zo[HK][2] = {};          // even-odd accumulators (nodes 1..3)
    double p0[HK] = {}, q0[HK] = {};                // node 0: raw P, Q of planes 1..4 (x halo one step late)

    // node 0 of layer L: add its x halo (lane 0; the left CTA's lane 31), z step, output
    auto finish_node0 = [&](int L) {
      double Pz[5], Qz[5];
      Pz[0] = pc[0];
      Qz[0] = qc[0];
#pragma unroll
      for (int m = 1; m <= HK; ++m) {
        Pz[m] = p0[m - 1];
        Qz[m] = q0[m - 1];
      }
      if (rank > 0) {
        const int s = (L - Ls) % DHL;
#ifndef HALO_ONLY_CONS
        bar_wait_cluster(b_hl + 8 * s, ((L - Ls) / DHL) & 1);
#endif
        if (lane == 0) {
          const double *h = HL + s * HL_SLOT + w * 2;
          if (L == Ls) {
            Pz[0] += h[0];
            Qz[0] += h[1];
          }
#pragma unroll
          for (int m = 1; m <= HK; ++m) {
            Pz[m] += h[m * HROWS * 2];
            Qz[m] += h[m * HROWS * 2 + 1];
          }
        }
        __syncwarp();
        if (tid == 0 && L + DHL < cz_e) bar_expect(b_hl + 8 * s, hl_bytes(L + DHL));
      }
      double e[3], o[2], f[3], g[3], ve[3], vo[2], v[5];
      split5(Pz, e, o);
      split5(Qz, f, g);
      if (!ISO) {
#pragma unroll
        for (int i = 0; i < 3; ++i) f[i] *= rz;
        g[0] *= rz;
        g[1] *= rz;
      }
      mul5(P.M, e, o, ve, vo);
      acc5(P.K, f, g, ve, vo);
      comb5(ve, vo, v);
      v[0] += vc[0];
      vc[0] = v[HK];
      pc[0] = Pz[HK];
      qc[0] = Qz[HK];
      if (L >= cz_b) {
#pragma unroll
        for (int l = 0; l < HK; ++l) outw[l * OXP + xb] = v[l];
        store((int64_t)HK * L, HK);
      }
    };

#ifdef HALO_ONLY_PROD  // (timing experiment: the consumers only hand over buffers)
    for (int t = 0; t < nsteps; ++t) {
      bar_wait(b_full + 8 * (t % NB), (t / NB) & 1);
      __syncwarp();
      if (lane == 0) bar_arrive(b_empty + 8 * (t % NB));
    }
    if (nsteps < 0)
#endif
    for (int t = 0; t <= nsteps; ++t) {
      if (t == nsteps) {  // drain: node 0 of the last layer, then the top plane of the mesh
        finish_node0(cz_e - 1);
        if (cz_e == P.ncz) {
#pragma unroll
          for (int n = 0; n < HK; ++n) outw[xb + n] = vc[n];
          store((int64_t)HK * cz_e, 1);
        }
        break;
      }
      const int b = t % NB, s = t % DCOL;
      const int L = Ls + (t - 1) / 2, h = (t - 1) & 1;
      if (prof && tid == 0 && t < 28) prof[2 + t] = gtimer();
#ifndef HALO_NOFULL
      bar_wait(b_full + 8 * b, (t / NB) & 1);
#endif
      if (prof && tid == 0 && t < 24) prof[30 + 3 * t] = gtimer();
      if (prof && lane == 0 && t >= 10 && t < 20) prof[400 + w * 30 + (t - 10) * 3] = gtimer();
#ifndef HALO_ONLY_CONS
      if (!last_x) bar_wait_cluster(b_col + 8 * s, (t / DCOL) & 1);
#endif
      if (prof && tid == 0 && t < 24) prof[31 + 3 * t] = gtimer();
      if (t == 0) {
        double Pv[5], Qv[5];
        xstep(b, 0, s, Pv, Qv);
        __syncwarp();
        if (lane == 0) bar_arrive(b_empty + 8 * b);
        if (prof && lane == 0 && t >= 10 && t < 20) prof[400 + w * 30 + (t - 10) * 3 + 1] = gtimer();
        xpass(Pv, Qv, Ls, 0);
#pragma unroll
        for (int n = 0; n < HK; ++n) {
          pc[n] = Pv[n];
          qc[n] = Qv[n];
          vc[n] = 0.0;
        }
      } else if (h == 0) {
        // x steps and the x-halo send first (the right CTA's node 0 waits for it), then node 0
        // of the previous layer
        double P1[5], Q1[5], P3[5], Q3[5];
        xstep(b, 0, s, P1, Q1);
        xstep(b, 1, s, P3, Q3);
        __syncwarp();
        if (lane == 0) bar_arrive(b_empty + 8 * b);
        if (prof && lane == 0 && t >= 10 && t < 20) prof[400 + w * 30 + (t - 10) * 3 + 1] = gtimer();
        xpass(P1, Q1, L, 1);
        xpass(P3, Q3, L, 3);
        if (L > Ls) finish_node0(L - 1);
        p0[0] = P1[0];
        q0[0] = Q1[0];
        p0[2] = P3[0];
        q0[2] = Q3[0];
#pragma unroll
        for (int n = 1; n < HK; ++n) {
          double f1 = Q1[n] + Q3[n], g1 = Q1[n] - Q3[n];
          const double e1 = P1[n] + P3[n], o1 = P1[n] - P3[n];
          if (!ISO) {
            f1 *= rz;
            g1 *= rz;
          }
#pragma unroll
          for (int i = 0; i < 3; ++i) ze[n][i] = fma(P.K.E[i][1], f1, P.M.E[i][1] * e1);
#pragma unroll
          for (int i = 0; i < 2; ++i) zo[n][i] = fma(P.K.O[i][1], g1, P.M.O[i][1] * o1);
        }
      } else {
        double P2[5], Q2[5], P4[5], Q4[5];
        xstep(b, 0, s, P2, Q2);
        xpass(P2, Q2, L, 2);
        p0[1] = P2[0];
        q0[1] = Q2[0];
#pragma unroll
        for (int n = 1; n < HK; ++n) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
            ze[n][i] = fma(P.K.E[i][2], ISO ? Q2[n] : rz * Q2[n], fma(P.M.E[i][2], P2[n], ze[n][i]));
        }
        xstep(b, 1, s, P4, Q4);
        __syncwarp();
        if (lane == 0) bar_arrive(b_empty + 8 * b);
        if (prof && lane == 0 && t >= 10 && t < 20) prof[400 + w * 30 + (t - 10) * 3 + 1] = gtimer();
        xpass(P4, Q4, L, 4);
        p0[3] = P4[0];
        q0[3] = Q4[0];
#pragma unroll
        for (int n = 1; n < HK; ++n) {
          double f0 = qc[n] + Q4[n], g0 = qc[n] - Q4[n];
          const double e0 = pc[n] + P4[n], o0 = pc[n] - P4[n];
          if (!ISO) {
            f0 *= rz;
            g0 *= rz;
          }
#pragma unroll
          for (int i = 0; i < 3; ++i) ze[n][i] = fma(P.K.E[i][0], f0, fma(P.M.E[i][0], e0, ze[n][i]));
#pragma unroll
          for (int i = 0; i < 2; ++i) zo[n][i] = fma(P.K.O[i][0], g0, fma(P.M.O[i][0], o0, zo[n][i]));
          double v[5];
          comb5(ze[n], zo[n], v);
          v[0] += vc[n];
          vc[n] = v[HK];
          pc[n] = P4[n];
          qc[n] = Q4[n];
          if (L >= cz_b) {
#pragma unroll
            for (int l = 0; l < HK; ++l) outw[l * OXP + xb + n] = v[l];
          }
        }
      }
      if (prof && tid == 0 && t < 24) prof[32 + 3 * t] = gtimer();
      if (prof && lane == 0 && t >= 10 && t < 20) prof[400 + w * 30 + (t - 10) * 3 + 2] = gtimer();
      // re-arm this step's column slot for step t + DCOL (its producer runs at most that far ahead)
      if (tid == 0 && !last_x && t + DCOL < nsteps) bar_expect(b_col + 8 * s, col_bytes(t + DCOL));
    }
  }
  if (prof && tid == 0) prof[1] = gtimer();
  if (prof && tid == 32 * HROWS) prof[159] = gtimer();  // producer warp 8 done
  // no CTA leaves while a neighbour may still deliver into its shared memory
  if (clu) cluster_barrier();
}

// ---- host side -------------------------------------------------------------------------
void eo5_from(const double A[kMaxN][kMaxN], double f, EO5 *o) {
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 2; ++j) o->E[i][j] = 0.5 * f * (A[i][j] + A[i][4 - j]);
    o->E[i][2] = f * A[i][2];
  }
  for (int j = 0; j < 2; ++j) o->E[2][j] = f * A[2][j];  // middle row acts on unhalved e_j
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) o->O[i][j] = 0.5 * f * (A[i][j] - A[i][4 - j]);
}

struct DevCache {  // per-device kernel attributes (set once per device)
  bool init = false;
  int sms = 0;
};
DevCache g_dev[64];

cudaError_t halo_prepare(int *sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DevCache &c = g_dev[dev];
  if (!c.init) {
    for (auto kern : {k_apply_halo<true>, k_apply_halo<false>}) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HSMEM);
      if (e != cudaSuccess) return e;
    }
    e = cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    c.init = true;
  }
  *sms = c.sms;
  return cudaSuccess;
}

// z-chunks of the cell layers [lo, hi): balance (clusters x waves) against the per-chunk
// halo cost (one extra layer below a chunk that starts above layer 0, plus the init plane)
void halo_chunks(int lo, int hi, int items_per_chunk, int slots, std::vector<std::pair<int, int>> *out) {
  const int n = hi - lo;
  if (n <= 0) return;
  int best = 1;
  double bestc = 1e30;
  for (int nch = 1; nch <= std::min(n, HMAXCH); ++nch) {
    const int LZ = (n + nch - 1) / nch, real = (n + LZ - 1) / LZ;
    const double waves = std::ceil((double)items_per_chunk * real / std::max(slots, 1));
    const double cost = waves * (LZ + (lo > 0 || real > 1 ? 1.25 : 0.25));
    if (cost < bestc - 1e-9) {
      bestc = cost;
      best = real;
    }
  }
  const int LZ = (n + best - 1) / best;
  for (int b = lo; b < hi; b += LZ) out->push_back({b, std::min(hi, b + LZ)});
}

}  // namespace

bool cart_halo_supported(const Geo &g) {
  if (g.dim != 3 || g.k != HK || g.geom != MF_GEOM_CARTESIAN || g.coeff_kind != MF_COEFF_CONSTANT) return false;
  if (g.nc[0] > (int64_t)HTX * HMAXCLU || g.nc[1] > (1 << 24) || g.nc[2] > (1 << 24)) return false;
  // a full last tile leaves the x+ column / y+ row of the mesh to nobody's x / y step: they
  // must be identity rows
  if (g.nc[0] % HTX == 0 && !(g.dirichlet & 2u)) return false;
  if (g.nc[1] % HTY == 0 && !(g.dirichlet & 8u)) return false;
  return true;
}

// part 0: every layer; 1: the two boundary layers (chunks [0,1) and [ncz-1, ncz)); 2: the
// interior layers; 3: the layers [zr_lo, zr_hi) only
cudaError_t launch_apply_cart_halo(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                                   int64_t *launches, int part, int zr_lo, int zr_hi) {
  if ((reinterpret_cast<uintptr_t>(src) & 15) != 0) {  // TMA bulk copies need 16-byte aligned rows
    if (part == 3) return launch_apply_cart_plane_range(g, t, src, dst, s, launches, zr_lo, zr_hi);
    return launch_apply_cart_plane(g, t, src, dst, s, launches, part);
  }
  HaloParams P;
  std::memset(&P, 0, sizeof(P));
  eo5_from(t.Mr, 1.0, &P.M);
  eo5_from(t.Kr, g.fcart[0], &P.K);
  P.ry = g.fcart[1] / g.fcart[0];
  P.rz = g.fcart[2] / g.fcart[0];
  const bool iso = g.fcart[0] == g.fcart[1] && g.fcart[0] == g.fcart[2];
  auto kern = iso ? k_apply_halo<true> : k_apply_halo<false>;
  P.Nx = g.N[0];
  P.Ny = g.N[1];
  P.Nz = g.N[2];
  P.ncx = (int)g.nc[0];
  P.ncy = (int)g.nc[1];
  P.ncz = (int)g.nc[2];
  P.ntx = (P.ncx + HTX - 1) / HTX;
  P.nty = (P.ncy + HTY - 1) / HTY;
  P.dirichlet = g.dirichlet;
  P.skip_top_identity = g.skip_top_identity;
  int sms = 0;
  cudaError_t e = halo_prepare(&sms);
  if (e != cudaSuccess) return e;
  // clusters resident at once (one CTA per SM; a cluster's CTAs share a GPC, so wide clusters
  // fit fewer times than sms / ntx)
  int slots = std::max(1, sms / P.ntx);
  {
    static int cached[HMAXCLU + 1] = {};
    if (cached[P.ntx] == 0) {
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3((unsigned)P.ntx, 1);
      qc.blockDim = dim3(HNT);
      qc.dynamicSmemBytes = HSMEM;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = (unsigned)P.ntx;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.attrs = qa;
      qc.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_apply_halo<true>, &qc) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = slots;
      }
      cached[P.ntx] = n;
    }
    slots = std::min(slots, cached[P.ntx]);
  }
  std::vector<std::pair<int, int>> ch;
  const int ncz = P.ncz;
  if (part == 0) {
    halo_chunks(0, ncz, P.nty, slots, &ch);
  } else if (part == 1) {
    ch.push_back({0, 1});
    if (ncz > 1) ch.push_back({ncz - 1, ncz});
  } else if (part == 2) {
    halo_chunks(1, ncz - 1, P.nty, slots, &ch);
  } else {
    halo_chunks(zr_lo, zr_hi, P.nty, slots, &ch);
  }
  if (ch.empty()) return cudaSuccess;
  if ((int)ch.size() > HMAXCH) return cudaErrorInvalidValue;
  P.nch = (int)ch.size();
  for (int c = 0; c < P.nch; ++c) {
    P.cz[c][0] = ch[c].first;
    P.cz[c][1] = ch[c].second;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P.ntx, (unsigned)(P.nty * P.nch));
  cfg.blockDim = dim3(HNT);
  cfg.dynamicSmemBytes = HSMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)P.ntx;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = P.ntx > 1 ? 1 : 0;
  ++*launches;
#ifdef HALO_PROF
  static const bool profile = std::getenv("MF_HALO_PROF") != nullptr;
#else
  constexpr bool profile = false;
#endif
  if (!profile) return cudaLaunchKernelEx(&cfg, kern, P, src, dst);
  // debug timeline: per-CTA start / per-step (consumer warp 0) / end, printed to stderr
  const int ncta = P.ntx * P.nty * P.nch;
  unsigned long long *dp = nullptr;
  cudaMalloc(&dp, (size_t)ncta * 640 * 8);
  cudaMemset(dp, 0, (size_t)ncta * 640 * 8);
  P.prof = dp;
  e = cudaLaunchKernelEx(&cfg, kern, P, src, dst);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h((size_t)ncta * 640);
  cudaMemcpy(h.data(), dp, h.size() * 8, cudaMemcpyDeviceToHost);
  cudaFree(dp);
  unsigned long long t0 = ~0ull, tmax = 0;
  for (int c = 0; c < ncta; ++c) t0 = std::min(t0, h[(size_t)c * 640]);
  double sum = 0;
  for (int c = 0; c < ncta; ++c) {
    tmax = std::max(tmax, h[(size_t)c * 640 + 1]);
    sum += (double)(h[(size_t)c * 640 + 1] - h[(size_t)c * 640]);
  }
  fprintf(stderr, "[halo prof] %d CTAs, %d chunks; kernel span %.1f us, mean CTA %.1f us\n", ncta, P.nch,
          (tmax - t0) / 1e3, sum / ncta / 1e3);
  {
    const int c = std::min(ncta - 1, 42);
    const unsigned long long *q = &h[(size_t)c * 640];
    fprintf(stderr, "  cta %d detail (us from its start): step: cons[full, col, done] prod[empty, full]\n", c);
    for (int t = 0; t < 24; ++t)
      fprintf(stderr, "    t=%2d cons %7.2f %7.2f %7.2f  prod %7.2f %7.2f\n", t, (q[30 + 3 * t] - q[0]) / 1e3,
              (q[31 + 3 * t] - q[0]) / 1e3, (q[32 + 3 * t] - q[0]) / 1e3, (q[100 + 2 * t] - q[0]) / 1e3,
              (q[101 + 2 * t] - q[0]) / 1e3);
  }
  {
    const int c = std::min(ncta - 1, 42);
    const unsigned long long *q = &h[(size_t)c * 640];
    const unsigned long long b0 = q[400 + 0];
    fprintf(stderr, "  cta %d per-warp steps 10..19 (us from consumer warp 0's step 10):\n", c);
    for (int w = 0; w < 16; ++w) {
      fprintf(stderr, "   %s w%2d:", w < 8 ? "cons" : "prod", w);
      for (int t = 0; t < 10; ++t) {
        const unsigned long long *r = w < 8 ? &q[400 + w * 30 + t * 3] : &q[160 + (w - 8) * 30 + t * 3];
        fprintf(stderr, " [%.2f %.2f %.2f]", ((long long)(r[0] - b0)) / 1e3, ((long long)(r[1] - b0)) / 1e3,
                ((long long)(r[2] - b0)) / 1e3);
      }
      fprintf(stderr, "\n");
    }
  }
  for (int c = 0; c < ncta; c += std::max(1, ncta / 6)) {
    const unsigned long long *q = &h[(size_t)c * 640];
    fprintf(stderr, "  cta %3d: start %7.1f end %7.1f prod-end %7.1f | steps:", c, (q[0] - t0) / 1e3, (q[1] - t0) / 1e3,
            (q[159] - t0) / 1e3);
    for (int t = 0; t < 12; ++t) fprintf(stderr, " %.1f", q[2 + t] ? (q[2 + t] - t0) / 1e3 : -1.0);
    fprintf(stderr, "\n");
  }
  return e;
}

}  // namespace mf
