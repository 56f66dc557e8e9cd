// kernels_tile.cu -- the Cartesian, constant-coefficient 3D apply ("tile" kernel).
//
// On an affine box cell with constant coefficient the Gauss(k+1) quadrature of
// a(u,v) is exact, so the cell operator of §8(a) a4-a6 (S sweeps to the Gauss
// points, collocation gradient, w_q-scaling, transposed sweeps) contracts to
// the Kronecker form ("7-sweep Kronecker"):
//     A_c = Kx' (x) M (x) M + M (x) Ky' (x) M + M (x) M (x) Kz'     (x, y, z)
// with M = S^T W S (1D reference mass) and Ke' = c prod(h)/h_e^2 * D^T W D
// (1D reference stiffness, D = Co S), both formed on the host from the same
// 1D tables the general kernel uses.  Applied as
//     a = M_z u,  b = Kz' u;   c = M_y a,  f = Ky' a + M_y b;   v = Kx' c + M_x f.
// M and K are centro-symmetric, so every 1D product uses the even-odd
// decomposition.
//
// Data flow per thread block (a tile of TX x TY cells marching through LZ
// cell layers in z), per layer:
//   phase A  thread per UNIQUE (x,y) node column of the tile: u[0] carried in a
//            register from the previous layer, u[1..k] prefetched one layer
//            ahead by cp.async (HBM -> shared), a and b written to shared memory;
//   phase B  thread per (cell, z-level) slab: the y sweeps column by column and
//            the x sweeps accumulated in even-odd form, all in registers; the
//            (k+1)^2 slab result written to shared memory;
//   phase C  the same slab thread gathers the nodes it OWNS (local index < k in
//            x and y, plus the tile's last row/column) from its own slab and the
//            left / lower / diagonal neighbour slabs (compile-time offsets), adds
//            the z-carry of the shared plane (double-buffered in shared memory)
//            and stores.
// Nodes on internal tile edges and chunk planes are shared with other blocks:
// a small init kernel writes 0 there (src on Dirichlet rows) and the main
// kernel adds with FP64 atomics (REDG); every other node is written once with
// a plain store -- no full-vector zero fill, no atomics on ~88 % of the nodes.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tile_common.cuh"

namespace mf {

// Debug instrumentation (MF_TILE_PROF=1 in the environment): per-phase clock64
// sums of threads 0 and 128, printed by the host every 20 launches.  With the
// variable unset P.prof is null and each mark is one uniform branch.
#define MF_PROF_MARK(i)                                                                    \
  do {                                                                                     \
    if (P.prof && (threadIdx.x == 0 || threadIdx.x == 128)) {                              \
      const long long c_ = clock64();                                                      \
      atomicAdd(P.prof + (threadIdx.x / 128) * 8 + (i), (unsigned long long)(c_ - prof_last)); \
      prof_last = c_;                                                                      \
    }                                                                                      \
  } while (0)

// ---- layout ------------------------------------------------------------------
template <int K, int TX, int TY>
struct TileShape {
  static constexpr int N = K + 1;
  static constexpr int NXc = K * TX + 1, NYc = K * TY + 1, NCOL = NXc * NYc;
  static constexpr int PX = NXc;              // row pitch of a / b (column id = y * PX + x)
  static constexpr int LVL = (NYc * PX) | 1;  // odd level pitch: 4 cells x 4 levels hit 16 distinct banks
  static constexpr int NSLAB = TX * TY * N;   // slab id = x-cell + TX (level + N y-cell)
  static constexpr int NT = ((NSLAB + 31) / 32) * 32;
  static constexpr int CPT = (NCOL + NT - 1) / NT;  // unique columns per thread (phase A)
  static constexpr int STAGE = CPT * (K + 1) * NT;  // cp.async staging of the next layer (+ bottom plane)
  static constexpr int CARRY = 2 * TX * TY * N * N; // double-buffered z-carry of the owned nodes
  static constexpr int EDGE = NSLAB * (2 * K + 1);  // right column + top row of every slab
  static constexpr size_t SMEM = sizeof(double) * (2 * N * LVL + EDGE + STAGE + CARRY);
};

// ---- main kernel ---------------------------------------------------------------
template <int K, int TX, int TY, bool ISO>
__global__ void __launch_bounds__(TileShape<K, TX, TY>::NT, 2)
    k_apply_tile(const __grid_constant__ TileParams P, const double *__restrict__ src, double *__restrict__ dst) {
  using S = TileShape<K, TX, TY>;
  constexpr int N = S::N, NXc = S::NXc, PX = S::PX, LVL = S::LVL, CPT = S::CPT, NT = S::NT;
  constexpr int m = N / 2, h = (N + 1) / 2;
  extern __shared__ double sm[];
  double *As = sm, *Bs = sm + N * LVL, *Es = sm + 2 * N * LVL;
  double *Ss = Es + S::EDGE, *Cb = Ss + S::STAGE;

  // Persistent blocks: work item = (tile, z-chunk), items b, b + gridDim.x, ...;
  // the first layer (and bottom plane) of the next item is prefetched during
  // the last layer of the current one, so the HBM pipeline never drains.
  const int ntile = P.ntx * P.nty, nitems = ntile * P.nch;
  const int Nx = (int)P.Nx;
  const int64_t plane = P.Nx * P.Ny;
  const uint32_t d = P.dirichlet;
  const int tid = threadIdx.x;
  const bool z_lo_c = (d & 16u) != 0, z_hi_c = (d & 32u) != 0;
  const int scx = tid % TX, sl = (tid / TX) % N, scy = tid / (TX * N);  // slab of this thread (phases B, C)

  struct Item {
    int tx, ty, chunk, cx0, cy0, nvx, nvy, cz_begin, cz_end;
    int64_t base0;  // node (K cx0, K cy0, K cz_begin); all in-item offsets are 32-bit
  };
  auto item_of = [&](int it) {
    Item I;
    const int tile = it % ntile;
    I.chunk = it / ntile;
    I.tx = tile % P.ntx;
    I.ty = tile / P.ntx;
    I.cx0 = TX * I.tx;
    I.cy0 = TY * I.ty;
    I.nvx = min(TX, P.ncx - I.cx0);  // valid cells of the tile
    I.nvy = min(TY, P.ncy - I.cy0);
    I.cz_begin = I.chunk * P.LZ;
    I.cz_end = min(I.cz_begin + P.LZ, P.ncz);
    I.base0 = (int64_t)K * I.cz_begin * plane + (int64_t)K * I.cy0 * P.Nx + (int64_t)K * I.cx0;
    return I;
  };
  // phase-A column bookkeeping of an item: in-plane offset (y Nx + x), load flag
  int coff[CPT];
  unsigned ldmask = 0;
  auto columns_of = [&](const Item &I) {
    ldmask = 0;
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const int col = tid + r * NT;
      const int x = col % NXc, y = col / NXc;
      const int gx = K * I.cx0 + x, gy = K * I.cy0 + y;
      const bool valid = col < S::NCOL && x <= K * I.nvx && y <= K * I.nvy;
      const bool cons = ((d & 1u) && gx == 0) || ((d & 2u) && gx == Nx - 1) || ((d & 4u) && gy == 0) ||
                        ((d & 8u) && gy == (int)P.Ny - 1);
      coff[r] = y * Nx + x;
      if (valid && !cons) ldmask |= 1u << r;
    }
  };
  // cp.async of node planes l0..K of layer cz of item I into this thread's private slots
  auto prefetch = [&](const Item &I, int cz, int l0) {
    const double *sp = src + I.base0 + (int64_t)K * (cz - I.cz_begin) * plane;
    const int64_t gzb = (int64_t)K * cz;
#pragma unroll
    for (int l = 0; l <= K; ++l) {
      if (l < l0) continue;
      const bool zc = (z_lo_c && gzb + l == 0) || (z_hi_c && gzb + l == P.Nz - 1);
      const double *spl = sp + l * plane;
#pragma unroll
      for (int r = 0; r < CPT; ++r) {
        // zero-fill (src-size 0) for constrained / outside columns: no branch, no STS
        const bool ok = ((ldmask >> r) & 1u) && !zc;
        cp_async8z(Ss + ((r * (K + 1) + l) * NT + tid), ok ? spl + coff[r] : src, ok ? 8u : 0u);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  int item = blockIdx.x;
  if (item >= nitems) return;
  long long prof_last = clock64();
  Item G = item_of(item);
  columns_of(G);
  prefetch(G, G.cz_begin, 0);
  double ucar[CPT];

  while (true) {
  const int tx = G.tx, ty = G.ty, chunk = G.chunk, cx0 = G.cx0, cy0 = G.cy0, nvx = G.nvx, nvy = G.nvy;
  const int cz_begin = G.cz_begin, cz_end = G.cz_end;
  const int64_t base0 = G.base0;
  const int next = item + gridDim.x;
  const bool slab_ok = tid < S::NSLAB && scx < nvx && scy < nvy;
  const bool hasL = scx > 0, hasB = scy > 0;
  const bool ownR = scx == nvx - 1, ownT = scy == nvy - 1;  // owns the tile's last column / row
  const int gxs = K * (cx0 + scx), gys = K * (cy0 + scy);    // node of local (0,0)
  // shared-with-another-tile and Dirichlet flags of the owned node classes
  const bool shL = scx == 0 && tx > 0, shR = ownR && cx0 + scx + 1 < P.ncx;
  const bool shB = scy == 0 && ty > 0, shT = ownT && cy0 + scy + 1 < P.ncy;
  const bool cL = (d & 1u) && gxs == 0, cR = (d & 2u) && ownR && cx0 + scx + 1 == P.ncx;
  const bool cB = (d & 4u) && gys == 0, cT = (d & 8u) && ownT && cy0 + scy + 1 == P.ncy;
  const int soff = (K * scy) * Nx + K * scx;  // in-plane offset of the slab's node (0,0)
  double *CbMine = Cb + (scy * TX + scx) * N * N;

  for (int cz = cz_begin; cz < cz_end; ++cz) {
    MF_PROF_MARK(0);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    MF_PROF_MARK(1);
    // ---- phase A: z-sweeps on unique columns
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const int col = tid + r * NT;
      if (col < S::NCOL) {
        double u[N];
        u[0] = cz == cz_begin ? Ss[(r * (K + 1)) * NT + tid] : ucar[r];
#pragma unroll
        for (int l = 1; l <= K; ++l) u[l] = Ss[(r * (K + 1) + l) * NT + tid];
        ucar[r] = u[K];
        double e[h], o[h], ve[h], vo[h], a[N], b[N];
        eo_split<N>(u, e, o);
        eo_first<N>(P.M, e, o, ve, vo);
        eo_combine<N>(ve, vo, a);
        if (!ISO) {
#pragma unroll
          for (int q = 0; q < h; ++q) {
            e[q] *= P.rz;
            o[q] *= P.rz;
          }
        }
        eo_first<N>(P.K, e, o, ve, vo);
        eo_combine<N>(ve, vo, b);
#pragma unroll
        for (int l = 0; l < N; ++l) {
          As[l * LVL + col] = a[l];
          Bs[l * LVL + col] = b[l];
        }
      }
    }
    // in flight during phases B and C
    if (cz + 1 < cz_end) {
      prefetch(G, cz + 1, 1);
    } else if (next < nitems) {
      G = item_of(next);
      columns_of(G);
      prefetch(G, G.cz_begin, 0);
    }
    MF_PROF_MARK(2);
    __syncthreads();
    MF_PROF_MARK(3);

    // ---- phase B: y sweeps per column, x sweeps accumulated in even-odd form
    double own[2 * K - 1];  // the slab's bottom row and left column, kept for phase C
    if (tid < S::NSLAB) {
      const double *Al = As + sl * LVL + (K * scy) * PX + K * scx;
      const double *Bl = Bs + sl * LVL + (K * scy) * PX + K * scx;
      // column i of c = M_y a and f = Ky' a + M_y b
      auto colcf = [&](int i, double *c, double *f) {
        double av[N], bv[N], e[h], o[h], ve[h], vo[h];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          av[j] = Al[j * PX + i];
          bv[j] = Bl[j * PX + i];
        }
        eo_split<N>(av, e, o);
        eo_first<N>(P.M, e, o, ve, vo);
        eo_combine<N>(ve, vo, c);
        if (!ISO) {
#pragma unroll
          for (int q = 0; q < h; ++q) {
            e[q] *= P.ry;
            o[q] *= P.ry;
          }
        }
        eo_first<N>(P.K, e, o, ve, vo);
        eo_split<N>(bv, e, o);
        eo_acc<N>(P.M, e, o, ve, vo);
        eo_combine<N>(ve, vo, f);
      };
      double xe[N][h], xo[N][h > 0 ? h : 1];  // row j of v = Kx' c[j] + M f[j], even/odd along x
#pragma unroll
      for (int p = 0; p < m; ++p) {
        double c1[N], f1[N], c2[N], f2[N];
        colcf(p, c1, f1);
        colcf(N - 1 - p, c2, f2);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double ec = c1[j] + c2[j], oc = c1[j] - c2[j], ef = f1[j] + f2[j], of = f1[j] - f2[j];
#pragma unroll
          for (int r = 0; r < h; ++r) {
            const double t = p == 0 ? P.K.E[r][p] * ec : fma(P.K.E[r][p], ec, xe[j][r]);
            xe[j][r] = fma(P.M.E[r][p], ef, t);
          }
#pragma unroll
          for (int r = 0; r < m; ++r) {
            const double t = p == 0 ? P.K.O[r][p] * oc : fma(P.K.O[r][p], oc, xo[j][r]);
            xo[j][r] = fma(P.M.O[r][p], of, t);
          }
        }
      }
      if (N & 1) {
        double cm[N], fm[N];
        colcf(m, cm, fm);
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int r = 0; r < h; ++r) xe[j][r] = fma(P.M.E[r][m], fm[j], fma(P.K.E[r][m], cm[j], xe[j][r]));
      }
      // v = this slab's contribution.  Interior nodes of the slab face (no
      // neighbour shares them) leave straight from registers; the right column
      // and top row go to the edge buffer for the neighbours; the slab's own
      // left column / bottom row values wait in registers for phase C.
      const bool first = cz == cz_begin, last = cz + 1 == cz_end;
      const int par = cz & 1;
      const int64_t gz = (int64_t)K * cz + sl;
      const bool zcons = (z_lo_c && gz == 0) || (z_hi_c && gz == P.Nz - 1);
      const bool zshared = (sl == 0 && first && chunk > 0) || (sl == K && last && chunk < P.nch - 1);
      const bool cw = sl == K && !last, addc = sl == 0 && !first;
      const double *carry = Cb + (1 - par) * (TX * TY * N * N) + (scy * TX + scx) * N * N;
      double *cwrite = CbMine + par * (TX * TY * N * N);
      double *out = dst + base0 + (int64_t)K * (cz - cz_begin) * plane + sl * plane + soff;
      double *Em = Es + tid * (2 * K + 1);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double v[N];
        eo_combine<N>(xe[j], xo[j], v);
        Em[j] = v[K];                                  // right column (j = 0..K)
        if (j == K)
#pragma unroll
          for (int i = 0; i < K; ++i) Em[K + 1 + i] = v[i];  // top row (i = 0..K-1)
        if (j == 0)
#pragma unroll
          for (int i = 0; i < K; ++i) own[i] = v[i];         // bottom row (i = 0..K-1)
        if (j > 0 && j < K) {
          own[K + j - 1] = v[0];                       // left column (j = 1..K-1)
          if (slab_ok) {
#pragma unroll
            for (int i = 1; i < K; ++i) {
              double s = v[i];
              if (cw) {
                cwrite[j * N + i] = s;
              } else if (!zcons) {
                if (addc) s += carry[j * N + i];
                if (zshared) atomicAdd(out + j * Nx + i, s);
                else out[j * Nx + i] = s;
              }
            }
          }
        }
      }
    }
    MF_PROF_MARK(4);
    __syncthreads();
    MF_PROF_MARK(5);

    // ---- phase C: the slab's owned edge nodes (left column, bottom row, and the
    // tile's last column / row), summed with the neighbour slabs' edges
    if (slab_ok) {
      const double *EL = Es + (tid - 1) * (2 * K + 1), *EB = Es + (tid - TX * N) * (2 * K + 1);
      const double *EM = Es + tid * (2 * K + 1), *ELB = EB - (2 * K + 1);
      const bool first = cz == cz_begin, last = cz + 1 == cz_end;
      const int par = cz & 1;
      const int64_t gz = (int64_t)K * cz + sl;
      const bool zcons = (z_lo_c && gz == 0) || (z_hi_c && gz == P.Nz - 1);
      const bool zshared = (sl == 0 && first && chunk > 0) || (sl == K && last && chunk < P.nch - 1);
      const double *carry = Cb + (1 - par) * (TX * TY * N * N) + (scy * TX + scx) * N * N;
      double *cwrite = CbMine + par * (TX * TY * N * N);
      double *out = dst + base0 + (int64_t)K * (cz - cz_begin) * plane + sl * plane + soff;
      auto emit = [&](int i, int j, double s) {
        if (sl == 0 && !first) s += carry[j * N + i];
        if (sl == K && !last) {
          cwrite[j * N + i] = s;  // level K becomes level 0 of the next layer
          return;
        }
        const bool cons = zcons || (i == 0 && cL) || (i == K && cR) || (j == 0 && cB) || (j == K && cT);
        if (cons) return;
        const bool shared = zshared || (i == 0 && shL) || (i == K && shR) || (j == 0 && shB) || (j == K && shT);
        double *p = out + j * Nx + i;
        if (shared) atomicAdd(p, s);
        else *p = s;
      };
      // bottom row j = 0, i = 0..K-1 (the corner (0,0) also gets the left / diagonal slabs)
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double s = own[i];
        if (hasB) s += EB[K + 1 + i];
        if (i == 0 && hasL) s += EL[0];
        if (i == 0 && hasL && hasB) s += ELB[K];
        emit(i, 0, s);
      }
      // left column i = 0, j = 1..K-1
#pragma unroll
      for (int j = 1; j < K; ++j) emit(0, j, own[K + j - 1] + (hasL ? EL[j] : 0.0));
      if (ownR) {  // the tile's last column: i = K, j = 0..K-1
#pragma unroll
        for (int j = 0; j < K; ++j) emit(K, j, EM[j] + (j == 0 && hasB ? EB[K] : 0.0));
      }
      if (ownT) {  // the tile's last row: j = K, i = 0..K-1
#pragma unroll
        for (int i = 0; i < K; ++i) emit(i, K, EM[K + 1 + i] + (i == 0 && hasL ? EL[K] : 0.0));
      }
      if (ownR && ownT) emit(K, K, EM[K]);
    }
  }
  MF_PROF_MARK(6);
  if (next >= nitems) break;
  item = next;  // G, coff, ldmask already describe it (set at the last prefetch)
  }
}

bool cart_tile_supported(const Geo &g) {
  return g.dim == 3 && g.geom == MF_GEOM_CARTESIAN && g.coeff_kind == MF_COEFF_CONSTANT &&
         (g.k == 2 || g.k == 3 || g.k == 4);
}

template <int K, int TX, int TY, bool ISO>
static cudaError_t launch_tile_t(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                                 int64_t *launches) {
  using S = TileShape<K, TX, TY>;
  TileParams P;
  tile_params_common(g, t, TX, TY, &P);
  static int occ = 0, sms = 0;
  if (occ == 0) {
    cudaFuncSetAttribute(k_apply_tile<K, TX, TY, ISO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply_tile<K, TX, TY, ISO>, S::NT, S::SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (occ < 1) occ = 1;
    if (sms < 1) sms = 148;
  }
  const int slots = sms * occ;
  tile_choose_chunks(&P, slots, 0.5);
  cudaError_t e = tile_launch_init(P, g, K, TX, TY, src, dst, s, launches);
  if (e != cudaSuccess) return e;
  ++*launches;
  static unsigned long long *prof = nullptr;
  static int prof_calls = 0;
  if (getenv("MF_TILE_PROF")) {
    if (!prof) {
      cudaMalloc(&prof, 16 * sizeof(unsigned long long));
      cudaMemset(prof, 0, 16 * sizeof(unsigned long long));
    }
    P.prof = prof;
    if (++prof_calls % 20 == 0) {
      unsigned long long h[16];
      cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
      for (int q = 0; q < 2; ++q)
        printf("tile prof thread %d: C+loop %llu wait %llu A %llu bar1 %llu B %llu bar2 %llu item-end %llu\n",
               q * 128, h[q * 8 + 0], h[q * 8 + 1], h[q * 8 + 2], h[q * 8 + 3], h[q * 8 + 4], h[q * 8 + 5],
               h[q * 8 + 6]);
      cudaMemset(prof, 0, sizeof(h));
    }
  }
  const int items = P.ntx * P.nty * P.nch;
  const int blocks = std::min(items, slots);  // persistent: each block walks items blockIdx.x + i * gridDim.x
  k_apply_tile<K, TX, TY, ISO><<<blocks, S::NT, S::SMEM, s>>>(P, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_apply_cart_tile(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                                   int64_t *launches) {
  // MF_TILE=<TX>x<TY> selects an alternative tile shape (experiments; default 8x4)
  static int shape = -1;
  if (shape < 0) {
    const char *e = getenv("MF_TILE");
    shape = 1;
    if (e && !strcmp(e, "4x8")) shape = 0;
    if (e && !strcmp(e, "16x2")) shape = 2;
  }
  const bool iso = g.fcart[0] == g.fcart[1] && g.fcart[0] == g.fcart[2];
#define MF_TILE_LAUNCH(KK, TXX, TYY)                                              \
  return iso ? launch_tile_t<KK, TXX, TYY, true>(g, t, src, dst, s, launches)     \
             : launch_tile_t<KK, TXX, TYY, false>(g, t, src, dst, s, launches)
  switch (g.k) {
    case 2: MF_TILE_LAUNCH(2, 8, 8);
    case 3: MF_TILE_LAUNCH(3, 8, 4);
    case 4:
      if (shape == 0) MF_TILE_LAUNCH(4, 4, 8);
      if (shape == 2) MF_TILE_LAUNCH(4, 16, 2);
      MF_TILE_LAUNCH(4, 8, 4);
  }
#undef MF_TILE_LAUNCH
  return cudaErrorNotSupported;
}

}  // namespace mf
