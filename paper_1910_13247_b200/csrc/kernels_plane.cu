// kernels_plane.cu -- Cartesian, constant-coefficient 3D apply in "2D first, z last"
// form (apply variant 3, the default for k = 2..4).
//
// The cell operator of the affine box cell is the Gauss(k+1)-exact Kronecker form
//
//     A_c = [Kx' (x) My + Mx (x) Ky'] (x) Mz  +  [Mx (x) My] (x) Kz'     (x, y | z)
// so with the x-y operators applied on every DoF plane p and summed over the
// cells that share a node in x-y,
//     P_p = sum_{cells} (Kx' (x) M + M (x) Ky') u_p,      Q_p = sum_{cells} (M (x) M) u_p,
// the result is a 1D operator in z per node column:
//     v = sum_{z-cells} (Mz P + Kz' Q).
// P and Q are computed ONCE per DoF plane (k planes per cell layer instead of
// the k+1 z-levels of the slab form), the z-sweep runs in registers of one
// thread per node column, and nothing but u, P and Q goes through shared
// memory: ~40 FP64 instructions and ~8 shared-memory accesses per DoF.
//
// Per thread block: a tile of TX x TY cells marching through a z-chunk of cell
// layers (persistent blocks walk (tile, chunk) items).  Per layer:
//   face phase    thread per (cell, plane p = 1..k): u_p on the cell face from the
//                 cp.async stage, y sweeps column by column, x sweeps row by row,
//                 even-odd; P and Q of the face written to shared memory;
//   column phase  thread per (cell, row j): the k node columns (i = 0..k-1, j) the
//                 cell owns -- the gather of P and Q from the own / left / lower /
//                 diagonal face is compile-time in i -- plus one of the tile's
//                 right-edge / top-edge columns; prefetch of the next layer
//                 (cp.async), z-sweep in even-odd form with the plane-0 values
//                 carried from the previous layer, store the k finished planes.
// Shared tile-edge / chunk-plane nodes: init kernel + FP64 atomics (tile_common.cuh).
#include <cstdlib>
#include <cstring>

#include "tile_common.cuh"

namespace mf {

template <int K, int TX, int TY>
struct PlaneShape {
  static constexpr int N = K + 1;
  static constexpr int NXc = K * TX + 1, NYc = K * TY + 1, NCOL = NXc * NYc;
  static constexpr int NCELL = TX * TY;
  static constexpr int NT = NCELL * K;          // face phase: (cell, p = 1..K); column phase: (cell, j)
  static_assert(NT % 32 == 0, "tile must give whole warps");
  static_assert(NXc + NYc - 1 <= NT, "one edge column per thread");
  // stage layout: node x of a row sits at XS(x) = x + x / 16 (a pad double every 16 nodes), the
  // row pitch is NXp and the plane pitch SPL = 2 (mod 16): the face phase's warp (8 cells 4
  // nodes apart x 4 planes) then hits 16 distinct bank pairs per half-warp (FP64)
  static constexpr int XS(int x) { return x + (x >> 4); }
  static constexpr int NXp = XS(NXc - 1) + 1;
  static constexpr int SPL = NXp * NYc + ((2 - (NXp * NYc) % 16) + 16) % 16;  // stage plane pitch
  static constexpr int STG = N * SPL;           // u on planes 0..K of a layer
  static constexpr int FACE = N * N;
  static constexpr int NV = NCELL * N * FACE;   // P (or Q): faces of planes 0..K
  template <class T>
  static constexpr size_t smem() { return sizeof(T) * (STG + 2 * NV); }
};

template <int K, int TX, int TY, bool ISO, class T>
__global__ void __launch_bounds__(PlaneShape<K, TX, TY>::NT, sizeof(T) == 8 ? 2 : 3)
    k_apply_plane(const __grid_constant__ TileParams P, const T *__restrict__ src, T *__restrict__ dst) {
  using S = PlaneShape<K, TX, TY>;
  constexpr int N = S::N, NXp = S::NXp, NCELL = S::NCELL, SPL = S::SPL, FACE = S::FACE;
  constexpr int h = (N + 1) / 2;
  constexpr int PSTRIDE = TX * FACE;       // face slot of (cx, cy, p) = cx + TX (p + N cy)
  constexpr int YSTRIDE = TX * N * FACE;   // cy -> cy + 1
  extern __shared__ __align__(16) unsigned char smraw[];
  T *const sm = reinterpret_cast<T *>(smraw);
  T *Us = sm, *Vp = sm + S::STG, *Vq = Vp + S::NV;
  const EOMatT<T> &Mm = tp_M<T>(P), &Km = tp_K<T>(P);
  const T ry = (T)P.ry, rz = (T)P.rz;

  const int ntile = P.ntx * P.nty, nitems = ntile * tile_pass_chunks(P);
  const int Nx = (int)P.Nx, Ny = (int)P.Ny;
  const int64_t plane = P.Nx * P.Ny;
  const uint32_t d = P.dirichlet;
  const int tid = threadIdx.x;
  const bool z_lo_c = (d & 16u) != 0, z_hi_c = (d & 32u) != 0;
  // face phase: (x-cell fastest, then plane, then y-cell)
  const int fcx = tid % TX, fp = 1 + (tid / TX) % K, fcy = tid / (TX * K);
  // column phase: cell c = (ccx, ccy) and row jr of its owned columns
  const int cc = tid % NCELL, jr = tid / NCELL, ccx = cc % TX, ccy = cc / TX;

  struct Item {
    int tx, ty, chunk, cx0, cy0, nvx, nvy, cz_begin, cz_end;
    int64_t base0;
  };
  auto item_of = [&](int it) {
    Item I;
    const int tile = it % ntile;
    I.chunk = tile_pass_chunk(P, it / ntile);
    I.tx = tile % P.ntx;
    I.ty = tile / P.ntx;
    I.cx0 = TX * I.tx;
    I.cy0 = TY * I.ty;
    I.nvx = min(TX, P.ncx - I.cx0);
    I.nvy = min(TY, P.ncy - I.cy0);
    tile_chunk_layers(P, I.chunk, I.cz_begin, I.cz_end);
    I.base0 = (int64_t)K * I.cz_begin * plane + (int64_t)K * I.cy0 * P.Nx + (int64_t)K * I.cx0;
    return I;
  };
  // this thread's edge column of an item: tile right edge x = K nvx (e <= K nvy),
  // then the top edge y = K nvy (x < K nvx); -1 if none
  auto edge_xy = [&](const Item &I, int &x, int &y) {
    const int nr = K * I.nvy + 1, ne = nr + K * I.nvx;
    if (tid >= ne) return false;
    if (tid < nr) {
      x = K * I.nvx;
      y = tid;
    } else {
      x = tid - nr;
      y = K * I.nvy;
    }
    return true;
  };
  auto xy_cons = [&](const Item &I, int x, int y) {
    const int gx = K * I.cx0 + x, gy = K * I.cy0 + y;
    return ((d & 1u) && gx == 0) || ((d & 2u) && gx == Nx - 1) || ((d & 4u) && gy == 0) ||
           ((d & 8u) && gy == Ny - 1);
  };

  // cp.async of node planes l0..K of layer cz of item I (this thread's columns) into the stage
  // (constrained nodes are zero-filled: their addresses are valid vector entries,
  // only the byte count drops to 0)
  auto prefetch = [&](const Item &I, int cz, int l0) {
    const T *sp0 = src + I.base0 + (int64_t)K * (cz - I.cz_begin) * plane;
    const bool zlo = z_lo_c && cz == 0, zhi = z_hi_c && cz == P.ncz - 1;  // planes l = 0 / l = K
    const bool own_ok = ccx < I.nvx && ccy < I.nvy;
    const int y = K * ccy + jr;
    const bool ycons = (d & 4u) && K * I.cy0 + y == 0;
    const bool xcons0 = (d & 1u) && K * (I.cx0 + ccx) == 0;  // the cell's i = 0 column on the x- face
    int ex = 0, ey = 0;
    const bool has_e = edge_xy(I, ex, ey);
    const bool e_ok = has_e && !xy_cons(I, ex, ey);
    const T *go = sp0 + y * Nx + K * ccx, *ge = sp0 + ey * Nx + ex;
    T *so = Us + y * NXp, *se = Us + ey * NXp + S::XS(ex);
#pragma unroll
    for (int l = 0; l <= K; ++l) {
      if (l >= l0) {
        const bool zc = (l == 0 && zlo) || (l == K && zhi);
        if (own_ok) {
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const bool ok = !zc && !ycons && !(i == 0 && xcons0);
            cp_async_z<T>(so + l * SPL + S::XS(K * ccx + i), go + i, ok ? 8u : 0u);
          }
        }
        if (has_e) cp_async_z<T>(se + l * SPL, ge, (e_ok && !zc) ? 8u : 0u);
      }
      go += plane;
      ge += plane;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  // ---- face: P and Q on the face of cell (fcx, fcy) at plane p from u on that plane
  auto face = [&](int p) {
    const T *Ul = Us + p * SPL + (K * fcy) * NXp;
    T *Pf = Vp + (fcx + TX * (p + N * fcy)) * FACE, *Qf = Vq + (fcx + TX * (p + N * fcy)) * FACE;
    T c[N][N], g[N][N];  // [j][i]: c = M_y u, g = Ky' u
#pragma unroll
    for (int i = 0; i < N; ++i) {
      T uv[N], e[h], o[h], ve[h], vo[h], t[N];
#pragma unroll
      for (int j = 0; j < N; ++j) uv[j] = Ul[j * NXp + S::XS(K * fcx + i)];
      eo_split<N>(uv, e, o);
      eo_first<N>(Mm, e, o, ve, vo);
      eo_combine<N>(ve, vo, t);
#pragma unroll
      for (int j = 0; j < N; ++j) c[j][i] = t[j];
      if (!ISO) {
#pragma unroll
        for (int q = 0; q < h; ++q) {
          e[q] *= ry;
          o[q] *= ry;
        }
      }
      eo_first<N>(Km, e, o, ve, vo);
      eo_combine<N>(ve, vo, t);
#pragma unroll
      for (int j = 0; j < N; ++j) g[j][i] = t[j];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      T ec[h], oc[h], eg[h], og[h], ve[h], vo[h], t[N];
      eo_split<N>(c[j], ec, oc);
      eo_split<N>(g[j], eg, og);
      eo_first<N>(Km, ec, oc, ve, vo);  // P = Kx' c + Mx g
      eo_acc<N>(Mm, eg, og, ve, vo);
      eo_combine<N>(ve, vo, t);
#pragma unroll
      for (int i = 0; i < N; ++i) Pf[j * N + i] = t[i];
      eo_first<N>(Mm, ec, oc, ve, vo);  // Q = Mx c
      eo_combine<N>(ve, vo, t);
#pragma unroll
      for (int i = 0; i < N; ++i) Qf[j * N + i] = t[i];
    }
  };

  // ---- z-sweep of one column: v = Mz P + Kz' Q (even-odd), carries, stores
  // zm / am: the layer's planes l that are z-constrained / shared with the
  // neighbouring z-chunk (bit l, warp-uniform)
  auto zcolumn = [&](const T *pb, const T *qb, T &vcar, bool first, bool last, bool cons, bool shared,
                     T *out, uint32_t zm, uint32_t am) {
    T e[h], o[h], ve[h], vo[h], v[N];
    eo_split<N>(pb, e, o);
    eo_first<N>(Mm, e, o, ve, vo);
    eo_split<N>(qb, e, o);
    if (!ISO) {
#pragma unroll
      for (int q = 0; q < h; ++q) {
        e[q] *= rz;
        o[q] *= rz;
      }
    }
    eo_acc<N>(Km, e, o, ve, vo);
    eo_combine<N>(ve, vo, v);
    if (!first) v[0] += vcar;
    vcar = v[K];
    if (cons) return;
#pragma unroll
    for (int l = 0; l <= K; ++l) {
      if (l == K && !last) break;  // carried to the next layer
      if (!((zm >> l) & 1u)) {
        // predicated red / st, no divergent branch (shared varies across lanes)
        const int at = (shared || ((am >> l) & 1u)) ? 1 : 0;
        red_or_st(out, v[l], at);
      }
      out += plane;
    }
  };

  int item = blockIdx.x;
  if (item >= nitems) return;
  Item G = item_of(item);
  prefetch(G, G.cz_begin, 0);
  T pcar[K + 1], qcar[K + 1], vcar[K + 1];  // owned columns i = 0..K-1, [K] = edge column
  bool dep_done = false;

  while (true) {
    const int cz_begin = G.cz_begin, cz_end = G.cz_end, chunk = G.chunk;
    const int64_t base0 = G.base0;
    const int next = item + gridDim.x;
    const bool face_ok = fcx < G.nvx && fcy < G.nvy;
    // owned columns (i, jr) of cell (ccx, ccy)
    const bool own_ok = ccx < G.nvx && ccy < G.nvy;
    const bool hasL = ccx > 0, hasB = ccy > 0 && jr == 0;
    const int yown = K * ccy + jr;
    const bool ycons = (d & 4u) && K * G.cy0 + yown == 0;
    const bool xcons0 = (d & 1u) && K * (G.cx0 + ccx) == 0;
    const bool shx0 = ccx == 0 && G.tx > 0, shy = jr == 0 && ccy == 0 && G.ty > 0;
    const int own0 = (ccx + YSTRIDE / FACE * ccy) * FACE + jr * N;  // face offset of (i = 0, jr), plane 0
    // the edge column: faces of the tile containing it
    int ex = 0, ey = 0;
    const bool has_e = edge_xy(G, ex, ey);
    bool e_cons = false, e_sh = false;
    int eo[4] = {-1, -1, -1, -1};
    if (has_e) {
      e_cons = xy_cons(G, ex, ey);
      const int gx = K * G.cx0 + ex, gy = K * G.cy0 + ey;
      e_sh = (ex == 0 && G.tx > 0) || (ex == K * G.nvx && gx < Nx - 1) || (ey == 0 && G.ty > 0) ||
             (ey == K * G.nvy && gy < Ny - 1);
      const int cxa = ex / K - (ex % K == 0 ? 1 : 0), cxb = min(ex / K, G.nvx - 1);
      const int cya = ey / K - (ey % K == 0 ? 1 : 0), cyb = min(ey / K, G.nvy - 1);
      int n = 0;
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const int cx = a == 0 ? cxa : cxb, cy = b == 0 ? cya : cyb;
          const bool ok = cx >= 0 && cy >= 0 && (a == 0 || cxb != cxa) && (b == 0 || cyb != cya);
          if (ok) {
            const int o = (cx + TX * N * cy) * FACE + (ey - K * cy) * N + (ex - K * cx);
            if (n == 0) eo[0] = o;
            else if (n == 1) eo[1] = o;
            else if (n == 2) eo[2] = o;
            else eo[3] = o;
            ++n;
          }
        }
    }

    for (int cz = cz_begin; cz < cz_end; ++cz) {
      const bool first = cz == cz_begin, last = cz + 1 == cz_end;
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      // ---- face phase
      if (face_ok) {
        face(fp);
        if (first && fp == 1) face(0);  // the chunk's bottom plane (once per item)
      }
      __syncthreads();
      // ---- column phase: prefetch the next layer, then gather P, Q and sweep in z
      if (!dep_done) {  // the init grid (zeroed shared planes, identity rows) is complete
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        dep_done = true;
      }
      if (!last) {
        prefetch(G, cz + 1, 1);
      } else if (next < nitems) {
        prefetch(item_of(next), item_of(next).cz_begin, 0);
      }
      const uint32_t zm = ((z_lo_c && cz == 0) ? 1u : 0u) | ((z_hi_c && cz == P.ncz - 1) ? 1u << K : 0u);
      const uint32_t am = ((first && (chunk > 0 || P.lo_shared)) ? 1u : 0u) |
                          ((last && (chunk < P.nch - 1 || P.hi_shared)) ? 1u << K : 0u);
      T *outl = dst + base0 + (int64_t)K * (cz - cz_begin) * plane;
      if (own_ok) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          T pb[N], qb[N];
#pragma unroll
          for (int p = 0; p < N; ++p) {
            if (p == 0 && !first) {
              pb[0] = pcar[i];
              qb[0] = qcar[i];
              continue;
            }
            const int o = own0 + p * PSTRIDE + i;
            T sp_ = Vp[o], sq_ = Vq[o];
            if (i == 0 && hasL) {  // left face, its local (K, jr)
              sp_ += Vp[o - FACE + K];
              sq_ += Vq[o - FACE + K];
            }
            if (hasB) {  // lower face, its local (i, K)
              sp_ += Vp[o - YSTRIDE + K * N];
              sq_ += Vq[o - YSTRIDE + K * N];
              if (i == 0 && hasL) {  // diagonal face, its local (K, K)
                sp_ += Vp[o - YSTRIDE - FACE + K * N + K];
                sq_ += Vq[o - YSTRIDE - FACE + K * N + K];
              }
            }
            pb[p] = sp_;
            qb[p] = sq_;
          }
          pcar[i] = pb[K];
          qcar[i] = qb[K];
          const bool cons = ycons || (i == 0 && xcons0), shared = shy || (i == 0 && shx0);
          zcolumn(pb, qb, vcar[i], first, last, cons, shared, outl + yown * Nx + K * ccx + i, zm, am);
        }
      }
      if (has_e) {
        T pb[N], qb[N];
#pragma unroll
        for (int p = 0; p < N; ++p) {
          if (p == 0 && !first) {
            pb[0] = pcar[K];
            qb[0] = qcar[K];
            continue;
          }
          T sp_ = 0.0, sq_ = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (eo[q] >= 0) {
              sp_ += Vp[eo[q] + p * PSTRIDE];
              sq_ += Vq[eo[q] + p * PSTRIDE];
            }
          pb[p] = sp_;
          qb[p] = sq_;
        }
        pcar[K] = pb[K];
        qcar[K] = qb[K];
        zcolumn(pb, qb, vcar[K], first, last, e_cons, e_sh, outl + ey * Nx + ex, zm, am);
      }
    }
    if (next >= nitems) break;
    item = next;
    G = item_of(item);
  }
}

// part 0: init + every chunk; part 1: init + the two boundary chunks of the z-split;
// part 2: the interior chunks of the z-split (see TileParams::zsplit)
// part 3: init + the cell layers [zr_lo, zr_hi) only (the pipelined host apply)
template <int K, int TX, int TY, bool ISO, class T>
static cudaError_t launch_plane_t(const Geo &g, const Tables &t, const T *src, T *dst, cudaStream_t s,
                                  int64_t *launches, int part, int zr_lo = 0, int zr_hi = 0) {
  using S = PlaneShape<K, TX, TY>;
  TileParams P;
  tile_params_common(g, t, TX, TY, &P);
  static int occ_d[kMaxDevices] = {}, sms_d[kMaxDevices] = {};  // per device
  const int dev = current_device();
  int &occ = occ_d[dev], &sms = sms_d[dev];
  if (occ == 0) {
    cudaFuncSetAttribute(k_apply_plane<K, TX, TY, ISO, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S::template smem<T>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_apply_plane<K, TX, TY, ISO, T>, S::NT, S::template smem<T>());
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (occ < 1) occ = 1;
    if (sms < 1) sms = 148;
  }
  const int slots = sms * occ;
  // the bottom plane costs one extra face per cell
  if (part == 0) {
    tile_choose_chunks(&P, slots, 1.0 / K + 0.25);
  } else if (part == 3) {
    TileParams Q = P;
    Q.ncz = zr_hi - zr_lo;
    tile_choose_chunks(&Q, slots, 1.0 / K + 0.25);
    P.LZ = Q.LZ;
    P.nch = Q.nch;
    P.zr_lo = zr_lo;
    P.zr_hi = zr_hi;
    P.lo_shared = zr_lo > 0;
    P.hi_shared = zr_hi < P.ncz;
  } else {
    tile_choose_chunks_split(&P, slots, 1.0 / K + 0.25);
  }
  P.pass = part;
  if (part != 2) {
    cudaError_t e = tile_launch_init(P, g, K, TX, TY, src, dst, s, launches);
    if (e != cudaSuccess) return e;
  }
  const int items = P.ntx * P.nty * tile_pass_chunks(P);
  if (items == 0) return cudaSuccess;
  ++*launches;
  const int blocks = std::min(items, slots);
  if (part == 2) {
    k_apply_plane<K, TX, TY, ISO, T><<<blocks, S::NT, S::template smem<T>(), s>>>(P, src, dst);
    return cudaGetLastError();
  }
  // programmatic dependent launch on the init kernel: the blocks start while it runs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(S::NT);
  cfg.dynamicSmemBytes = S::template smem<T>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool off = std::getenv("MF_NO_PDL") != nullptr;  // plain stream order (comparisons)
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k_apply_plane<K, TX, TY, ISO, T>, P, src, dst);
}

bool cart_plane_supported(const Geo &g) {
  return g.dim == 3 && g.geom == MF_GEOM_CARTESIAN && g.coeff_kind == MF_COEFF_CONSTANT &&
         (g.k == 2 || g.k == 3 || g.k == 4);
}

// k = 4 tiles: 16 x 2 cells by default -- 3 instead of 7 strided x tile-edge planes in
// the init on 64^3 (its y-edge planes are contiguous rows); cfg 3 168.0 vs 173.9 us per
// apply.  MF_PLANE_TILE=8x4 selects the square-ish tile (comparisons).
static bool wide_tiles() {
  static const bool w = [] {
    const char *e = std::getenv("MF_PLANE_TILE");
    return !(e && std::strcmp(e, "8x4") == 0);
  }();
  return w;
}

template <class T>
static cudaError_t launch_cart_plane_any(const Geo &g, const Tables &t, const T *src, T *dst, cudaStream_t s,
                                        int64_t *launches, int part, int zr_lo = 0, int zr_hi = 0) {
  const bool iso = g.fcart[0] == g.fcart[1] && g.fcart[0] == g.fcart[2];
#define MF_PLANE_LAUNCH(KK, TXX, TYY)                                                                   \
  return iso ? launch_plane_t<KK, TXX, TYY, true, T>(g, t, src, dst, s, launches, part, zr_lo, zr_hi)  \
             : launch_plane_t<KK, TXX, TYY, false, T>(g, t, src, dst, s, launches, part, zr_lo, zr_hi)
  switch (g.k) {
    case 2: MF_PLANE_LAUNCH(2, 8, 8);
    case 3: MF_PLANE_LAUNCH(3, 8, 4);
    case 4:
      if (wide_tiles()) MF_PLANE_LAUNCH(4, 16, 2);
      MF_PLANE_LAUNCH(4, 8, 4);
  }
#undef MF_PLANE_LAUNCH
  return cudaErrorNotSupported;
}

cudaError_t launch_apply_cart_plane(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                                    int64_t *launches, int part) {
  return launch_cart_plane_any<double>(g, t, src, dst, s, launches, part);
}

cudaError_t launch_apply_cart_plane_f32(const Geo &g, const Tables &t, const float *src, float *dst, cudaStream_t s,
                                        int64_t *launches) {
  return launch_cart_plane_any<float>(g, t, src, dst, s, launches, 0);
}

cudaError_t launch_apply_cart_plane_range(const Geo &g, const Tables &t, const double *src, double *dst,
                                          cudaStream_t s, int64_t *launches, int zr_lo, int zr_hi) {
  return launch_cart_plane_any<double>(g, t, src, dst, s, launches, 3, zr_lo, zr_hi);
}

}  // namespace mf
