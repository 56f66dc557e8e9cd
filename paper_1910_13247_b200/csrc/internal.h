// internal.h -- shared declarations of libmf_b200 (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <functional>
#include <map>
#include <mutex>
#include <string>

#include "../../include/mf.h"

namespace mf {

constexpr int kMaxN = 9;  // k <= 8

// 1D tables on [0,1] for degree k (n = k+1 nodes = Gauss points), passed to
// kernels BY VALUE so they live in the constant bank (DFMA c[0x0][...] operands).
//   S[q][i]   = l_i(xi_q)         GLL Lagrange basis at Gauss point q
//   D[q][i]   = l_i'(xi_q)        its derivative (metric / diagonal kernels)
//   Co[q][p]  = lG_p'(xi_q)       collocation derivative on the Gauss points
//   w[q]      Gauss weights
struct Tables {
  double S[kMaxN][kMaxN];
  double D[kMaxN][kMaxN];
  double Co[kMaxN][kMaxN];
  double w[kMaxN];
  double gll[kMaxN];
  double xi[kMaxN];
  // reference 1D mass M = S^T W S and stiffness K = D^T W D on [0,1] (Gauss(k+1) is
  // exact for both): the Kronecker form of the Cartesian constant-coefficient operator
  double Mr[kMaxN][kMaxN];
  double Kr[kMaxN][kMaxN];
  // their even-odd parts (both are centro-symmetric): rows i < (n+1)/2 of E act on
  // e_j = u_j + u_{n-1-j} (j < n/2; e_{n/2} = u_{n/2} for odd n), rows i < n/2 of O on
  // o_j = u_j - u_{n-1-j}; v_i = ve_i + vo_i, v_{n-1-i} = ve_i - vo_i, v_{n/2} = ve_{n/2}
  double Me[5][5], Mo[5][5], Ke[5][5], Ko[5][5];
};

// Host-side construction (tables.cpp): an implementation of the 1D rules
// written independently of oracle/ (long double Newton iterations).
void build_tables(int k, Tables *t);

// Geometry / coefficient description shared by the kernels.
struct Geo {
  int dim, k;
  int64_t nc[3];        // local cells per direction (z local for slabs)
  int64_t N[3];         // local nodes per direction
  int64_t cz0;          // global z offset of the local slab (in cells)
  int64_t ncz_global;
  double lo[3], hi[3], h[3];
  double eps;
  int geom;             // MF_GEOM_*
  int coeff_kind;       // MF_COEFF_*
  double coeff;         // constant value
  uint32_t dirichlet;   // face bits, with z faces masked for inner slab boundaries
  int skip_top_identity;  // lower rank of a shared top plane: upper rank writes the identity rows there
  double fcart[3];      // c * prod(h) / h_e^2 (Cartesian, constant coefficient)
};

enum Variant {
  kVariantAuto = 0,
  kVariantGeneral = 1,  // 12-sweep collocation kernel, any dim/k/geometry
  kVariantCartTile = 2, // (removed in r02: the slab-form tile kernel, slower than the plane kernel)
  kVariantCartPlane = 3, // Cartesian constant-coefficient 3D, 2D-first / z-last form
  kVariantDG = 4,        // mf_create_dg (reported by mf_get_info)
  kVariantHex = 5,       // mf_create_hex (reported by mf_get_info)
  kVariantCartHalo = 6,  // Cartesian constant-coefficient 3D k = 4: owner-writes, no init / atomics
};

// Kernel launchers (return cudaError_t of the launch).
// part: 0 = the whole apply; for the halo overlap on z-slabs (§8(e)) 1 = zero dst +
// the cell layers next to the shared z-planes (first and last), 2 = the interior layers
// (part 1 then part 2 = part 0).  The 2D and tile paths take part 0 only.
cudaError_t launch_apply_general(const Geo &g, const Tables &t, const double *src, double *dst,
                                 const double *metric, cudaStream_t s, int64_t *launches, int part = 0);
cudaError_t launch_apply_cart_plane(const Geo &g, const Tables &t, const double *src, double *dst,
                                    cudaStream_t s, int64_t *launches, int part = 0);
// FP32 versions for the mixed-precision multigrid (§8(f) f2): the same kernels
// instantiated for float (dst zeroed by the caller for the general kernel)
cudaError_t launch_apply_cart_plane_f32(const Geo &g, const Tables &t, const float *src, float *dst,
                                        cudaStream_t s, int64_t *launches);
// the cell layers [zr_lo, zr_hi) only, with their share of dst initialisation (the
// pipelined host apply: ranges launched in increasing z complete the apply)
cudaError_t launch_apply_cart_plane_range(const Geo &g, const Tables &t, const double *src, double *dst,
                                          cudaStream_t s, int64_t *launches, int zr_lo, int zr_hi);
cudaError_t launch_apply_general_cells(const Geo &g, const Tables &t, const double *src, double *dst,
                                       const double *metric, cudaStream_t s, int64_t *launches, int64_t cb,
                                       int64_t ce);
cudaError_t launch_apply_general_f32(const Geo &g, const Tables &t, const float *src, float *dst,
                                     const float *metric, cudaStream_t s, int64_t *launches);
bool cart_plane_supported(const Geo &g);
// kernels_halo.cu: part 0 = every layer, 1 = the two boundary layers, 2 = the interior
// layers, 3 = the cell layers [zr_lo, zr_hi) (no dst initialisation needed in any part)
cudaError_t launch_apply_cart_halo(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                                   int64_t *launches, int part = 0, int zr_lo = 0, int zr_hi = 0);
bool cart_halo_supported(const Geo &g);
// kernels_tc.cu: Cartesian constant-coefficient 3D k = 5..7 on the FP64 tensor cores, the cell
// layers [cz_lo, cz_hi) (scatter-add: dst zeroed by the caller; MF_NO_TC=1 disables it)
cudaError_t launch_apply_tc(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                            int cz_lo, int cz_hi);
bool tc_supported(const Geo &g);
// DG-SIP operator and its diagonal (kernels_dg.cu, §8(f) f4)
// cells [cbeg, cend) only (cend < 0: every cell); DoFs cell-major, plain stores
cudaError_t launch_apply_dg(const Geo &g, const Tables &t, const double *src, double *dst, cudaStream_t s,
                            int64_t *launches, int64_t cbeg = 0, int64_t cend = -1);
cudaError_t launch_diagonal_dg(const Geo &g, const Tables &t, double *diag, cudaStream_t s, int64_t *launches);
cudaError_t launch_metric(const Geo &g, const Tables &t, double *metric, int *bad, cudaStream_t s,
                          int64_t *launches);
cudaError_t launch_diagonal(const Geo &g, const Tables &t, double *diag, const double *metric,
                            cudaStream_t s, int64_t *launches);
cudaError_t launch_zero(double *x, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_set_constrained(const Geo &g, double *x, double value, cudaStream_t s, int64_t *launches);

// vector kernels (kernels_vec.cu)
cudaError_t launch_splitmix(double *x, int64_t n, int64_t first_global, uint64_t seed, cudaStream_t s,
                            int64_t *launches);
// nd dot products in one pass (fixed block count, last block reduces in block order) into
// out[0..nd); partials: 3 kDotBlocks doubles, ticket: a zeroed device counter
cudaError_t launch_dots(int ndots, const double *const *a, const double *const *b, int64_t n,
                        double *partials, unsigned *ticket, double *out, cudaStream_t s, int64_t *launches);
// fused CG / Chebyshev steps with the step lengths on the device and the next dot in the same pass
cudaError_t launch_cg_xr_rr(const double *rz, const double *pv, double *x, double *r, const double *p,
                            const double *v, int64_t n, int64_t n_owned, double *partials, unsigned *ticket,
                            double *rr, cudaStream_t s, int64_t *launches);
cudaError_t launch_cg_p_dev(const double *rz_new, const double *rz_old, const double *z, double *p, int64_t n,
                            cudaStream_t s, int64_t *launches);
// three-term Chebyshev step over x_{k-1} (xp; first: x_{k-1} = 0), optional fused r.x_{k+1}
cudaError_t launch_cheb3(const double *r, const double *ax, const double *dinv, double c1, double c2,
                         const double *x, double *xp, bool first, int64_t n, int64_t n_owned, double *partials,
                         unsigned *ticket, double *rz, cudaStream_t s, int64_t *launches);
cudaError_t launch_cheb_init1(const double *r, const double *dinv, double c0, double *x, int64_t n, cudaStream_t s,
                              int64_t *launches);
// y = a*x + b*y   (and variants used by CG / Chebyshev)
cudaError_t launch_axpby(double a, const double *x, double b, double *y, int64_t n, cudaStream_t s,
                         int64_t *launches);
// out = a * b elementwise (Jacobi), y = 1 / x
cudaError_t launch_mul(const double *a, const double *b, double *out, int64_t n, cudaStream_t s,
                       int64_t *launches);
cudaError_t launch_recip(const double *x, double *y, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_plane_add(double *dst, const double *recv, int64_t n, cudaStream_t s, int64_t *launches);

// FP32 vector kernels (mixed-precision multigrid)
cudaError_t launch_zero_f(float *x, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_d2f(const double *x, float *y, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_f2d(const float *x, double *y, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_cheb_init_f(const float *r, const float *dinv, float c0, float *x, float *d, int64_t n,
                               cudaStream_t s, int64_t *launches);
cudaError_t launch_cheb_step_f(const float *r, const float *ax, const float *dinv, float c1, float c2, float *x,
                               float *d, int64_t n, cudaStream_t s, int64_t *launches);

// unstructured hex operator (mf_create_hex; kernels_general.cu), device pointers
constexpr int32_t kHexDirichlet = INT32_MIN;  // cell_dofs entry of a Dirichlet DoF
struct HexDev {
  int64_t ncells, ndofs, ndir;
  const int32_t *cell_dofs;  // [ncells][(k+1)^3]: >= 0 DoF, kHexDirichlet, else -1 - line
  const int32_t *line_ptr, *line_dof;  // constraint lines (Dirichlet entries removed)
  const double *line_w;
  const uint8_t *cell_lines;  // 1 if the cell has a constraint-line entry
  const double *metric;       // [6][ncells][(k+1)^3]
  const int32_t *dir;         // Dirichlet DoFs
};
cudaError_t launch_hex_metric(int k, const Tables &t, const double *V, const int32_t *CV, int64_t ncells,
                              int coeff_kind, double coeff, double *metric, int *bad, cudaStream_t s,
                              int64_t *launches);
// dst must be zero; adds the cell contributions and writes the identity rows
cudaError_t launch_apply_hex(int k, const Tables &t, const HexDev &h, const double *src, double *dst,
                             cudaStream_t s, int64_t *launches);
// diag must be zero
cudaError_t launch_diagonal_hex(int k, const Tables &t, const HexDev &h, double *diag, cudaStream_t s,
                                int64_t *launches);
cudaError_t launch_hex_set(const HexDev &h, double *x, double value, cudaStream_t s, int64_t *launches);
// DoF numbering of a conforming hex mesh (hex_dofs.cpp)
mf_status hex_number_dofs(int k, int64_t n_cells, const int32_t *cell_vertices, int32_t *cell_dofs,
                          int64_t *n_dofs, uint8_t *is_boundary, int64_t capacity, std::string *err);

constexpr int kDotBlocks = 592;  // 4 x 148 SMs

// Kernel attributes are per device: set them once per (kernel instance, device) -- ADVICE r01
// (function-local statics had set them on the first device only)
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}
// keyed by (kernel address, device): a function-local static in a template over the kernel's
// TYPE would be shared by every kernel of the same signature (k_apply_dg2<5> and <6>), and the
// second one would launch without its attribute; a later larger request sets it again
inline void smem_attr_once(const void *kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> set;
  const int d = current_device();
  std::lock_guard<std::mutex> lock(mu);
  size_t &have = set[{kernel, d}];
  if (have < bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    have = bytes;
  }
}
template <class K>
inline void smem_attr_once(K kernel, size_t bytes) {
  smem_attr_once(reinterpret_cast<const void *>(kernel), bytes);
}

}  // namespace mf

// api.cu internals shared with mg.cu (C++ linkage, not part of the C ABI)
// precond(r, z, rz_dev): z = P r and rz_dev = r.z (device scalar, summed over ranks)
mf_status cg_core(mf_op *op, const double *b, double *x, double rel_tol, int max_iter,
                  const std::function<mf_status(const double *, double *, double *)> &precond, mf_cg_result *res,
                  double *history, int32_t history_cap);
mf_status dot_dev(mf_op *op, const double *a, const double *b, double *out_dev);
mf_status mf_set_error(mf_status s, const std::string &msg);  // sets mf_last_error, returns s
// FP32 operator and Chebyshev polynomial of an op (3D, one rank)
mf_status apply_f32(mf_op *op, const float *src, float *dst);
mf_status cheb_f32(mf_op *op, const float *r, float *x, double lam, int degree, double range);
