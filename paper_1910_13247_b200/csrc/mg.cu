// mg.cu -- geometric multigrid on the globally refined brick (
// PAPER.md P:845-877, §6.1), built on the level
// operators of api.cu (one mf_op per level, all on one stream):
//   * transfer: prolongation = interpolation of the coarse Q_k function at the fine
//     GLL support points.  On the brick it is the tensor product Pz (x) Py (x) Px of
//     1D interpolations, applied as three sweeps (x, then y, then z), each output
//     node reading the k+1 coarse nodes of the coarse cell that contains it;
//     restriction = the exact transpose (z^T, y^T, x^T sweeps, gather form);
//     constrained DoFs are zeroed on both levels (the identity-row convention R3);
//   * smoother: the level's Chebyshev(degree) polynomial (mf_chebyshev) on
//     [lam_l / range, lam_l]; pre: x = Cheb(b); post: x += Cheb(b - A x);
//   * coarse solver: the dense inverse of the level-0 operator, formed once on the
//     GPU (columns A e_j by mf_apply, then Gauss-Jordan), applied as a GEMV;
//   * V-cycle: pre-smooth, residual, restrict, recurse, prolongate + correct,
//     post-smooth -- no host synchronisation inside a cycle.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"

using namespace mf;

namespace {

constexpr int kMaxK = 8;
constexpr int64_t kMaxCoarse = 2048;

// W[m][j] = l_j(t_m): coarse basis j at fine node m = 0..2k of one coarse cell
template <class T>
struct InterpT {
  T W[2 * kMaxK + 1][kMaxK + 1];
  int k;
};

struct Dims {
  int64_t n[3];
};

// out (dims in, axis refined: n_out = 2 n_in - 1) = 1D interpolation along `axis`
template <class T>
__global__ void k_interp_axis(const __grid_constant__ InterpT<T> I, int axis, Dims din, const T *__restrict__ in,
                              T *__restrict__ out) {
  const int k = I.k;
  Dims dout = din;
  dout.n[axis] = 2 * din.n[axis] - 1;
  const int64_t total = dout.n[0] * dout.n[1] * dout.n[2];
  const int64_t ncc = (din.n[axis] - 1) / k;  // coarse cells along the axis
  const int64_t sin = axis == 0 ? 1 : (axis == 1 ? din.n[0] : din.n[0] * din.n[1]);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3];
    c[0] = o % dout.n[0];
    const int64_t r = o / dout.n[0];
    c[1] = r % dout.n[1];
    c[2] = r / dout.n[1];
    const int64_t f = c[axis];
    int64_t cc = f / (2 * k);
    int m = (int)(f - 2 * k * cc);
    if (cc == ncc) {
      cc = ncc - 1;
      m = 2 * k;
    }
    c[axis] = k * cc;
    const T *ip = in + (c[2] * din.n[1] + c[1]) * din.n[0] + c[0];
    T s = 0;
    for (int j = 0; j <= k; ++j) s = fma(I.W[m][j], ip[j * sin], s);
    out[o] = s;
  }
}

// out (dims of the coarse output: the input has n_in = 2 n_out - 1 along `axis`) = the
// transpose of k_interp_axis: coarse node c = k cc + j gathers the fine nodes of the
// coarse cells containing it; a fine node on a coarse vertex belongs to the cell on its
// right (the last one to the last cell), exactly as in k_interp_axis
template <class T>
__global__ void k_restrict_axis(const __grid_constant__ InterpT<T> I, int axis, Dims dout, const T *__restrict__ in,
                                T *__restrict__ out) {
  const int k = I.k;
  Dims din = dout;
  din.n[axis] = 2 * dout.n[axis] - 1;
  const int64_t total = dout.n[0] * dout.n[1] * dout.n[2];
  const int64_t ncc = (dout.n[axis] - 1) / k;
  const int64_t sin = axis == 0 ? 1 : (axis == 1 ? din.n[0] : din.n[0] * din.n[1]);
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[3];
    c[0] = o % dout.n[0];
    const int64_t r = o / dout.n[0];
    c[1] = r % dout.n[1];
    c[2] = r / dout.n[1];
    const int64_t cn = c[axis], cc = cn / k;
    const int j = (int)(cn - k * cc);
    c[axis] = 0;
    const T *ip = in + (c[2] * din.n[1] + c[1]) * din.n[0] + c[0];
    T s = 0;
    if (j != 0) {
      for (int m = 0; m <= 2 * k; ++m) s = fma(I.W[m][j], ip[(2 * k * cc + m) * sin], s);
    } else {
      if (cc < ncc)
        for (int m = 0; m < 2 * k; ++m) s = fma(I.W[m][0], ip[(2 * k * cc + m) * sin], s);
      if (cc > 0)
        for (int m = 0; m < 2 * k; ++m) s = fma(I.W[m][k], ip[(2 * k * (cc - 1) + m) * sin], s);
      if (cc == ncc) s = fma(I.W[2 * k][k], ip[(2 * k * ncc) * sin], s);
    }
    out[o] = s;
  }
}

template <class T>
__global__ void k_zero_constrained(T *__restrict__ x, Dims d, uint32_t dir) {
  const int64_t total = d.n[0] * d.n[1] * d.n[2];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gx = o % d.n[0], r = o / d.n[0], gy = r % d.n[1], gz = r / d.n[1];
    const bool cons = ((dir & 1u) && gx == 0) || ((dir & 2u) && gx == d.n[0] - 1) || ((dir & 4u) && gy == 0) ||
                      ((dir & 8u) && gy == d.n[1] - 1) || ((dir & 16u) && gz == 0) ||
                      ((dir & 32u) && gz == d.n[2] - 1);
    if (cons) x[o] = T(0);
  }
}

// y = a x + b y (element-wise combination used by the V-cycle)
template <class T>
__global__ void k_axpby2(T a, const T *__restrict__ x, T b, const T *__restrict__ y, T *__restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

__global__ void k_d2f_mg(const double *__restrict__ x, float *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}

__global__ void k_unit(double *x, int64_t n, int64_t j) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = i == j ? 1.0 : 0.0;
}

// one Gauss-Jordan step on the augmented row-major [A | I] (n x 2n), pivot p; SPD A,
// no pivoting needed
__global__ void k_gj_step(const double *__restrict__ M, double *__restrict__ Mo, int64_t n, int64_t p) {
  const int64_t w = 2 * n, total = n * w;
  const double piv = M[p * w + p];
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o / w, jj = o - i * w;
    const double rp = M[p * w + jj] / piv;
    Mo[o] = i == p ? rp : M[o] - M[i * w + p] * rp;
  }
}

// y = A x, A row-major n x n with leading dimension lda; one warp per row
template <class T>
__global__ void k_gemv(const T *__restrict__ A, int64_t lda, const T *__restrict__ x, T *__restrict__ y, int64_t n) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  T s = 0;
  for (int64_t j = lane; j < n; j += 32) s = fma(A[row * lda + j], x[j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

// l_j(t) on the GLL nodes by the product formula
double lagrange(const double *x, int k, int j, double t) {
  double v = 1.0;
  for (int m = 0; m <= k; ++m)
    if (m != j) v *= (t - x[m]) / (x[j] - x[m]);
  return v;
}

}  // namespace

// the V-cycle's vectors in one precision
template <class T>
struct MGBufs {
  // per level: b, x (levels < L-1, all levels for FP32), r, t, z (levels >= 1)
  std::vector<T *> b, x, r, t, z;
  T *tmp1 = nullptr, *tmp2 = nullptr;  // transfer intermediates (<= finest size)
  T *ainv = nullptr;                   // dense inverse of level 0, n0 x n0 row-major
  InterpT<T> I;
  void free_all() {
    for (auto *v : {&b, &x, &r, &t, &z})
      for (T *p : *v) cudaFree(p);
    cudaFree(tmp1);
    cudaFree(tmp2);
    cudaFree(ainv);
  }
};

struct mf_mg {
  int L = 0, k = 0;
  uint32_t dirichlet = 0;
  int precision = 0;  // 0 FP64 V-cycle, 1 FP32 V-cycle
  std::vector<mf_op *> ops;
  std::vector<Dims> dims;
  std::vector<int64_t> n;
  std::vector<double> lam;
  MGBufs<double> d;
  MGBufs<float> f;
  int degree = 6;
  double range = 20.0;
  cudaStream_t stream = 0;
  int64_t launches = 0;
};

template <class T>
static MGBufs<T> &bufs(mf_mg *mg);
template <>
MGBufs<double> &bufs<double>(mf_mg *mg) {
  return mg->d;
}
template <>
MGBufs<float> &bufs<float>(mf_mg *mg) {
  return mg->f;
}
// the level operator and smoother in precision T
static mf_status level_apply(mf_op *op, const double *x, double *y, int64_t n) { return mf_apply(op, x, n, y, n); }
static mf_status level_apply(mf_op *op, const float *x, float *y, int64_t) { return apply_f32(op, x, y); }
static mf_status level_cheb(mf_mg *mg, int l, const double *r, double *x) {
  return mf_chebyshev(mg->ops[l], r, x, mg->n[l], mg->lam[l], mg->degree, mg->range);
}
static mf_status level_cheb(mf_mg *mg, int l, const float *r, float *x) {
  return cheb_f32(mg->ops[l], r, x, mg->lam[l], mg->degree, mg->range);
}

#define MG_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return mf_set_error(e_ == cudaErrorMemoryAllocation ? MF_ERR_OUT_OF_MEMORY : MF_ERR_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)
#define MG_TRY(call)              \
  do {                            \
    mf_status s_ = (call);        \
    if (s_ != MF_OK) return s_;   \
  } while (0)

template <class T>
static mf_status zero_constrained(mf_mg *mg, int l, T *v) {
  if (!mg->dirichlet) return MF_OK;
  ++mg->launches;
  k_zero_constrained<T><<<grid_for(mg->n[l]), 256, 0, mg->stream>>>(v, mg->dims[l], mg->dirichlet);
  MG_CUDA(cudaGetLastError());
  return MF_OK;
}

// fine(l) = P coarse(l-1), then the fine constrained DoFs zeroed
template <class T>
static mf_status prolongate(mf_mg *mg, int l, const T *coarse, T *fine) {
  MGBufs<T> &B = bufs<T>(mg);
  Dims d = mg->dims[l - 1];
  const T *in = coarse;
  T *bufs[3] = {B.tmp1, B.tmp2, fine};
  for (int axis = 0; axis < 3; ++axis) {
    Dims dn = d;
    dn.n[axis] = 2 * d.n[axis] - 1;
    ++mg->launches;
    k_interp_axis<T><<<grid_for(dn.n[0] * dn.n[1] * dn.n[2]), 256, 0, mg->stream>>>(B.I, axis, d, in, bufs[axis]);
    MG_CUDA(cudaGetLastError());
    in = bufs[axis];
    d = dn;
  }
  return zero_constrained(mg, l, fine);
}

// coarse(l-1) = P^T fine(l) (fine constrained entries must already be 0), then the
// coarse constrained DoFs zeroed
template <class T>
static mf_status restrict_(mf_mg *mg, int l, const T *fine, T *coarse) {
  MGBufs<T> &B = bufs<T>(mg);
  Dims d = mg->dims[l];
  const T *in = fine;
  T *bufs[3] = {B.tmp1, B.tmp2, coarse};
  for (int s = 0; s < 3; ++s) {
    const int axis = 2 - s;
    Dims dn = d;
    dn.n[axis] = (d.n[axis] + 1) / 2;
    ++mg->launches;
    k_restrict_axis<T><<<grid_for(dn.n[0] * dn.n[1] * dn.n[2]), 256, 0, mg->stream>>>(B.I, axis, dn, in, bufs[s]);
    MG_CUDA(cudaGetLastError());
    in = bufs[s];
    d = dn;
  }
  return zero_constrained(mg, l - 1, coarse);
}

template <class T>
static mf_status axpby2(mf_mg *mg, T a, const T *x, T b, const T *y, T *out, int64_t n) {
  ++mg->launches;
  k_axpby2<T><<<grid_for(n), 256, 0, mg->stream>>>(a, x, b, y, out, n);
  MG_CUDA(cudaGetLastError());
  return MF_OK;
}

// x_l = V_l(b_l), in precision T
template <class T>
static mf_status vcycle(mf_mg *mg, int l, const T *b, T *x) {
  MGBufs<T> &B = bufs<T>(mg);
  const int64_t n = mg->n[l];
  if (l == 0) {
    ++mg->launches;
    k_gemv<T><<<(unsigned)((n * 32 + 255) / 256), 256, 0, mg->stream>>>(B.ainv, n, b, x, n);
    MG_CUDA(cudaGetLastError());
    return MF_OK;
  }
  mf_op *op = mg->ops[l];
  T *r = B.r[l], *t = B.t[l], *z = B.z[l];
  MG_TRY(level_cheb(mg, l, b, x));  // pre-smoothing from 0
  MG_TRY(level_apply(op, x, t, n));
  MG_TRY(axpby2<T>(mg, T(1), b, T(-1), t, r, n));  // r = b - A x
  MG_TRY(zero_constrained(mg, l, r));
  MG_TRY(restrict_(mg, l, (const T *)r, B.b[l - 1]));
  MG_TRY(vcycle(mg, l - 1, (const T *)B.b[l - 1], B.x[l - 1]));
  MG_TRY(prolongate(mg, l, (const T *)B.x[l - 1], t));
  MG_TRY(axpby2<T>(mg, T(1), x, T(1), t, x, n));  // x += P x_c
  MG_TRY(level_apply(op, x, t, n));
  MG_TRY(axpby2<T>(mg, T(1), b, T(-1), t, r, n));
  MG_TRY(level_cheb(mg, l, (const T *)r, z));  // post-smoothing
  return axpby2<T>(mg, T(1), x, T(1), z, x, n);
}

// z = V(r) on the finest level in the hierarchy's precision (FP64 in / out)
static mf_status vcycle_top(mf_mg *mg, const double *r, double *z) {
  const int top = mg->L - 1;
  if (mg->precision == 0) return vcycle<double>(mg, top, r, z);
  const int64_t n = mg->n[top];
  MG_CUDA(launch_d2f(r, mg->f.b[top], n, mg->stream, &mg->launches));
  MG_TRY(vcycle<float>(mg, top, mg->f.b[top], mg->f.x[top]));
  MG_CUDA(launch_f2d(mg->f.x[top], z, n, mg->stream, &mg->launches));
  return MF_OK;
}

extern "C" void mf_mg_destroy(mf_mg *mg) {
  if (!mg) return;
  mg->d.free_all();
  mg->f.free_all();
  for (mf_op *op : mg->ops) mf_destroy(op);
  delete mg;
}

extern "C" mf_status mf_mg_create(const mf_mesh *finest, int32_t degree, const mf_coeff *coeff,
                                  const mf_mg_params *prm, mf_mg **out) {
  if (!finest || !coeff || !prm || !out) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (finest->dim != 3) return mf_set_error(MF_ERR_ARGUMENT, "multigrid: dim must be 3");
  if (degree < 1 || degree > kMaxK) return mf_set_error(MF_ERR_ARGUMENT, "multigrid: degree out of range");
  if ((finest->dirichlet_faces & 63u) == 0)
    return mf_set_error(MF_ERR_SINGULAR, "multigrid: pure Neumann operator is singular (no coarse inverse)");
  if (prm->smooth_degree < 1 || !(prm->smooth_range > 1.0) || !(prm->smooth_safety > 0.0) || prm->eig_cg_steps < 1 ||
      prm->n_levels < 0 || prm->precision < 0 || prm->precision > 1)
    return mf_set_error(MF_ERR_ARGUMENT, "multigrid: bad smoother parameters");
  int64_t nc[3] = {finest->n_cells[0], finest->n_cells[1], finest->n_cells[2]};
  int L = prm->n_levels;
  if (L == 0) {  // halve while even and the coarser level is still above max_coarse_dofs
    L = 1;
    int64_t c[3] = {nc[0], nc[1], nc[2]};
    while (c[0] % 2 == 0 && c[1] % 2 == 0 && c[2] % 2 == 0 &&
           (degree * c[0] + 1) * (degree * c[1] + 1) * (degree * c[2] + 1) > prm->max_coarse_dofs) {
      for (int e = 0; e < 3; ++e) c[e] /= 2;
      ++L;
    }
  }
  const int64_t f = int64_t(1) << (L - 1);
  for (int e = 0; e < 3; ++e)
    if (nc[e] % f) return mf_set_error(MF_ERR_ARGUMENT, "multigrid: n_cells not divisible by 2^(levels-1)");
  const int64_t n0 = (degree * nc[0] / f + 1) * (degree * nc[1] / f + 1) * (degree * nc[2] / f + 1);
  if (n0 > kMaxCoarse) return mf_set_error(MF_ERR_ARGUMENT, "multigrid: coarse level above 2048 DoFs");

  mf_mg *mg = new mf_mg();
  auto cleanup = [&](mf_status s) {
    mf_mg_destroy(mg);
    return s;
  };
  mg->L = L;
  mg->k = degree;
  mg->dirichlet = finest->dirichlet_faces;
  mg->degree = prm->smooth_degree;
  mg->range = prm->smooth_range;
  for (int l = 0; l < L; ++l) {
    const int64_t fl = int64_t(1) << (L - 1 - l);
    mf_mesh m = *finest;
    for (int e = 0; e < 3; ++e) m.n_cells[e] = nc[e] / fl;
    mf_op *op = nullptr;
    const mf_status st = mf_create(&m, degree, coeff, nullptr, &op);
    if (st != MF_OK) return cleanup(st);
    mg->ops.push_back(op);
    Dims d;
    for (int e = 0; e < 3; ++e) d.n[e] = degree * m.n_cells[e] + 1;
    mg->dims.push_back(d);
    mg->n.push_back(d.n[0] * d.n[1] * d.n[2]);
  }
  // 1D interpolation weights from the library's own GLL nodes
  Tables tab;
  build_tables(degree, &tab);
  std::memset(&mg->d.I, 0, sizeof(mg->d.I));
  std::memset(&mg->f.I, 0, sizeof(mg->f.I));
  mg->d.I.k = mg->f.I.k = degree;
  for (int m = 0; m <= 2 * degree; ++m) {
    const int child = m < degree ? 0 : (m < 2 * degree ? 1 : 2);
    const double tm = child == 2 ? 1.0 : 0.5 * (child + tab.gll[m - child * degree]);
    for (int j = 0; j <= degree; ++j) {
      mg->d.I.W[m][j] = lagrange(tab.gll, degree, j, tm);
      mg->f.I.W[m][j] = (float)mg->d.I.W[m][j];
    }
  }
  // vectors
  const size_t bytes_f = mg->n[L - 1] * sizeof(double);
  // FP64 buffers (always: the public transfer calls and the FP64 V-cycle), FP32 ones for
  // the mixed-precision V-cycle
  auto alloc = [&](auto &B, size_t es, bool all_bx) -> bool {
    B.b.assign(L, nullptr);
    B.x.assign(L, nullptr);
    B.r.assign(L, nullptr);
    B.t.assign(L, nullptr);
    B.z.assign(L, nullptr);
    for (int l = 0; l < L; ++l) {
      const size_t bytes = mg->n[l] * es;
      if ((l < L - 1 || all_bx) && (cudaMalloc((void **)&B.b[l], bytes) != cudaSuccess ||
                                    cudaMalloc((void **)&B.x[l], bytes) != cudaSuccess))
        return false;
      if (l >= 1 && (cudaMalloc((void **)&B.r[l], bytes) != cudaSuccess ||
                     cudaMalloc((void **)&B.t[l], bytes) != cudaSuccess ||
                     cudaMalloc((void **)&B.z[l], bytes) != cudaSuccess))
        return false;
    }
    return cudaMalloc((void **)&B.tmp1, mg->n[L - 1] * es) == cudaSuccess &&
           cudaMalloc((void **)&B.tmp2, mg->n[L - 1] * es) == cudaSuccess;
  };
  (void)bytes_f;
  mg->precision = prm->precision;
  if (!alloc(mg->d, sizeof(double), false) || (mg->precision == 1 && !alloc(mg->f, sizeof(float), true)))
    return cleanup(mf_set_error(MF_ERR_OUT_OF_MEMORY, "multigrid vectors"));
  // smoother intervals
  mg->lam.assign(L, 0.0);
  for (int l = 1; l < L; ++l) {
    double lam = 0.0;
    const mf_status st = mf_estimate_lambda_max(mg->ops[l], prm->eig_cg_steps, &lam);
    if (st != MF_OK) return cleanup(st);
    mg->lam[l] = prm->smooth_safety * lam;
  }
  // coarse solver: A_0 e_j column by column (symmetric, so row-major = column-major),
  // then Gauss-Jordan on [A_0 | I]
  const int64_t m0 = mg->n[0];
  double *aug = nullptr, *aug2 = nullptr, *e = nullptr, *col = nullptr;
  const size_t abytes = (size_t)m0 * 2 * m0 * sizeof(double);
  if (cudaMalloc(&aug, abytes) != cudaSuccess || cudaMalloc(&aug2, abytes) != cudaSuccess ||
      cudaMalloc(&e, m0 * sizeof(double)) != cudaSuccess || cudaMalloc(&col, m0 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&mg->d.ainv, (size_t)m0 * m0 * sizeof(double)) != cudaSuccess ||
      (mg->precision == 1 && cudaMalloc(&mg->f.ainv, (size_t)m0 * m0 * sizeof(float)) != cudaSuccess)) {
    cudaFree(aug);
    cudaFree(aug2);
    cudaFree(e);
    cudaFree(col);
    return cleanup(mf_set_error(MF_ERR_OUT_OF_MEMORY, "coarse solver"));
  }
  mf_status st = MF_OK;
  cudaError_t ce = cudaSuccess;
  // row j of [A | I] = (A e_j)^T, e_j^T  (A symmetric)
  for (int64_t j = 0; j < m0 && st == MF_OK && ce == cudaSuccess; ++j) {
    k_unit<<<grid_for(m0), 256, 0, mg->stream>>>(e, m0, j);
    st = mf_apply(mg->ops[0], e, m0, col, m0);
    if (st == MF_OK) ce = cudaMemcpyAsync(aug + j * 2 * m0, col, m0 * sizeof(double), cudaMemcpyDeviceToDevice, mg->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(aug + j * 2 * m0 + m0, e, m0 * sizeof(double), cudaMemcpyDeviceToDevice,
                                                mg->stream);
  }
  for (int64_t p = 0; p < m0 && st == MF_OK && ce == cudaSuccess; ++p) {
    k_gj_step<<<grid_for(2 * m0 * m0), 256, 0, mg->stream>>>(aug, aug2, m0, p);
    std::swap(aug, aug2);
    ce = cudaGetLastError();
  }
  if (st == MF_OK && ce == cudaSuccess)
    ce = cudaMemcpy2DAsync(mg->d.ainv, m0 * sizeof(double), aug + m0, 2 * m0 * sizeof(double), m0 * sizeof(double), m0,
                           cudaMemcpyDeviceToDevice, mg->stream);
  if (ce == cudaSuccess && mg->precision == 1) {
    k_d2f_mg<<<grid_for(m0 * m0), 256, 0, mg->stream>>>(mg->d.ainv, mg->f.ainv, m0 * m0);
    ce = cudaGetLastError();
  }
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(mg->stream);
  cudaFree(aug);
  cudaFree(aug2);
  cudaFree(e);
  cudaFree(col);
  if (st != MF_OK) return cleanup(st);
  if (ce != cudaSuccess) return cleanup(mf_set_error(MF_ERR_CUDA, std::string("coarse solver: ") + cudaGetErrorString(ce)));
  *out = mg;
  return MF_OK;
}

extern "C" mf_status mf_mg_levels(const mf_mg *mg, int32_t *n_levels) {
  if (!mg || !n_levels) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  *n_levels = mg->L;
  return MF_OK;
}

extern "C" mf_status mf_mg_level_size(const mf_mg *mg, int32_t level, int64_t *n_local) {
  if (!mg || !n_local || level < 0 || level >= mg->L) return mf_set_error(MF_ERR_ARGUMENT, "bad level");
  *n_local = mg->n[level];
  return MF_OK;
}

extern "C" mf_status mf_mg_level_op(mf_mg *mg, int32_t level, mf_op **op) {
  if (!mg || !op || level < 0 || level >= mg->L) return mf_set_error(MF_ERR_ARGUMENT, "bad level");
  *op = mg->ops[level];
  return MF_OK;
}

extern "C" mf_status mf_mg_level_lambda(const mf_mg *mg, int32_t level, double *lambda) {
  if (!mg || !lambda || level < 0 || level >= mg->L) return mf_set_error(MF_ERR_ARGUMENT, "bad level");
  *lambda = mg->lam[level];
  return MF_OK;
}

extern "C" mf_status mf_mg_prolongate(mf_mg *mg, int32_t level, const double *coarse, double *fine) {
  if (!mg || !coarse || !fine || level < 1 || level >= mg->L) return mf_set_error(MF_ERR_ARGUMENT, "bad level");
  // the masked prolongation D_f P D_c: zero the coarse constrained entries first (the
  // V-cycle's coarse corrections are zero there already)
  double *xc = mg->d.x[level - 1];
  MG_CUDA(cudaMemcpyAsync(xc, coarse, mg->n[level - 1] * sizeof(double), cudaMemcpyDeviceToDevice, mg->stream));
  MG_TRY(zero_constrained(mg, level - 1, xc));
  return prolongate(mg, level, xc, fine);
}

extern "C" mf_status mf_mg_restrict(mf_mg *mg, int32_t level, const double *fine, double *coarse) {
  if (!mg || !coarse || !fine || level < 1 || level >= mg->L) return mf_set_error(MF_ERR_ARGUMENT, "bad level");
  // the transpose of the masked prolongation: zero the fine constrained entries first
  MG_CUDA(cudaMemcpyAsync(mg->d.r[level], fine, mg->n[level] * sizeof(double), cudaMemcpyDeviceToDevice,
                          mg->stream));
  MG_TRY(zero_constrained(mg, level, mg->d.r[level]));
  return restrict_(mg, level, (const double *)mg->d.r[level], coarse);
}

extern "C" mf_status mf_mg_vcycle(mf_mg *mg, const double *b, double *x, int64_t n) {
  if (!mg || !b || !x) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  if (n != mg->n[mg->L - 1]) return mf_set_error(MF_ERR_LENGTH, "vector length != finest n_local");
  if (b == x) return mf_set_error(MF_ERR_ARGUMENT, "b and x must be distinct");
  return vcycle_top(mg, b, x);
}

extern "C" mf_status mf_mg_cg_solve(mf_mg *mg, const double *b, double *x, int64_t n, double rel_tol,
                                    int32_t max_iter, mf_cg_result *result, double *history, int32_t history_cap) {
  if (!mg || !b || !x || !result) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  if (n != mg->n[mg->L - 1]) return mf_set_error(MF_ERR_LENGTH, "vector length != finest n_local");
  if (!(rel_tol > 0.0) || max_iter < 1) return mf_set_error(MF_ERR_ARGUMENT, "bad CG parameters");
  result->lambda_max = mg->lam[mg->L - 1];
  auto precond = [&](const double *r, double *z, double *rz_dev) -> mf_status {
    const mf_status st = vcycle_top(mg, r, z);
    return st != MF_OK ? st : dot_dev(mg->ops[mg->L - 1], r, z, rz_dev);
  };
  return cg_core(mg->ops[mg->L - 1], b, x, rel_tol, max_iter, precond, result, history, history_cap);
}

extern "C" mf_status mf_mg_set_stream(mf_mg *mg, void *cuda_stream) {
  if (!mg) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  mg->stream = (cudaStream_t)cuda_stream;
  for (mf_op *op : mg->ops) MG_TRY(mf_set_stream(op, cuda_stream));
  return MF_OK;
}

// ---------------------------------------------------------------------------
// Hanging nodes (restricted): the two-block mesh of a coarse lower
// brick and a once-refined upper brick meeting at z = z_mid (R20).  The fine
// interface nodes hang; continuity makes them the coarse face function interpolated at
// the fine nodes, u_f(plane 0) = (P_y (x) P_x) u_c(top plane), so the matrix-free apply
// is the gather/scatter of the constraint around the two block operators:
//   y_c = A_c x_c;   x_f = [P2D x_c(top) | x(fine part)];   y_f = A_f x_f;
//   y(fine part) = y_f(planes >= 1);   y_c(top) += P2D^T y_f(plane 0)
// (coarse Dirichlet lines of the top plane masked on both sides, the identity rows of
// either block kept).
struct mf_hng {
  mf_op *oc = nullptr, *of = nullptr;
  Dims dc{}, df{};  // node counts of the two grids
  int64_t nC = 0, nF = 0, n = 0, pc_n = 0, pf_n = 0;  // pc_n / pf_n: coarse / fine plane sizes
  InterpT<double> I;
  double *xf = nullptr, *yf = nullptr, *t1 = nullptr, *t2 = nullptr, *pc = nullptr;
  cudaStream_t stream = 0;
  int64_t launches = 0;
};

extern "C" void mf_hng_destroy(mf_hng *h) {
  if (!h) return;
  for (double *p : {h->xf, h->yf, h->t1, h->t2, h->pc}) cudaFree(p);
  mf_destroy(h->oc);
  mf_destroy(h->of);
  delete h;
}

extern "C" mf_status mf_hng_create(const double *lower, const double *upper, double z_mid,
                                   const int64_t *n_cells_coarse, int64_t nz_fine, int32_t degree,
                                   const mf_coeff *coeff, mf_hng **out) {
  if (!lower || !upper || !n_cells_coarse || !coeff || !out) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (!(lower[2] < z_mid && z_mid < upper[2]) || nz_fine < 1 || coeff->kind != MF_COEFF_CONSTANT)
    return mf_set_error(MF_ERR_ARGUMENT, "hanging nodes: lower z < z_mid < upper z, nz_fine >= 1, constant coefficient");
  mf_mesh mc{}, mfm{};
  mc.dim = mfm.dim = 3;
  for (int e = 0; e < 3; ++e) {
    mc.n_cells[e] = n_cells_coarse[e];
    mc.lower[e] = mfm.lower[e] = lower[e];
    mc.upper[e] = mfm.upper[e] = upper[e];
  }
  mc.upper[2] = z_mid;
  mfm.lower[2] = z_mid;
  mfm.n_cells[0] = 2 * n_cells_coarse[0];
  mfm.n_cells[1] = 2 * n_cells_coarse[1];
  mfm.n_cells[2] = nz_fine;
  mc.geometry = mfm.geometry = MF_GEOM_CARTESIAN;
  mc.dirichlet_faces = 0b011111u;   // x, y, bottom; the interface is natural
  mfm.dirichlet_faces = 0b101111u;  // x, y, top
  mf_hng *h = new mf_hng();
  auto cleanup = [&](mf_status s) {
    mf_hng_destroy(h);
    return s;
  };
  mf_status st = mf_create(&mc, degree, coeff, nullptr, &h->oc);
  if (st == MF_OK) st = mf_create(&mfm, degree, coeff, nullptr, &h->of);
  if (st != MF_OK) return cleanup(st);
  for (int e = 0; e < 3; ++e) {
    h->dc.n[e] = degree * mc.n_cells[e] + 1;
    h->df.n[e] = degree * mfm.n_cells[e] + 1;
  }
  h->pc_n = h->dc.n[0] * h->dc.n[1];
  h->pf_n = h->df.n[0] * h->df.n[1];
  h->nC = h->pc_n * h->dc.n[2];
  h->nF = h->pf_n * h->df.n[2];
  h->n = h->nC + h->nF - h->pf_n;
  Tables tab;
  build_tables(degree, &tab);
  std::memset(&h->I, 0, sizeof(h->I));
  h->I.k = degree;
  for (int m = 0; m <= 2 * degree; ++m) {
    const int child = m < degree ? 0 : (m < 2 * degree ? 1 : 2);
    const double tm = child == 2 ? 1.0 : 0.5 * (child + tab.gll[m - child * degree]);
    for (int j = 0; j <= degree; ++j) h->I.W[m][j] = lagrange(tab.gll, degree, j, tm);
  }
  if (cudaMalloc(&h->xf, h->nF * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->yf, h->nF * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->t1, h->pf_n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->t2, h->pf_n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->pc, h->pc_n * sizeof(double)) != cudaSuccess)
    return cleanup(mf_set_error(MF_ERR_OUT_OF_MEMORY, "hanging-node buffers"));
  *out = h;
  return MF_OK;
}

extern "C" mf_status mf_hng_sizes(const mf_hng *h, int64_t *n, int64_t *n_coarse) {
  if (!h) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  if (n) *n = h->n;
  if (n_coarse) *n_coarse = h->nC;
  return MF_OK;
}

extern "C" mf_status mf_hng_set_stream(mf_hng *h, void *cuda_stream) {
  if (!h) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  h->stream = (cudaStream_t)cuda_stream;
  MG_TRY(mf_set_stream(h->oc, cuda_stream));
  return mf_set_stream(h->of, cuda_stream);
}

extern "C" mf_status mf_hng_apply(mf_hng *h, const double *src, int64_t n_src, double *dst, int64_t n_dst) {
  if (!h || !src || !dst) return mf_set_error(MF_ERR_ARGUMENT, "null argument");
  if (n_src != h->n || n_dst != h->n) return mf_set_error(MF_ERR_LENGTH, "vector length != n");
  if (src == dst) return mf_set_error(MF_ERR_ARGUMENT, "src and dst must be distinct");
  cudaStream_t s = h->stream;
  const Dims dp{{h->dc.n[0], h->dc.n[1], 1}};  // the coarse interface plane
  const uint32_t lines = 0b1111u;              // its Dirichlet lines (x and y faces)
  // coarse block
  MG_TRY(mf_apply(h->oc, src, h->nC, dst, h->nC));
  // gather: fine grid input = [P2D (masked coarse top plane) | fine part]
  MG_CUDA(cudaMemcpyAsync(h->pc, src + h->nC - h->pc_n, h->pc_n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  k_zero_constrained<double><<<grid_for(h->pc_n), 256, 0, s>>>(h->pc, dp, lines);
  Dims d1 = dp;
  d1.n[0] = 2 * dp.n[0] - 1;
  k_interp_axis<double><<<grid_for(d1.n[0] * d1.n[1]), 256, 0, s>>>(h->I, 0, dp, h->pc, h->t1);
  k_interp_axis<double><<<grid_for(h->pf_n), 256, 0, s>>>(h->I, 1, d1, h->t1, h->xf);
  MG_CUDA(cudaMemcpyAsync(h->xf + h->pf_n, src + h->nC, (h->nF - h->pf_n) * sizeof(double),
                          cudaMemcpyDeviceToDevice, s));
  h->launches += 3;
  // fine block
  MG_TRY(mf_apply(h->of, h->xf, h->nF, h->yf, h->nF));
  // scatter: fine part, and P2D^T of the interface plane into the coarse top plane
  MG_CUDA(cudaMemcpyAsync(dst + h->nC, h->yf + h->pf_n, (h->nF - h->pf_n) * sizeof(double),
                          cudaMemcpyDeviceToDevice, s));
  const Dims dfp{{h->df.n[0], h->df.n[1], 1}};
  k_zero_constrained<double><<<grid_for(h->pf_n), 256, 0, s>>>(h->yf, dfp, lines);
  k_restrict_axis<double><<<grid_for(d1.n[0] * d1.n[1]), 256, 0, s>>>(h->I, 1, d1, h->yf, h->t1);
  k_restrict_axis<double><<<grid_for(h->pc_n), 256, 0, s>>>(h->I, 0, dp, h->t1, h->pc);
  k_zero_constrained<double><<<grid_for(h->pc_n), 256, 0, s>>>(h->pc, dp, lines);
  double *top = dst + h->nC - h->pc_n;
  k_axpby2<double><<<grid_for(h->pc_n), 256, 0, s>>>(1.0, top, 1.0, h->pc, top, h->pc_n);
  h->launches += 5;
  MG_CUDA(cudaGetLastError());
  return MF_OK;
}
