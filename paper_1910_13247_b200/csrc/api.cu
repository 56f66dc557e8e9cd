// api.cu -- the C ABI of include/mf.h: operator setup, apply (with the z-slab
// halo exchange over NCCL), diagonal, eigenvalue estimate, Chebyshev and the
// preconditioned CG host loop (§8(a) a8-a10, §8(b)).
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <thread>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace mf;

struct mf_op {
  Geo g;
  Tables t;
  int rank = 0, world = 1, device = 0;
  cudaStream_t stream = 0;
  int64_t n_local = 0, first_global = 0, n_global = 0, n_owned = 0, plane = 0;
  int variant = kVariantAuto;
  int64_t launches = 0;
  double *metric = nullptr;  // [ncomp][cells][q] for MF_GEOM_SINE
  // solver scratch (lazily allocated, n_local each)
  double *diag = nullptr, *dinv = nullptr;
  double *r = nullptr, *p = nullptr, *v = nullptr, *z = nullptr, *cd = nullptr, *cax = nullptr;
  // FP32 copies / scratch for the mixed-precision multigrid (lazily allocated)
  float *metric_f = nullptr, *dinv_f = nullptr, *cd_f = nullptr, *cax_f = nullptr;
  float *r_f = nullptr, *z_f = nullptr;  // mixed-precision Chebyshev-PCG (mf_cg_params.precision = 1)
  // dev_scal / host_scal (16 doubles): [0..3) dots, [8] p.v, [9] r.r, [10], [11] r.z (ping-pong)
  double *partials = nullptr, *dev_scal = nullptr, *host_scal = nullptr;
  unsigned *ticket = nullptr;  // last-block counter of the one-pass dot kernels
  double *h_src = nullptr, *h_dst = nullptr;  // device buffers for mf_apply_host
  double *recv_lo = nullptr, *recv_hi = nullptr;
  ncclComm_t comm = nullptr;
  // halo overlap (§8(e)): the boundary cell layers first, the NCCL exchange of the shared
  // planes on comm_stream while the interior layers run on stream
  bool zsplit = false;  // world > 1, or MF_ZSPLIT=1 (the same launch sequence on one GPU)
  // world > 1 without an NCCL unique id: the rank's slab operator with no communicator; the
  // apply / diagonal return local partial sums on the shared planes, the caller exchanges them
  bool detached = false;
  bool dg = false;      // discontinuous (SIP) discretization, mf_create_dg
  bool hex = false;     // unstructured hex mesh, mf_create_hex (device arrays in hx)
  HexDev hx{};
  // pipelined mf_apply_host: copy-in / copy-out streams and per-range events
  cudaStream_t h2d_s = nullptr, d2h_s = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
  // live kernel timing (mf_set_kernel_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // pairs (start, stop)
  size_t ev_used = 0;
};

static thread_local std::string g_err;
static mf_status stream_wait(mf_op *op);

static mf_status fail(mf_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(call)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(e_ == cudaErrorMemoryAllocation ? MF_ERR_OUT_OF_MEMORY : MF_ERR_CUDA,      \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                       \
  } while (0)

#define NCCL_TRY(call)                                                                                   \
  do {                                                                                                   \
    ncclResult_t r_ = (call);                                                                            \
    if (r_ != ncclSuccess) return fail(MF_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define STATUS_TRY(call)          \
  do {                            \
    mf_status s_ = (call);        \
    if (s_ != MF_OK) return s_;   \
  } while (0)

extern "C" const char *mf_last_error(void) { return g_err.c_str(); }
mf_status mf_set_error(mf_status s, const std::string &msg) { return fail(s, msg); }

extern "C" mf_status mf_nccl_unique_id(uint8_t *out128) {
  if (!out128) return fail(MF_ERR_ARGUMENT, "null output");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "NCCL unique id is 128 bytes");
  std::memcpy(out128, &id, 128);
  return MF_OK;
}

static int ncomp(int dim) { return dim == 3 ? 6 : 3; }
static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
static int64_t ncells_local(const Geo &g) { return g.nc[0] * g.nc[1] * (g.dim == 3 ? g.nc[2] : 1); }

static mf_status check_mesh(const mf_mesh *mesh, int32_t degree) {
  if (!mesh) return fail(MF_ERR_ARGUMENT, "null mesh");
  if (mesh->dim != 2 && mesh->dim != 3) return fail(MF_ERR_ARGUMENT, "dim must be 2 or 3");
  if (degree < 1 || degree > 8) return fail(MF_ERR_ARGUMENT, "degree must be in 1..8");
  for (int e = 0; e < mesh->dim; ++e) {
    if (mesh->n_cells[e] < 1) return fail(MF_ERR_ARGUMENT, "n_cells must be >= 1");
    if (!(mesh->lower[e] < mesh->upper[e])) return fail(MF_ERR_ARGUMENT, "lower must be < upper");
  }
  return MF_OK;
}

extern "C" mf_status mf_partition(const mf_mesh *mesh, int32_t degree, int32_t rank, int32_t world,
                                  int64_t *cz0, int64_t *cz1, int64_t *first_global, int64_t *n_local,
                                  int64_t *n_owned, int64_t *plane) {
  STATUS_TRY(check_mesh(mesh, degree));
  if (world < 1 || rank < 0 || rank >= world) return fail(MF_ERR_ARGUMENT, "bad rank/world_size");
  const bool d3 = mesh->dim == 3;
  const int64_t nz = d3 ? mesh->n_cells[2] : 1;
  if (world > 1 && (!d3 || nz < world)) return fail(MF_ERR_ARGUMENT, "z-slabs need dim 3 and nz >= world_size");
  const int64_t Nx = (int64_t)degree * mesh->n_cells[0] + 1, Ny = (int64_t)degree * mesh->n_cells[1] + 1;
  const int64_t a = d3 ? (int64_t)rank * nz / world : 0, b = d3 ? (int64_t)(rank + 1) * nz / world : 1;
  const int64_t pl = Nx * Ny;
  const int64_t nl = d3 ? pl * ((int64_t)degree * (b - a) + 1) : pl;
  if (cz0) *cz0 = a;
  if (cz1) *cz1 = b;
  if (first_global) *first_global = d3 ? (int64_t)degree * a * pl : 0;
  if (n_local) *n_local = nl;
  if (n_owned) *n_owned = (world > 1 && rank < world - 1) ? nl - pl : nl;
  if (plane) *plane = pl;
  return MF_OK;
}

extern "C" mf_status mf_create(const mf_mesh *mesh, int32_t degree, const mf_coeff *coeff, const mf_dist *dist,
                               mf_op **out) {
  if (!mesh || !coeff || !out) return fail(MF_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  STATUS_TRY(check_mesh(mesh, degree));
  if (mesh->geometry != MF_GEOM_CARTESIAN && mesh->geometry != MF_GEOM_SINE)
    return fail(MF_ERR_ARGUMENT, "unknown geometry");
  if (coeff->kind != MF_COEFF_CONSTANT && coeff->kind != MF_COEFF_VARIABLE)
    return fail(MF_ERR_ARGUMENT, "unknown coefficient kind");
  if (coeff->kind == MF_COEFF_CONSTANT && !(coeff->value > 0.0))
    return fail(MF_ERR_ARGUMENT, "constant coefficient must be > 0");
  int rank = 0, world = 1, device = -1;
  if (dist) {
    rank = dist->rank;
    world = dist->world_size;
    device = dist->device;
    if (world < 1 || rank < 0 || rank >= world) return fail(MF_ERR_ARGUMENT, "bad rank/world_size");
    if (world > 1 && mesh->dim != 3) return fail(MF_ERR_ARGUMENT, "world_size > 1 needs dim 3");
    if (world > 1 && mesh->n_cells[2] < world) return fail(MF_ERR_ARGUMENT, "fewer z cell layers than ranks");
  }
  if (device >= 0) CUDA_TRY(cudaSetDevice(device));
  else CUDA_TRY(cudaGetDevice(&device));

  mf_op *op = new mf_op();
  op->rank = rank;
  op->world = world;
  op->device = device;
  op->detached = world > 1 && !dist->nccl_unique_id;
  Geo &g = op->g;
  std::memset(&g, 0, sizeof(Geo));
  g.dim = mesh->dim;
  g.k = degree;
  for (int e = 0; e < 3; ++e) {
    g.nc[e] = e < g.dim ? mesh->n_cells[e] : 1;
    g.lo[e] = e < g.dim ? mesh->lower[e] : 0.0;
    g.hi[e] = e < g.dim ? mesh->upper[e] : 1.0;
    g.h[e] = (g.hi[e] - g.lo[e]) / (double)g.nc[e];
  }
  g.ncz_global = g.nc[2];
  // z-slab of whole cell layers (mf_partition is the single source of the arithmetic)
  int64_t cz0 = 0, cz1 = 1;
  {
    mf_status ps = mf_partition(mesh, degree, rank, world, &cz0, &cz1, &op->first_global, &op->n_local,
                                &op->n_owned, &op->plane);
    if (ps != MF_OK) {
      delete op;
      return ps;
    }
  }
  g.cz0 = cz0;
  if (g.dim == 3) g.nc[2] = cz1 - cz0;
  for (int e = 0; e < 3; ++e) g.N[e] = e < g.dim ? (int64_t)degree * g.nc[e] + 1 : 1;
  g.eps = mesh->deform_eps;
  g.geom = mesh->geometry;
  g.coeff_kind = coeff->kind;
  g.coeff = coeff->value;
  g.dirichlet = mesh->dirichlet_faces & ((1u << (2 * g.dim)) - 1u);
  if (world > 1) {
    if (rank > 0) g.dirichlet &= ~16u;
    if (rank < world - 1) g.dirichlet &= ~32u;
    g.skip_top_identity = rank < world - 1;
  }
  const double vol = g.h[0] * g.h[1] * (g.dim == 3 ? g.h[2] : 1.0);
  for (int e = 0; e < g.dim; ++e) g.fcart[e] = coeff->value * vol / (g.h[e] * g.h[e]);
  build_tables(degree, &op->t);

  op->n_global = g.dim == 3 ? op->plane * ((int64_t)degree * g.ncz_global + 1) : op->n_local;

  auto cleanup = [&](mf_status s) {
    mf_destroy(op);
    return s;
  };
  if (cudaMallocHost(&op->host_scal, 16 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&op->dev_scal, 16 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&op->ticket, sizeof(unsigned)) != cudaSuccess || cudaMemset(op->ticket, 0, sizeof(unsigned)) ||
      cudaMalloc(&op->partials, 3 * kDotBlocks * sizeof(double)) != cudaSuccess)
    return cleanup(fail(MF_ERR_OUT_OF_MEMORY, "scalar buffers"));

  if (g.geom == MF_GEOM_SINE) {
    const int64_t nm = (int64_t)ncomp(g.dim) * ncells_local(g) * ipow(degree + 1, g.dim);
    if (cudaMalloc(&op->metric, nm * sizeof(double)) != cudaSuccess)
      return cleanup(fail(MF_ERR_OUT_OF_MEMORY, "metric"));
    int *bad = nullptr;
    if (cudaMalloc(&bad, sizeof(int)) != cudaSuccess) return cleanup(fail(MF_ERR_OUT_OF_MEMORY, "flag"));
    cudaMemset(bad, 0, sizeof(int));
    cudaError_t e = launch_metric(g, op->t, op->metric, bad, 0, &op->launches);
    int hbad = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(bad);
    if (e != cudaSuccess) return cleanup(fail(MF_ERR_CUDA, std::string("metric: ") + cudaGetErrorString(e)));
    if (hbad) return cleanup(fail(MF_ERR_SINGULAR, "det J <= 0 at a quadrature point"));
  }
  if (world > 1 && !op->detached) {
    ncclUniqueId id;
    std::memcpy(&id, dist->nccl_unique_id, 128);
    ncclResult_t nr = ncclCommInitRank(&op->comm, world, id, rank);
    if (nr != ncclSuccess) {
      op->comm = nullptr;
      return cleanup(fail(MF_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(nr)));
    }
    if (cudaMalloc(&op->recv_lo, op->plane * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&op->recv_hi, op->plane * sizeof(double)) != cudaSuccess)
      return cleanup(fail(MF_ERR_OUT_OF_MEMORY, "halo buffers"));
    if (cudaStreamCreateWithFlags(&op->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&op->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&op->ev_halo, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(fail(MF_ERR_CUDA, "halo stream / events"));
  }
  const char *zs = std::getenv("MF_ZSPLIT");
  op->zsplit = world > 1 || (zs && std::atoi(zs) != 0);
  *out = op;
  return MF_OK;
}

extern "C" void mf_destroy(mf_op *op) {
  if (!op) return;
  cudaFree(op->metric);
  for (float *b : {op->metric_f, op->dinv_f, op->cd_f, op->cax_f, op->r_f, op->z_f}) cudaFree(b);
  for (double *b : {op->diag, op->dinv, op->r, op->p, op->v, op->z, op->cd, op->cax, op->partials, op->dev_scal,
                    op->h_src, op->h_dst, op->recv_lo, op->recv_hi})
    cudaFree(b);
  cudaFree((void *)op->hx.cell_dofs);
  cudaFree((void *)op->hx.line_ptr);
  cudaFree((void *)op->hx.line_dof);
  cudaFree((void *)op->hx.line_w);
  cudaFree((void *)op->hx.cell_lines);
  cudaFree((void *)op->hx.dir);
  if (op->host_scal) cudaFreeHost(op->host_scal);
  cudaFree(op->ticket);
  for (cudaEvent_t e : op->ev) cudaEventDestroy(e);
  if (op->comm) ncclCommDestroy(op->comm);
  for (cudaEvent_t e : op->ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : op->ev_out) cudaEventDestroy(e);
  if (op->h2d_s) cudaStreamDestroy(op->h2d_s);
  if (op->d2h_s) cudaStreamDestroy(op->d2h_s);
  if (op->ev_bnd) cudaEventDestroy(op->ev_bnd);
  if (op->ev_halo) cudaEventDestroy(op->ev_halo);
  if (op->comm_stream) cudaStreamDestroy(op->comm_stream);
  delete op;
}

// DG-SIP operator: the same brick, discontinuous Q_k on the GLL nodes
// of each cell, DoFs cell-major; weak (Nitsche) Dirichlet on every face
extern "C" mf_status mf_create_dg(const mf_mesh *mesh, int32_t degree, const mf_coeff *coeff, mf_op **out) {
  if (!mesh || !coeff || !out) return fail(MF_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (mesh->dim != 3 || mesh->geometry != MF_GEOM_CARTESIAN || coeff->kind != MF_COEFF_CONSTANT)
    return fail(MF_ERR_ARGUMENT, "DG: 3D Cartesian brick with a constant coefficient");
  if ((mesh->dirichlet_faces & 63u) != 63u) return fail(MF_ERR_ARGUMENT, "DG: weak Dirichlet on all six faces");
  mf_op *op = nullptr;
  STATUS_TRY(mf_create(mesh, degree, coeff, nullptr, &op));
  const Geo &g = op->g;
  op->dg = true;
  op->first_global = 0;
  op->n_local = op->n_global = op->n_owned = g.nc[0] * g.nc[1] * g.nc[2] * ipow(degree + 1, 3);
  *out = op;
  return MF_OK;
}

// Unstructured hex mesh: cell_dofs / constraint lines / Dirichlet list
// checked and copied to the device, the trilinear metric computed once
extern "C" mf_status mf_create_hex(const mf_hex_mesh *m, int32_t degree, const mf_coeff *coeff, mf_op **out) {
  if (!m || !coeff || !out) return fail(MF_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (degree < 1 || degree > 8) return fail(MF_ERR_ARGUMENT, "degree must be in 1..8");
  if (coeff->kind != MF_COEFF_CONSTANT && coeff->kind != MF_COEFF_VARIABLE)
    return fail(MF_ERR_ARGUMENT, "unknown coefficient kind");
  if (coeff->kind == MF_COEFF_CONSTANT && !(coeff->value > 0.0))
    return fail(MF_ERR_ARGUMENT, "constant coefficient must be > 0");
  if (m->n_cells < 0 || m->n_vertices < 1 || m->n_dofs < 1 || m->n_dofs > INT32_MAX || m->n_lines < 0 ||
      m->n_dirichlet < 0)
    return fail(MF_ERR_ARGUMENT, "bad sizes");
  if (!m->vertices || !m->cell_vertices || !m->cell_dofs || (m->n_lines > 0 && (!m->line_ptr || !m->line_dof ||
                                                                                !m->line_w)) ||
      (m->n_dirichlet > 0 && !m->dirichlet_dofs))
    return fail(MF_ERR_ARGUMENT, "null array");
  const int64_t NV = ipow(degree + 1, 3), nc = m->n_cells, nd = m->n_dofs;
  for (int64_t i = 0; i < 8 * nc; ++i)
    if (m->cell_vertices[i] < 0 || m->cell_vertices[i] >= m->n_vertices)
      return fail(MF_ERR_ARGUMENT, "cell_vertices entry out of range");
  std::vector<uint8_t> is_dir(nd, 0);
  for (int64_t i = 0; i < m->n_dirichlet; ++i) {
    const int32_t d = m->dirichlet_dofs[i];
    if (d < 0 || d >= nd) return fail(MF_ERR_ARGUMENT, "dirichlet_dofs entry out of range");
    is_dir[d] = 1;
  }
  std::vector<int32_t> dir;
  for (int64_t d = 0; d < nd; ++d)
    if (is_dir[d]) dir.push_back((int32_t)d);
  // constraint lines without their Dirichlet entries (those values are zero)
  std::vector<int32_t> lp(1, 0), ld;
  std::vector<double> lw;
  if (m->n_lines > 0 && (m->line_ptr[0] != 0)) return fail(MF_ERR_ARGUMENT, "line_ptr[0] != 0");
  for (int64_t l = 0; l < m->n_lines; ++l) {
    if (m->line_ptr[l + 1] < m->line_ptr[l]) return fail(MF_ERR_ARGUMENT, "line_ptr not monotone");
    for (int32_t j = m->line_ptr[l]; j < m->line_ptr[l + 1]; ++j) {
      const int32_t d = m->line_dof[j];
      if (d < 0 || d >= nd) return fail(MF_ERR_ARGUMENT, "line_dof entry out of range");
      if (is_dir[d]) continue;
      ld.push_back(d);
      lw.push_back(m->line_w[j]);
    }
    lp.push_back((int32_t)ld.size());
  }
  std::vector<int32_t> cd(m->cell_dofs, m->cell_dofs + nc * NV);
  std::vector<uint8_t> cl(nc, 0);
  for (int64_t c = 0; c < nc; ++c)
    for (int64_t i = 0; i < NV; ++i) {
      int32_t &d = cd[c * NV + i];
      if (d >= 0) {
        if (d >= nd) return fail(MF_ERR_ARGUMENT, "cell_dofs entry >= n_dofs");
        if (is_dir[d]) d = kHexDirichlet;
      } else {
        if (d == kHexDirichlet || -1 - (int64_t)d >= m->n_lines)
          return fail(MF_ERR_ARGUMENT, "cell_dofs refers to a missing constraint line");
        cl[c] = 1;
      }
    }
  int device = 0;
  CUDA_TRY(cudaGetDevice(&device));
  mf_op *op = new mf_op();
  op->device = device;
  op->hex = true;
  Geo &g = op->g;
  std::memset(&g, 0, sizeof(Geo));
  g.dim = 3;
  g.k = degree;
  g.nc[0] = nc;
  g.nc[1] = g.nc[2] = 1;
  g.geom = MF_GEOM_SINE;  // a stored metric (reported as curved geometry)
  g.coeff_kind = coeff->kind;
  g.coeff = coeff->value;
  build_tables(degree, &op->t);
  op->n_local = op->n_global = op->n_owned = nd;
  auto cleanup = [&](mf_status st) {
    mf_destroy(op);
    return st;
  };
  auto upload = [&](const void *h, size_t bytes, void **d) -> bool {
    if (bytes == 0) bytes = 8;  // a valid pointer for empty arrays
    if (cudaMalloc(d, bytes) != cudaSuccess) return false;
    return h == nullptr || cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  HexDev &h = op->hx;
  h.ncells = nc;
  h.ndofs = nd;
  h.ndir = (int64_t)dir.size();
  void *p_cd, *p_lp, *p_ld, *p_lw, *p_cl, *p_dir, *p_v = nullptr, *p_cv = nullptr;
  bool ok = upload(cd.data(), cd.size() * 4, &p_cd) && upload(lp.data(), lp.size() * 4, &p_lp) &&
            upload(ld.empty() ? nullptr : ld.data(), ld.size() * 4, &p_ld) &&
            upload(lw.empty() ? nullptr : lw.data(), lw.size() * 8, &p_lw) && upload(cl.data(), cl.size(), &p_cl) &&
            upload(dir.empty() ? nullptr : dir.data(), dir.size() * 4, &p_dir);
  h.cell_dofs = (const int32_t *)p_cd;
  h.line_ptr = (const int32_t *)p_lp;
  h.line_dof = (const int32_t *)p_ld;
  h.line_w = (const double *)p_lw;
  h.cell_lines = (const uint8_t *)p_cl;
  h.dir = (const int32_t *)p_dir;
  if (!ok) return cleanup(fail(MF_ERR_OUT_OF_MEMORY, "hex mesh arrays"));
  if (cudaMallocHost(&op->host_scal, 16 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&op->dev_scal, 16 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&op->ticket, sizeof(unsigned)) != cudaSuccess || cudaMemset(op->ticket, 0, sizeof(unsigned)) ||
      cudaMalloc(&op->partials, 3 * kDotBlocks * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&op->metric, 6 * nc * NV * sizeof(double) + 8) != cudaSuccess)
    return cleanup(fail(MF_ERR_OUT_OF_MEMORY, "scalar / metric buffers"));
  h.metric = op->metric;
  int *bad = nullptr;
  ok = upload(m->vertices, m->n_vertices * 3 * sizeof(double), &p_v) &&
       upload(m->cell_vertices, nc * 8 * sizeof(int32_t), &p_cv) && cudaMalloc(&bad, sizeof(int)) == cudaSuccess;
  cudaError_t e = ok ? cudaMemset(bad, 0, sizeof(int)) : cudaErrorMemoryAllocation;
  if (e == cudaSuccess)
    e = launch_hex_metric(degree, op->t, (const double *)p_v, (const int32_t *)p_cv, nc, coeff->kind, coeff->value,
                          op->metric, bad, 0, &op->launches);
  int hbad = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  cudaFree(p_v);
  cudaFree(p_cv);
  if (e != cudaSuccess) return cleanup(fail(MF_ERR_CUDA, std::string("hex metric: ") + cudaGetErrorString(e)));
  if (hbad) return cleanup(fail(MF_ERR_SINGULAR, "det J <= 0 at a quadrature point"));
  *out = op;
  return MF_OK;
}

extern "C" mf_status mf_hex_number_dofs(int32_t degree, int64_t n_cells, const int32_t *cell_vertices,
                                        int32_t *cell_dofs, int64_t *n_dofs, uint8_t *is_boundary,
                                        int64_t capacity) {
  if (!cell_vertices || !cell_dofs || !n_dofs) return fail(MF_ERR_ARGUMENT, "null argument");
  if (degree < 1 || degree > 8) return fail(MF_ERR_ARGUMENT, "degree must be in 1..8");
  if (n_cells < 0) return fail(MF_ERR_ARGUMENT, "n_cells < 0");
  std::string err;
  mf_status st = hex_number_dofs(degree, n_cells, cell_vertices, cell_dofs, n_dofs, is_boundary, capacity, &err);
  return st == MF_OK ? MF_OK : fail(st, err);
}

extern "C" mf_status mf_sizes(const mf_op *op, int64_t *n_local, int64_t *first_global, int64_t *n_global,
                              int64_t *n_owned) {
  if (!op) return fail(MF_ERR_ARGUMENT, "null op");
  if (n_local) *n_local = op->n_local;
  if (first_global) *first_global = op->first_global;
  if (n_global) *n_global = op->n_global;
  if (n_owned) *n_owned = op->n_owned;
  return MF_OK;
}

extern "C" mf_status mf_set_stream(mf_op *op, void *s) {
  if (!op) return fail(MF_ERR_ARGUMENT, "null op");
  op->stream = (cudaStream_t)s;
  return MF_OK;
}

static int chosen_variant(const mf_op *op) {
  if (op->hex) return kVariantHex;
  if (op->dg) return kVariantDG;
  if (op->variant != kVariantAuto) return op->variant;
  if (cart_halo_supported(op->g)) return kVariantCartHalo;
  return cart_plane_supported(op->g) ? kVariantCartPlane : kVariantGeneral;
}

extern "C" mf_status mf_set_apply_variant(mf_op *op, int32_t variant) {
  if (!op) return fail(MF_ERR_ARGUMENT, "null op");
  if (op->hex || op->dg) return fail(MF_ERR_ARGUMENT, "DG / hex operators have one kernel family");
  if (variant == kVariantCartTile)
    return fail(MF_ERR_ARGUMENT, "variant 2 (the slab-form tile kernel) was removed: use 3 (plane) or 6 (halo)");
  if (variant == kVariantCartPlane && !cart_plane_supported(op->g))
    return fail(MF_ERR_ARGUMENT, "the plane kernel needs dim 3, Cartesian geometry, constant coefficient, k 2..4");
  if (variant == kVariantCartHalo && !cart_halo_supported(op->g))
    return fail(MF_ERR_ARGUMENT,
                "halo kernel needs dim 3, Cartesian, constant coefficient, k 4, n_cells x <= 256, and Dirichlet "
                "x+ / y+ faces when n_cells x % 32 == 0 / n_cells y % 2 == 0");
  if (variant < 0 || (variant > kVariantCartPlane && variant != kVariantCartHalo))
    return fail(MF_ERR_ARGUMENT, "unknown variant");
  op->variant = variant;
  return MF_OK;
}

// symmetric exchange of the partial sums on shared z-planes (§8(e)):
// send my partial of each shared plane, receive the neighbour's (on stream s) ...
static mf_status halo_post(mf_op *op, double *dst, cudaStream_t s) {
  if (!op->comm) return fail(MF_ERR_NCCL, "communicator was aborted after an earlier NCCL error");
  const int64_t np = op->plane;
  double *lo = dst, *hi = dst + op->n_local - np;
  const bool has_lo = op->rank > 0, has_hi = op->rank < op->world - 1;
  NCCL_TRY(ncclGroupStart());
  if (has_hi) {
    NCCL_TRY(ncclSend(hi, np, ncclDouble, op->rank + 1, op->comm, s));
    NCCL_TRY(ncclRecv(op->recv_hi, np, ncclDouble, op->rank + 1, op->comm, s));
  }
  if (has_lo) {
    NCCL_TRY(ncclSend(lo, np, ncclDouble, op->rank - 1, op->comm, s));
    NCCL_TRY(ncclRecv(op->recv_lo, np, ncclDouble, op->rank - 1, op->comm, s));
  }
  NCCL_TRY(ncclGroupEnd());
  return MF_OK;
}

// ... and add it (on op->stream; a+b = b+a, so both copies of a shared plane agree bitwise)
static mf_status halo_add(mf_op *op, double *dst) {
  const int64_t np = op->plane;
  double *lo = dst, *hi = dst + op->n_local - np;
  if (op->rank < op->world - 1) CUDA_TRY(launch_plane_add(hi, op->recv_hi, np, op->stream, &op->launches));
  if (op->rank > 0) CUDA_TRY(launch_plane_add(lo, op->recv_lo, np, op->stream, &op->launches));
  return MF_OK;
}

static mf_status halo_exchange(mf_op *op, double *dst) {
  if (op->world == 1 || op->detached) return MF_OK;
  STATUS_TRY(halo_post(op, dst, op->stream));
  return halo_add(op, dst);
}

static mf_status timing_mark(mf_op *op) {
  if (!op->timing) return MF_OK;
  if (op->ev_used == op->ev.size()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    op->ev.push_back(e);
  }
  CUDA_TRY(cudaEventRecord(op->ev[op->ev_used++], op->stream));
  return MF_OK;
}

// the overlapped apply on z-slabs: part 1 (dst init + the cell layers next to the
// shared planes), then the NCCL exchange of those planes on comm_stream while part 2
// (the interior layers, which never touch the shared planes) runs on stream
static mf_status apply_split(mf_op *op, const double *src, double *dst, int var) {
  STATUS_TRY(timing_mark(op));
  if (var == kVariantCartHalo) {
    CUDA_TRY(launch_apply_cart_halo(op->g, op->t, src, dst, op->stream, &op->launches, 1));
  } else if (var == kVariantCartPlane) {
    CUDA_TRY(launch_apply_cart_plane(op->g, op->t, src, dst, op->stream, &op->launches, 1));
  } else {
    CUDA_TRY(launch_zero(dst, op->n_local, op->stream, &op->launches));
    CUDA_TRY(launch_apply_general(op->g, op->t, src, dst, op->metric, op->stream, &op->launches, 1));
  }
  if (op->world > 1 && !op->detached) {
    CUDA_TRY(cudaEventRecord(op->ev_bnd, op->stream));
    CUDA_TRY(cudaStreamWaitEvent(op->comm_stream, op->ev_bnd, 0));
    STATUS_TRY(halo_post(op, dst, op->comm_stream));
    CUDA_TRY(cudaEventRecord(op->ev_halo, op->comm_stream));
  }
  if (var == kVariantCartHalo)
    CUDA_TRY(launch_apply_cart_halo(op->g, op->t, src, dst, op->stream, &op->launches, 2));
  else if (var == kVariantCartPlane)
    CUDA_TRY(launch_apply_cart_plane(op->g, op->t, src, dst, op->stream, &op->launches, 2));
  else
    CUDA_TRY(launch_apply_general(op->g, op->t, src, dst, op->metric, op->stream, &op->launches, 2));
  STATUS_TRY(timing_mark(op));
  if (op->world > 1 && !op->detached) {
    CUDA_TRY(cudaStreamWaitEvent(op->stream, op->ev_halo, 0));
    STATUS_TRY(halo_add(op, dst));
  }
  return MF_OK;
}

extern "C" mf_status mf_apply_split_part(mf_op *op, const double *src, int64_t n_src, double *dst, int64_t n_dst,
                                         int32_t part) {
  if (!op || !src || !dst) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n_src != op->n_local || n_dst != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  if (op->hex || op->dg || op->g.dim != 3 || (part != 1 && part != 2))
    return fail(MF_ERR_ARGUMENT, "split parts: 3D brick operator, part 1 or 2");
  const int var = chosen_variant(op);
  if (var == kVariantCartHalo) {
    CUDA_TRY(launch_apply_cart_halo(op->g, op->t, src, dst, op->stream, &op->launches, part));
  } else if (var == kVariantCartPlane) {
    CUDA_TRY(launch_apply_cart_plane(op->g, op->t, src, dst, op->stream, &op->launches, part));
  } else {
    if (part == 1) CUDA_TRY(launch_zero(dst, op->n_local, op->stream, &op->launches));
    CUDA_TRY(launch_apply_general(op->g, op->t, src, dst, op->metric, op->stream, &op->launches, part));
  }
  return MF_OK;
}

static mf_status apply_impl(mf_op *op, const double *src, double *dst) {
  if (op->hex) {
    STATUS_TRY(timing_mark(op));
    CUDA_TRY(launch_zero(dst, op->n_local, op->stream, &op->launches));
    CUDA_TRY(launch_apply_hex(op->g.k, op->t, op->hx, src, dst, op->stream, &op->launches));
    return timing_mark(op);
  }
  if (op->dg) {
    STATUS_TRY(timing_mark(op));
    CUDA_TRY(launch_apply_dg(op->g, op->t, src, dst, op->stream, &op->launches));
    return timing_mark(op);
  }
  const int var = chosen_variant(op);
  if (op->zsplit && op->g.dim == 3) return apply_split(op, src, dst, var);
  if (var == kVariantCartHalo) {
    STATUS_TRY(timing_mark(op));
    CUDA_TRY(launch_apply_cart_halo(op->g, op->t, src, dst, op->stream, &op->launches));
    STATUS_TRY(timing_mark(op));
  } else if (var == kVariantCartPlane) {
    STATUS_TRY(timing_mark(op));
    CUDA_TRY(launch_apply_cart_plane(op->g, op->t, src, dst, op->stream, &op->launches));
    STATUS_TRY(timing_mark(op));
  } else {
    STATUS_TRY(timing_mark(op));  // (zeroing + kernel, as the plane path's init + kernel)
    CUDA_TRY(launch_zero(dst, op->n_local, op->stream, &op->launches));
    CUDA_TRY(launch_apply_general(op->g, op->t, src, dst, op->metric, op->stream, &op->launches));
    STATUS_TRY(timing_mark(op));
  }
  return halo_exchange(op, dst);
}

extern "C" mf_status mf_set_kernel_timing(mf_op *op, int32_t enable) {
  if (!op) return fail(MF_ERR_ARGUMENT, "null op");
  op->timing = enable != 0;
  if (op->timing) op->ev_used = 0;  // a new window; disabling keeps the events for mf_kernel_timing
  return MF_OK;
}

extern "C" mf_status mf_kernel_timing(mf_op *op, double *ms_total, int64_t *count) {
  if (!op || !ms_total || !count) return fail(MF_ERR_ARGUMENT, "null argument");
  double total = 0.0;
  for (size_t i = 0; i + 1 < op->ev_used; i += 2) {
    CUDA_TRY(cudaEventSynchronize(op->ev[i + 1]));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, op->ev[i], op->ev[i + 1]));
    total += ms;
  }
  *ms_total = total;
  *count = (int64_t)(op->ev_used / 2);
  return MF_OK;
}

extern "C" mf_status mf_apply(mf_op *op, const double *src, int64_t n_src, double *dst, int64_t n_dst) {
  if (!op || !src || !dst) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n_src != op->n_local || n_dst != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  if (src == dst) return fail(MF_ERR_ARGUMENT, "src and dst must be distinct");
  return apply_impl(op, src, dst);
}

extern "C" mf_status mf_apply_host(mf_op *op, const double *src_host, int64_t n_src, double *dst_host,
                                   int64_t n_dst) {
  if (!op || !src_host || !dst_host) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n_src != op->n_local || n_dst != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  const size_t bytes = op->n_local * sizeof(double);
  if (!op->h_src) {
    CUDA_TRY(cudaMalloc(&op->h_src, bytes));
    CUDA_TRY(cudaMalloc(&op->h_dst, bytes));
  }
  const Geo &g = op->g;
  const char *pe = std::getenv("MF_HOST_PIPELINE");
  const int C = (pe && std::atoi(pe) > 0) ? std::atoi(pe) : 8;
  const int var = chosen_variant(op);
  const bool pipelined = !op->hex && op->world == 1 && g.dim == 3 &&
                         (var == kVariantCartPlane || var == kVariantCartHalo || var == kVariantGeneral ||
                          var == kVariantDG) &&
                         C > 1 &&
                         g.nc[2] >= 2 * C;
  if (!pipelined) {
    CUDA_TRY(cudaMemcpyAsync(op->h_src, src_host, bytes, cudaMemcpyHostToDevice, op->stream));
    STATUS_TRY(apply_impl(op, op->h_src, op->h_dst));
    CUDA_TRY(cudaMemcpyAsync(dst_host, op->h_dst, bytes, cudaMemcpyDeviceToHost, op->stream));
    STATUS_TRY(stream_wait(op));
    return MF_OK;
  }
  // Pipelined: the cell layers in C z-ranges; range r's input planes go up on h2d_s, its
  // apply (init / zeroing + kernel for those layers) runs on the op's stream once they are in,
  // and its finished output planes come down on d2h_s while range r+1 is copied in and
  // computed -- host->device and device->host transfers overlap (full duplex).
  if (!op->h2d_s) {
    CUDA_TRY(cudaStreamCreateWithFlags(&op->h2d_s, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&op->d2h_s, cudaStreamNonBlocking));
  }
  while ((int)op->ev_in.size() < C) {
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    op->ev_in.push_back(a);
    op->ev_out.push_back(b);
  }
  const int64_t K = g.k, nz = g.nc[2], pl = op->plane;
  // the previous call's work on the op's stream is done before its buffers are reused
  CUDA_TRY(cudaEventRecord(op->ev_out[C - 1], op->stream));
  CUDA_TRY(cudaStreamWaitEvent(op->h2d_s, op->ev_out[C - 1], 0));
  if (var == kVariantDG) {
    // DG: cell-major DoFs, a cell layer is one contiguous run of L DoFs; range r computes
    // layers [z0, z1) and needs layer z1 for the z-couplings of its top layer
    const int64_t layer = g.nc[0] * g.nc[1], L = layer * ipow(K + 1, 3);
    int64_t up = 0;  // layers uploaded so far
    for (int r = 0; r < C; ++r) {
      const int64_t z0 = nz * r / C, z1 = nz * (r + 1) / C, need = std::min(z1 + 1, nz);
      if (need > up) {
        CUDA_TRY(cudaMemcpyAsync(op->h_src + up * L, src_host + up * L, (need - up) * L * sizeof(double),
                                 cudaMemcpyHostToDevice, op->h2d_s));
        up = need;
      }
      CUDA_TRY(cudaEventRecord(op->ev_in[r], op->h2d_s));
      CUDA_TRY(cudaStreamWaitEvent(op->stream, op->ev_in[r], 0));
      CUDA_TRY(launch_apply_dg(g, op->t, op->h_src, op->h_dst, op->stream, &op->launches, z0 * layer, z1 * layer));
      CUDA_TRY(cudaEventRecord(op->ev_out[r], op->stream));
      CUDA_TRY(cudaStreamWaitEvent(op->d2h_s, op->ev_out[r], 0));
      CUDA_TRY(cudaMemcpyAsync(dst_host + z0 * L, op->h_dst + z0 * L, (z1 - z0) * L * sizeof(double),
                               cudaMemcpyDeviceToHost, op->d2h_s));
    }
    CUDA_TRY(cudaStreamSynchronize(op->d2h_s));
    CUDA_TRY(cudaStreamSynchronize(op->stream));
    return MF_OK;
  }
  for (int r = 0; r < C; ++r) {
    const int64_t z0 = nz * r / C, z1 = nz * (r + 1) / C;
    const int64_t in0 = r == 0 ? 0 : K * z0 + 1, in1 = K * z1;  // node planes, inclusive
    CUDA_TRY(cudaMemcpyAsync(op->h_src + in0 * pl, src_host + in0 * pl, (in1 - in0 + 1) * pl * sizeof(double),
                             cudaMemcpyHostToDevice, op->h2d_s));
    CUDA_TRY(cudaEventRecord(op->ev_in[r], op->h2d_s));
    CUDA_TRY(cudaStreamWaitEvent(op->stream, op->ev_in[r], 0));
    if (var == kVariantCartHalo) {  // owner-writes: no zeroing, planes shared with range r+1 written there
      CUDA_TRY(launch_apply_cart_halo(g, op->t, op->h_src, op->h_dst, op->stream, &op->launches, 3, (int)z0,
                                      (int)z1));
    } else if (var == kVariantCartPlane) {
      CUDA_TRY(launch_apply_cart_plane_range(g, op->t, op->h_src, op->h_dst, op->stream, &op->launches, (int)z0,
                                             (int)z1));
    } else {  // zero the planes no earlier range has touched, then add this range's cells
      CUDA_TRY(launch_zero(op->h_dst + in0 * pl, (in1 - in0 + 1) * pl, op->stream, &op->launches));
      const int64_t layer = g.nc[0] * g.nc[1];
      CUDA_TRY(launch_apply_general_cells(g, op->t, op->h_src, op->h_dst, op->metric, op->stream, &op->launches,
                                          z0 * layer, z1 * layer));
    }
    CUDA_TRY(cudaEventRecord(op->ev_out[r], op->stream));
    const int64_t out0 = K * z0, out1 = r == C - 1 ? K * z1 : K * z1 - 1;  // finished planes
    CUDA_TRY(cudaStreamWaitEvent(op->d2h_s, op->ev_out[r], 0));
    CUDA_TRY(cudaMemcpyAsync(dst_host + out0 * pl, op->h_dst + out0 * pl, (out1 - out0 + 1) * pl * sizeof(double),
                             cudaMemcpyDeviceToHost, op->d2h_s));
  }
  CUDA_TRY(cudaStreamSynchronize(op->d2h_s));
  CUDA_TRY(cudaStreamSynchronize(op->stream));
  return MF_OK;
}

static mf_status diagonal_impl(mf_op *op, double *diag) {
  if (op->hex) {
    CUDA_TRY(launch_zero(diag, op->n_local, op->stream, &op->launches));
    CUDA_TRY(launch_diagonal_hex(op->g.k, op->t, op->hx, diag, op->stream, &op->launches));
    return MF_OK;
  }
  if (op->dg) {
    CUDA_TRY(launch_diagonal_dg(op->g, op->t, diag, op->stream, &op->launches));
    return MF_OK;
  }
  CUDA_TRY(launch_zero(diag, op->n_local, op->stream, &op->launches));
  CUDA_TRY(launch_diagonal(op->g, op->t, diag, op->metric, op->stream, &op->launches));
  return halo_exchange(op, diag);
}

extern "C" mf_status mf_diagonal(mf_op *op, double *diag, int64_t n) {
  if (!op || !diag) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  return diagonal_impl(op, diag);
}

static mf_status ensure_solver(mf_op *op) {
  // the solvers apply A repeatedly: a detached slab has no exchange, so they are refused
  if (op->detached) return fail(MF_ERR_ARGUMENT, "detached slab operator: solvers need a communicator");
  if (op->r) return MF_OK;
  const size_t bytes = op->n_local * sizeof(double);
  for (double **b : {&op->diag, &op->dinv, &op->r, &op->p, &op->v, &op->z, &op->cd, &op->cax})
    CUDA_TRY(cudaMalloc(b, bytes));
  STATUS_TRY(diagonal_impl(op, op->diag));
  CUDA_TRY(launch_recip(op->diag, op->dinv, op->n_local, op->stream, &op->launches));
  return MF_OK;
}

// Wait for the op's stream.  With world_size > 1 the wait polls the communicator:
// ncclCommGetAsyncError != ncclSuccess, or no completion within MF_NCCL_TIMEOUT_S seconds
// (a peer died or hung), aborts it and returns MF_ERR_NCCL (SURVEY §5 failure detection).
static mf_status stream_wait(mf_op *op) {
  if (op->world == 1 || op->detached) {
    CUDA_TRY(cudaStreamSynchronize(op->stream));
    return MF_OK;
  }
  if (!op->comm) return fail(MF_ERR_NCCL, "communicator was aborted after an earlier NCCL error");
  static const double timeout_s = [] {
    const char *e = std::getenv("MF_NCCL_TIMEOUT_S");
    return e && std::atof(e) > 0 ? std::atof(e) : 300.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (long it = 0;; ++it) {
    cudaError_t q = cudaStreamQuery(op->stream);
    if (q == cudaSuccess) return MF_OK;
    if (q != cudaErrorNotReady) return fail(MF_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(op->comm, &ar);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ar != ncclSuccess && ar != ncclInProgress) || el > timeout_s) {
      ncclCommAbort(op->comm);
      op->comm = nullptr;
      return fail(MF_ERR_NCCL, ar != ncclSuccess ? std::string("NCCL async error: ") + ncclGetErrorString(ar)
                                                  : std::string("no progress within MF_NCCL_TIMEOUT_S; "
                                                                "communicator aborted"));
    }
    if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

extern "C" mf_status mf_sync(mf_op *op) {
  if (!op) return fail(MF_ERR_ARGUMENT, "null op");
  return stream_wait(op);
}

// nd dot products over the owned prefix, summed over ranks; result to host_scal[0..nd)
static mf_status dots(mf_op *op, int nd, const double *const *a, const double *const *b) {
  if (op->detached) return fail(MF_ERR_ARGUMENT, "detached slab operator: collective calls need a communicator");
  CUDA_TRY(launch_dots(nd, a, b, op->n_owned, op->partials, op->ticket, op->dev_scal, op->stream, &op->launches));
  if (op->world > 1) {
    if (!op->comm) return fail(MF_ERR_NCCL, "communicator was aborted after an earlier NCCL error");
    NCCL_TRY(ncclAllReduce(op->dev_scal, op->dev_scal, nd, ncclDouble, ncclSum, op->comm, op->stream));
  }
  CUDA_TRY(cudaMemcpyAsync(op->host_scal, op->dev_scal, nd * sizeof(double), cudaMemcpyDeviceToHost, op->stream));
  return stream_wait(op);
}

// a device scalar summed over the ranks, in stream order (no host synchronisation)
static mf_status allreduce_dev(mf_op *op, double *x, int nd = 1) {
  if (op->world == 1) return MF_OK;
  if (op->detached) return fail(MF_ERR_ARGUMENT, "detached slab operator: collective calls need a communicator");
  if (!op->comm) return fail(MF_ERR_NCCL, "communicator was aborted after an earlier NCCL error");
  NCCL_TRY(ncclAllReduce(x, x, nd, ncclDouble, ncclSum, op->comm, op->stream));
  return MF_OK;
}

// out_dev = a.b over the owned prefix, summed over ranks; launched only (stream order)
mf_status dot_dev(mf_op *op, const double *a, const double *b, double *out_dev) {
  const double *aa[1] = {a}, *bb[1] = {b};
  CUDA_TRY(launch_dots(1, aa, bb, op->n_owned, op->partials, op->ticket, out_dev, op->stream, &op->launches));
  return allreduce_dev(op, out_dev);
}

// largest eigenvalue of the symmetric tridiagonal (d, e) by Sturm-sequence bisection
static double tridiag_max_eig(const std::vector<double> &d, const std::vector<double> &e) {
  const int m = (int)d.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {
    double r = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  auto count_below = [&](double x) {
    int c = 0;
    double q = 1.0;
    for (int i = 0; i < m; ++i) {
      q = d[i] - x - (i > 0 ? e[i - 1] * e[i - 1] / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-16 * std::max(std::fabs(hi), std::fabs(lo)); ++it) {
    double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= m) hi = mid;
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}

// O10 / S:639-647, with the reading of DESIGN.md R8
static mf_status lambda_impl(mf_op *op, int steps, double *lam) {
  STATUS_TRY(ensure_solver(op));
  const int64_t n = op->n_local;
  cudaStream_t s = op->stream;
  double *r = op->r, *z = op->z, *p = op->p, *v = op->v;
  CUDA_TRY(launch_splitmix(r, n, op->first_global, 0, s, &op->launches));
  if (op->hex) CUDA_TRY(launch_hex_set(op->hx, r, 0.0, s, &op->launches));
  else if (!op->dg) CUDA_TRY(launch_set_constrained(op->g, r, 0.0, s, &op->launches));  // (DG: no constrained DoFs)
  CUDA_TRY(launch_mul(op->dinv, r, z, n, s, &op->launches));
  CUDA_TRY(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  {
    const double *a[1] = {r}, *b[1] = {z};
    STATUS_TRY(dots(op, 1, a, b));
  }
  double rz = op->host_scal[0];
  const double rz0 = rz;
  std::vector<double> al, be;
  for (int j = 0; j < steps; ++j) {
    STATUS_TRY(apply_impl(op, p, v));
    const double *a[1] = {p}, *b[1] = {v};
    STATUS_TRY(dots(op, 1, a, b));
    const double pv = op->host_scal[0];
    if (!(pv > 0.0)) return fail(MF_ERR_BREAKDOWN, "p.Ap <= 0 in eigenvalue estimate");
    const double alpha = rz / pv;
    al.push_back(alpha);
    CUDA_TRY(launch_axpby(-alpha, v, 1.0, r, n, s, &op->launches));
    CUDA_TRY(launch_mul(op->dinv, r, z, n, s, &op->launches));
    const double *a2[1] = {r}, *b2[1] = {z};
    STATUS_TRY(dots(op, 1, a2, b2));
    const double rzn = op->host_scal[0];
    if (rzn <= 1e-28 * rz0) break;
    const double beta = rzn / rz;
    be.push_back(beta);
    CUDA_TRY(launch_axpby(1.0, z, beta, p, n, s, &op->launches));
    rz = rzn;
  }
  const int m = (int)al.size();
  std::vector<double> d(m), e(m > 0 ? m - 1 : 0);
  for (int j = 0; j < m; ++j) {
    d[j] = 1.0 / al[j] + (j > 0 ? be[j - 1] / al[j - 1] : 0.0);
    if (j + 1 < m) e[j] = std::sqrt(be[j]) / al[j];
  }
  *lam = m > 0 ? tridiag_max_eig(d, e) : 0.0;
  return MF_OK;
}

extern "C" mf_status mf_estimate_lambda_max(mf_op *op, int32_t steps, double *lambda_out) {
  if (!op || !lambda_out || steps < 1) return fail(MF_ERR_ARGUMENT, "bad argument");
  return lambda_impl(op, steps, lambda_out);
}

// O11 / S:648-656: z = Chebyshev(degree) for D^{-1}A on [lam/range, lam] from 0.  With rz_dev
// the CG's r.z is formed in the last step's pass (device scalar, summed over ranks).
static mf_status cheb_impl(mf_op *op, const double *r, double *x, double lam, int degree, double range,
                           double *rz_dev = nullptr) {
  STATUS_TRY(ensure_solver(op));
  const int64_t n = op->n_local;
  const double a = lam / range, b = lam;
  const double theta = 0.5 * (a + b), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  // three-term form (kernels_vec.cu::k_cheb3): the iterates ping-pong between x and op->cd,
  // the start x_1 = D^{-1} r / theta placed so that the last one lands in x
  const int steps = degree - 1;
  double *bx = (steps & 1) ? op->cd : x, *bp = (steps & 1) ? x : op->cd;
  CUDA_TRY(launch_cheb_init1(r, op->dinv, 1.0 / theta, bx, n, op->stream, &op->launches));
  for (int j = 1; j < degree; ++j) {
    const double rho_n = 1.0 / (2.0 * sigma - rho);
    STATUS_TRY(apply_impl(op, bx, op->cax));
    double *rz = (rz_dev && j == degree - 1) ? rz_dev : nullptr;  // r.z fused into the last step
    CUDA_TRY(launch_cheb3(r, op->cax, op->dinv, rho_n * rho, 2.0 * rho_n / delta, bx, bp, j == 1, n, op->n_owned,
                          op->partials, op->ticket, rz, op->stream, &op->launches));
    if (rz) return allreduce_dev(op, rz_dev);
    std::swap(bx, bp);
    rho = rho_n;
  }
  if (rz_dev) STATUS_TRY(dot_dev(op, r, x, rz_dev));
  return MF_OK;
}

extern "C" mf_status mf_chebyshev(mf_op *op, const double *r, double *z, int64_t n, double lambda, int32_t degree,
                                  double smoothing_range) {
  if (!op || !r || !z) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  if (degree < 1 || !(lambda > 0.0) || !(smoothing_range > 1.0)) return fail(MF_ERR_ARGUMENT, "bad parameters");
  return cheb_impl(op, r, z, lambda, degree, smoothing_range);
}

// ---- FP32 operator (mixed-precision multigrid, §8(f) f2; "run in single
// precision ... combined with some double-precision correction") ----------------
static mf_status ensure_f32(mf_op *op) {
  if (op->cd_f) return MF_OK;
  STATUS_TRY(ensure_solver(op));
  const int64_t n = op->n_local;
  CUDA_TRY(cudaMalloc(&op->dinv_f, n * sizeof(float)));
  CUDA_TRY(cudaMalloc(&op->cd_f, n * sizeof(float)));
  CUDA_TRY(cudaMalloc(&op->cax_f, n * sizeof(float)));
  CUDA_TRY(launch_d2f(op->dinv, op->dinv_f, n, op->stream, &op->launches));
  if (op->metric) {
    const int64_t nm = (int64_t)ncomp(op->g.dim) * ncells_local(op->g) * ipow(op->g.k + 1, op->g.dim);
    CUDA_TRY(cudaMalloc(&op->metric_f, nm * sizeof(float)));
    CUDA_TRY(launch_d2f(op->metric, op->metric_f, nm, op->stream, &op->launches));
  }
  return MF_OK;
}

mf_status apply_f32(mf_op *op, const float *src, float *dst) {
  if (op->world != 1 || op->g.dim != 3 || op->dg || op->hex)
    return fail(MF_ERR_ARGUMENT, "FP32 apply: 3D CG brick, one rank");
  STATUS_TRY(ensure_f32(op));
  if (chosen_variant(op) == kVariantCartPlane || chosen_variant(op) == kVariantCartHalo) {
    CUDA_TRY(launch_apply_cart_plane_f32(op->g, op->t, src, dst, op->stream, &op->launches));
  } else {
    CUDA_TRY(launch_zero_f(dst, op->n_local, op->stream, &op->launches));
    CUDA_TRY(launch_apply_general_f32(op->g, op->t, src, dst, op->metric_f, op->stream, &op->launches));
  }
  return MF_OK;
}

// the Chebyshev polynomial of cheb_impl in FP32 (coefficients rounded from FP64)
mf_status cheb_f32(mf_op *op, const float *r, float *x, double lam, int degree, double range) {
  STATUS_TRY(ensure_f32(op));
  const int64_t n = op->n_local;
  const double a = lam / range, b = lam;
  const double theta = 0.5 * (a + b), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  CUDA_TRY(launch_cheb_init_f(r, op->dinv_f, (float)(1.0 / theta), x, op->cd_f, n, op->stream, &op->launches));
  for (int j = 1; j < degree; ++j) {
    const double rho_n = 1.0 / (2.0 * sigma - rho);
    STATUS_TRY(apply_f32(op, x, op->cax_f));
    CUDA_TRY(launch_cheb_step_f(r, op->cax_f, op->dinv_f, (float)(rho_n * rho), (float)(2.0 * rho_n / delta), x,
                                op->cd_f, n, op->stream, &op->launches));
    rho = rho_n;
  }
  return MF_OK;
}

extern "C" mf_status mf_apply_f32(mf_op *op, const float *src, int64_t n_src, float *dst, int64_t n_dst) {
  if (!op || !src || !dst) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n_src != op->n_local || n_dst != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  if ((const void *)src == (const void *)dst) return fail(MF_ERR_ARGUMENT, "src and dst must be distinct");
  return apply_f32(op, src, dst);
}

// O9 / S:500-508: PCG from x0 = 0 with the preconditioner z = precond(r) (device
// buffers of n_local); stopping rule, history and errors of mf_cg_solve.  Also the
// outer loop of the multigrid solver (mg.cu).
mf_status cg_core(mf_op *op, const double *b, double *x, double rel_tol, int max_iter,
                  const std::function<mf_status(const double *, double *, double *)> &precond, mf_cg_result *res,
                  double *history, int32_t history_cap) {
  // One host synchronisation per iteration: alpha = (r.z)/(p.v) and beta = (r.z)'/(r.z) are
  // formed on the device by the update kernels, r.r is fused into the x / r update and r.z
  // into the preconditioner's last pass (precond(r, z, rz_dev) stores it); the host then
  // reads p.v, r.r and r.z together for the stopping test and the breakdown checks.  The
  // preconditioner of the final iteration runs before the test that ends the loop (unused).
  // Same arithmetic and reduction order as the host-scalar loop, so the same iterates.
  STATUS_TRY(ensure_solver(op));
  const int64_t n = op->n_local;
  cudaStream_t s = op->stream;
  double *r = op->r, *p = op->p, *v = op->v, *z = op->z;
  double *PV = op->dev_scal + 8, *RR = op->dev_scal + 9, *RZ[2] = {op->dev_scal + 10, op->dev_scal + 11};
  res->iterations = 0;
  res->final_rel_residual = 0.0;
  CUDA_TRY(launch_zero(x, n, s, &op->launches));
  CUDA_TRY(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  {
    const double *a[1] = {b}, *bb[1] = {b};
    STATUS_TRY(dots(op, 1, a, bb));
  }
  const double normb = std::sqrt(op->host_scal[0]);
  if (normb == 0.0) return MF_OK;
  int cur = 0;
  STATUS_TRY(precond(r, z, RZ[cur]));
  CUDA_TRY(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  int it = 0;
  while (true) {
    STATUS_TRY(apply_impl(op, p, v));
    ++it;
    STATUS_TRY(dot_dev(op, p, v, PV));
    CUDA_TRY(launch_cg_xr_rr(RZ[cur], PV, x, r, p, v, n, op->n_owned, op->partials, op->ticket, RR, s,
                             &op->launches));
    STATUS_TRY(allreduce_dev(op, RR));
    STATUS_TRY(precond(r, z, RZ[cur ^ 1]));
    CUDA_TRY(cudaMemcpyAsync(op->host_scal + 8, op->dev_scal + 8, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    STATUS_TRY(stream_wait(op));
    const double pv = op->host_scal[8], rr = op->host_scal[9], rzn = op->host_scal[10 + (cur ^ 1)];
    res->iterations = it;
    if (!(pv > 0.0)) return fail(MF_ERR_BREAKDOWN, "p.Ap <= 0");
    const double resn = std::sqrt(rr);
    if (history && it <= history_cap) history[it - 1] = resn;
    res->final_rel_residual = resn / normb;
    if (resn <= rel_tol * normb) return MF_OK;
    if (it >= max_iter) return fail(MF_ERR_MAX_ITERATIONS, "CG did not converge");
    if (!(rzn > 0.0)) return fail(MF_ERR_BREAKDOWN, "r.z <= 0");
    CUDA_TRY(launch_cg_p_dev(RZ[cur ^ 1], RZ[cur], z, p, n, s, &op->launches));
    cur ^= 1;
  }
}

// Chebyshev(cheb_degree)-Jacobi PCG (or plain Jacobi if 0)
extern "C" mf_status mf_cg_solve(mf_op *op, const double *b, double *x, int64_t n, const mf_cg_params *prm,
                                 mf_cg_result *res, double *history, int32_t history_cap) {
  if (!op || !b || !x || !prm || !res) return fail(MF_ERR_ARGUMENT, "null argument");
  if (n != op->n_local) return fail(MF_ERR_LENGTH, "vector length != n_local");
  if (!(prm->rel_tol > 0.0) || prm->max_iter < 1) return fail(MF_ERR_ARGUMENT, "bad CG parameters");
  STATUS_TRY(ensure_solver(op));
  res->iterations = 0;
  res->final_rel_residual = 0.0;
  res->lambda_max = 0.0;
  double lam = 0.0;
  if (prm->cheb_degree > 0) {
    STATUS_TRY(lambda_impl(op, prm->eig_cg_steps, &lam));
    lam *= prm->cheb_safety;
    res->lambda_max = lam;
  }
  if (prm->precision != 0 && prm->precision != 1) return fail(MF_ERR_ARGUMENT, "precision must be 0 or 1");
  const bool mixed = prm->precision == 1 && prm->cheb_degree > 0;
  if (mixed) {
    if (op->world != 1 || op->g.dim != 3 || op->dg || op->hex)
      return fail(MF_ERR_ARGUMENT, "FP32 Chebyshev: 3D brick operator, one rank");
    if (!op->r_f) {
      CUDA_TRY(cudaMalloc(&op->r_f, n * sizeof(float)));
      CUDA_TRY(cudaMalloc(&op->z_f, n * sizeof(float)));
    }
  }
  auto precond = [&](const double *rr, double *zz, double *rz_dev) -> mf_status {
    if (mixed) {  // z = P(r) in FP32: round r, run the same Chebyshev recurrence, widen z
      CUDA_TRY(launch_d2f(rr, op->r_f, n, op->stream, &op->launches));
      STATUS_TRY(cheb_f32(op, op->r_f, op->z_f, lam, prm->cheb_degree, prm->cheb_range));
      CUDA_TRY(launch_f2d(op->z_f, zz, n, op->stream, &op->launches));
      return dot_dev(op, rr, zz, rz_dev);
    }
    if (prm->cheb_degree > 0) return cheb_impl(op, rr, zz, lam, prm->cheb_degree, prm->cheb_range, rz_dev);
    CUDA_TRY(launch_mul(op->dinv, rr, zz, n, op->stream, &op->launches));
    return dot_dev(op, rr, zz, rz_dev);
  };
  return cg_core(op, b, x, prm->rel_tol, prm->max_iter, precond, res, history, history_cap);
}

extern "C" mf_status mf_get_info(const mf_op *op, mf_info *info) {
  if (!op || !info) return fail(MF_ERR_ARGUMENT, "null argument");
  const Geo &g = op->g;
  info->dim = g.dim;
  info->degree = g.k;
  info->geometry = g.geom;
  info->coeff_kind = g.coeff_kind;
  info->apply_variant = chosen_variant(op);
  info->n_cells_local = ncells_local(g);
  info->kernel_launches = op->launches;
  const int64_t nq = ipow(g.k + 1, g.dim);
  if (op->hex) {  // src + dst, metric (6 doubles) and cell_dofs (int32) per cell node / point
    info->bytes_algorithmic = 16 * op->n_local + (8 * 6 + 4) * op->hx.ncells * nq;
    info->flops_algorithmic = (double)op->hx.ncells * (2.0 * 12.0 * std::pow(g.k + 1.0, 4) + 18.0 * nq);
    return MF_OK;
  }
  info->bytes_algorithmic =
      16 * op->n_local + (g.geom == MF_GEOM_SINE ? 8 * (int64_t)ncomp(g.dim) * ncells_local(g) * nq : 0);
  // 12-sweep (3D) / 8-sweep (2D) collocation kernel: 2 * (2 dim sweeps) * N^{dim+1} FMA + q-point op
  const double N = g.k + 1;
  const double sweeps = 4.0 * g.dim;
  const double qop = g.geom == MF_GEOM_SINE ? 2.0 * g.dim * g.dim : 2.0 * g.dim;
  info->flops_algorithmic =
      (double)ncells_local(g) * (2.0 * sweeps * std::pow(N, g.dim + 1) + qop * std::pow(N, g.dim));
  return MF_OK;
}
