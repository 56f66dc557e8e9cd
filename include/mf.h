/* mf.h -- C ABI of the B200-native matrix-free Laplace library (libmf_b200.so).
 *
 * The library evaluates v = A u for the finite-element discretisation of the
 * Laplacian of PAPER.md Eq. (1) (§2.4: a(u,v) = (grad u, grad v)_Omega,
 * with a constant or variable coefficient c(x)) without ever building a matrix
 * (§3.6: "a global sparse matrix is never built and linear systems
 * are only solved by the action of the underlying linear operator on a vector
 * via the integrals in the weak form"), by sum factorisation over the
 * tensor-product Q_k shape functions (§3.6) on a structured brick of
 * hexahedra (quadrilaterals in 2D), affine or curved (isoparametric degree k).
 * Around it sit the operator diagonal and a Chebyshev(6)-Jacobi preconditioned
 * CG (§6.1 "Chebyshev smoothing of degree 6").
 *
 * Discretisation: Gauss-Legendre quadrature with k+1
 * points per direction (R1); Gauss-Lobatto support points, x-fastest
 * lexicographic global numbering g = (gz*Ny + gy)*Nx + gx with N_e = k*n_e + 1
 * (R2); homogeneous Dirichlet rows/columns replaced by the identity, dst_g = src_g
 * (R3); curved geometry Phi(x) = x + eps (hi-lo) prod_d sin(pi (x_d-lo_d)/(hi_d-lo_d))
 * (R4); variable coefficient c(x) = 1/(0.05 + 2|x|^2) (R5).
 *
 * Conventions
 *  - Every vector is caller-owned, contiguous FP64.  mf_apply / mf_diagonal /
 *    mf_chebyshev take DEVICE pointers (e.g. torch.Tensor.data_ptr()) and are
 *    asynchronous on the op's stream; mf_apply_host takes HOST pointers and
 *    blocks.  The library never frees or retains caller pointers.
 *  - With world_size > 1 the brick is cut into z-slabs of whole cell layers;
 *    rank r holds the contiguous global range [first_global, first_global +
 *    n_local): its DoF planes plus a duplicate of the shared upper plane
 *    (owned, for dot products, by the upper rank; the first n_owned entries are
 *    this rank's owned DoFs).  Every call is then collective (same order and
 *    arguments on every rank, as in NCCL).  The blocking calls (mf_cg_solve,
 *    mf_estimate_lambda_max, mf_apply_host, mf_sync) poll ncclCommGetAsyncError
 *    while they wait; an NCCL error, or no progress for MF_NCCL_TIMEOUT_S seconds
 *    (environment, default 300), aborts the communicator (ncclCommAbort) and
 *    returns MF_ERR_NCCL -- the op is unusable afterwards (destroy it).
 *  - Errors: negative mf_status, message from mf_last_error() (thread-local).
 *    An op is not thread-safe.
 */
#ifndef MF_B200_H
#define MF_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MF_OK = 0,
  MF_ERR_ARGUMENT = -1,       /* bad descriptor: dim, degree 1..8, n_cells < 1, lower >= upper, NULL (S:148 BadDomain) */
  MF_ERR_LENGTH = -2,         /* vector length != n_local (S:566 LengthMismatch) */
  MF_ERR_SINGULAR = -3,       /* det J <= 0 at a quadrature point (S:332 SingularTensor) */
  MF_ERR_MAX_ITERATIONS = -4, /* CG did not converge within max_iter */
  MF_ERR_BREAKDOWN = -5,      /* p.Ap <= 0 or r.z <= 0 in CG / eigenvalue estimate */
  MF_ERR_CUDA = -6,
  MF_ERR_NCCL = -7,
  MF_ERR_OUT_OF_MEMORY = -8
} mf_status;

enum { MF_GEOM_CARTESIAN = 0, MF_GEOM_SINE = 1 };
enum { MF_COEFF_CONSTANT = 0, MF_COEFF_VARIABLE = 1 };

/* Structured brick [lower, upper] with n_cells[e] cells per direction e < dim. */
typedef struct {
  int32_t dim;              /* 2 or 3 */
  int64_t n_cells[3];       /* >= 1 for e < dim; ignored otherwise */
  double lower[3], upper[3];
  int32_t geometry;         /* MF_GEOM_CARTESIAN or MF_GEOM_SINE (R4, isoparametric degree k) */
  double deform_eps;        /* eps of R4 (0.1 in BASELINE cfg 4) */
  uint32_t dirichlet_faces; /* bit f for face f = x-,x+,y-,y+,z-,z+ (S:147); 0 = pure Neumann */
} mf_mesh;

typedef struct {
  int32_t kind;  /* MF_COEFF_CONSTANT (c = value) or MF_COEFF_VARIABLE (c(x) of R5) */
  double value;
} mf_coeff;

/* Multi-GPU placement; pass NULL to mf_create for one GPU on the current device.
 * world_size > 1 with nccl_unique_id == NULL builds a DETACHED slab operator: rank's z-slab
 * exactly as in a distributed run (partition, interior z faces unconstrained, the upper rank
 * writes the identity rows of a shared Dirichlet plane) but without a communicator.  mf_apply,
 * mf_apply_split_part, mf_apply_host and mf_diagonal then return this rank's partial sums on
 * the shared first / last plane; the caller adds the neighbour's (any transport).  Collective
 * calls (dots, solvers, mf_chebyshev, lambda) fail with MF_ERR_ARGUMENT. */
typedef struct {
  int32_t rank, world_size;
  const uint8_t *nccl_unique_id; /* 128 bytes from mf_nccl_unique_id() on rank 0; NULL if world_size == 1
                                    (or for a detached slab) */
  int32_t device;                /* CUDA device ordinal for this rank */
} mf_dist;

typedef struct mf_op mf_op; /* opaque, owned by the library */

/* Build the operator: 1D tables, geometry (metric precompute for MF_GEOM_SINE,
 * MF_ERR_SINGULAR if det J <= 0), Dirichlet plan, z-slab partition and NCCL
 * communicator.  Collective when world_size > 1. */
mf_status mf_create(const mf_mesh *mesh, int32_t degree, const mf_coeff *coeff,
                    const mf_dist *dist, mf_op **out);
void mf_destroy(mf_op *op);
const char *mf_last_error(void);

/* The symmetric interior penalty DG Laplacian on the same brick (
 * PAPER.md P:1360-1364 §6.1 "symmetric interior penalty discontinuous Galerkin"):
 * discontinuous Q_k Lagrange on the GLL nodes of each cell, DoF index = cell (k+1)^3 +
 * local (both x-fastest), Gauss(k+1) on cells and faces, penalty 2 (k+1)^2 / h_n,
 * weak (Nitsche) homogeneous Dirichlet on every face (R16-R18).  3D,
 * Cartesian geometry, constant coefficient, dirichlet_faces = all six, one rank
 * (else MF_ERR_ARGUMENT).  The returned op works with mf_apply, mf_diagonal,
 * mf_estimate_lambda_max, mf_chebyshev and mf_cg_solve (no constrained DoFs;
 * mf_get_info reports apply_variant 4). */
mf_status mf_create_dg(const mf_mesh *mesh, int32_t degree, const mf_coeff *coeff, mf_op **out);

/* General unstructured hexahedral mesh (§3.1
 * "unstructured ... hexahedral meshes", §3.5 hanging-node constraints applied
 * inside the matrix-free loop; R21, R22).  All arrays are HOST memory, read
 * during mf_create_hex only (copied to the device; the caller keeps ownership).
 *   vertices       [n_vertices][3] fp64 coordinates
 *   cell_vertices  [n_cells][8] int32: the cell's vertices in its own lexicographic frame
 *                  (local vertex a + 2b + 4c at reference corner (a,b,c)); the mapping is
 *                  trilinear (R21) and must have det J > 0 at every Gauss point
 *                  (else MF_ERR_SINGULAR)
 *   cell_dofs      [n_cells][(k+1)^3] int32, local GLL node i = i0 + (k+1)(i1 + (k+1) i2):
 *                  >= 0 the global DoF (< n_dofs); < 0 constraint line -1 - value (R22)
 *   line_ptr       [n_lines+1] int32 CSR offsets into line_dof / line_w; a constrained
 *                  (hanging) local node takes u = sum line_w[j] u[line_dof[j]] in the gather
 *                  and receives the transpose in the scatter (may be NULL if n_lines == 0)
 *   dirichlet_dofs [n_dirichlet] int32: identity rows / columns (R3); gather reads them as
 *                  zero, line entries on them drop out
 * mf_hex_number_dofs builds cell_dofs for a conforming mesh.  The returned op works with
 * mf_apply, mf_apply_host, mf_diagonal, mf_estimate_lambda_max, mf_chebyshev and
 * mf_cg_solve (one rank; mf_get_info reports apply_variant 5, n_local = n_dofs).
 * Errors: MF_ERR_ARGUMENT for null arrays, indices out of range, degree outside 1..8. */
typedef struct {
  int64_t n_vertices, n_cells, n_dofs, n_lines, n_dirichlet;
  const double *vertices;
  const int32_t *cell_vertices;
  const int32_t *cell_dofs;
  const int32_t *line_ptr;
  const int32_t *line_dof;
  const double *line_w;
  const int32_t *dirichlet_dofs;
} mf_hex_mesh;
mf_status mf_create_hex(const mf_hex_mesh *mesh, int32_t degree, const mf_coeff *coeff, mf_op **out);

/* DoF numbering of a conforming hex mesh (host only; the DoF handler step of
 * P:694-705): one DoF per vertex, k-1 per edge, (k-1)^2 per face, (k-1)^3 per cell
 * interior, numbered in order of first appearance cell by cell.  Edge and face DoFs
 * are laid out in a frame fixed by the GLOBAL vertex numbers (an edge runs from its
 * smaller to its larger vertex; a face's origin is its smallest vertex, its first axis
 * points to the smaller of the origin's two face neighbours), so cells that see a
 * shared edge or face in different orientations agree on its DoFs (R21).
 *   cell_vertices [n_cells][8] as for mf_hex_mesh; cell_dofs [n_cells][(k+1)^3] output;
 *   *n_dofs output.  is_boundary (optional, may be NULL) [capacity] uint8 output: 1 on the
 *   DoFs of faces that belong to one cell only; MF_ERR_LENGTH if n_dofs > capacity.
 * Errors: MF_ERR_ARGUMENT for a cell with repeated vertices or a face shared by more
 * than two cells (non-manifold / non-conforming input). */
mf_status mf_hex_number_dofs(int32_t degree, int64_t n_cells, const int32_t *cell_vertices, int32_t *cell_dofs,
                             int64_t *n_dofs, uint8_t *is_boundary, int64_t capacity);

/* NCCL unique id (128 bytes) for mf_dist, created on rank 0 and broadcast by the caller. */
mf_status mf_nccl_unique_id(uint8_t *out128);

/* The z-slab partition mf_create uses for (rank, world_size), computed on the
 * host without a GPU: rank r owns cell layers [cz0, cz1) =
 * [r nz / P, (r+1) nz / P); its local vector is the global slice
 * [first_global, first_global + n_local) = DoF planes k cz0 .. k cz1 inclusive;
 * the first n_owned entries are owned (the shared upper plane belongs to the
 * upper rank); plane = Nx Ny doubles is the size of one halo message.
 * MF_ERR_ARGUMENT for an invalid mesh/degree or nz < world_size. */
mf_status mf_partition(const mf_mesh *mesh, int32_t degree, int32_t rank, int32_t world_size,
                       int64_t *cz0, int64_t *cz1, int64_t *first_global, int64_t *n_local,
                       int64_t *n_owned, int64_t *plane);

/* Local / global sizes (see Conventions). */
mf_status mf_sizes(const mf_op *op, int64_t *n_local, int64_t *first_global,
                   int64_t *n_global, int64_t *n_owned);

/* cudaStream_t on which every asynchronous call is enqueued (default: the
 * legacy default stream of the op's device). */
mf_status mf_set_stream(mf_op *op, void *cuda_stream);

/* dst = A src (§8(a) a3-a8: gather, sum factorisation to the Gauss points,
 * quadrature-point operation, transposed sweeps, scatter-add, Dirichlet
 * identity, halo exchange for world_size > 1).  src and dst are distinct
 * device buffers of n_local doubles; dst is overwritten.  Asynchronous. */
mf_status mf_apply(mf_op *op, const double *src, int64_t n_src, double *dst, int64_t n_dst);

/* The same with HOST buffers: H2D copy of src, apply, D2H copy of dst; blocks. */
mf_status mf_apply_host(mf_op *op, const double *src_host, int64_t n_src, double *dst_host,
                        int64_t n_dst);

/* The same operator evaluated in FP32 (device buffers of n_local floats): the FP32
 * instances of the apply kernels used by the mixed-precision multigrid (SURVEY
 * §8(f) f2).  3D, world_size 1 only (else MF_ERR_ARGUMENT).
 * Asynchronous. */
mf_status mf_apply_f32(mf_op *op, const float *src, int64_t n_src, float *dst, int64_t n_dst);

/* Testing hook for the overlapped multi-GPU apply (§8(e)): runs
 * ONE part of its launch sequence on one GPU, without the exchange -- part 1 = the
 * cell layers next to the shared z-planes (and, for kernels that need it, the
 * initialisation of dst), part 2 = the interior layers, which never write the
 * shared planes (first and last plane of the local vector) and never read dst.
 * Part 1 followed by part 2 is mf_apply on one rank.  3D brick operators only
 * (MF_ERR_ARGUMENT otherwise, or part not 1 / 2).  Asynchronous. */
mf_status mf_apply_split_part(mf_op *op, const double *src, int64_t n_src, double *dst, int64_t n_dst,
                              int32_t part);

/* Waits for the op's stream (and, with world_size > 1, watches the communicator as
 * described above).  MF_ERR_NCCL after an abort. */
mf_status mf_sync(mf_op *op);

/* diag = diagonal of A (§8(a) a9), 1 on constrained DoFs.  Asynchronous. */
mf_status mf_diagonal(mf_op *op, double *diag, int64_t n);

/* Largest Ritz value of D^{-1}A from `steps` Jacobi-PCG steps started from the
 * splitmix64 vector of the global DoF index (seed 0, zero on constrained DoFs),
 * without the safety factor (R8).  Blocks. */
mf_status mf_estimate_lambda_max(mf_op *op, int32_t steps, double *lambda_out);

/* z = Chebyshev(degree) approximation of A^{-1} r for D^{-1}A on
 * [lambda/smoothing_range, lambda], started from zero (R6, R7).
 * Device buffers of n_local doubles.  Asynchronous. */
mf_status mf_chebyshev(mf_op *op, const double *r, double *z, int64_t n, double lambda,
                       int32_t degree, double smoothing_range);

typedef struct {
  double rel_tol;        /* stop when ||r||_2 <= rel_tol ||b||_2 (recursive residual, R9) */
  int32_t max_iter;      /* applications of A, e.g. 10000 */
  int32_t cheb_degree;   /* 6; 0 selects plain Jacobi-PCG */
  double cheb_range;     /* 20 */
  double cheb_safety;    /* 1.2 */
  int32_t eig_cg_steps;  /* 12 */
  int32_t precision;     /* 0: FP64 Chebyshev; 1: the Chebyshev preconditioner in FP32 inside the FP64 CG
                            (§8(f) f2; 3D brick, one rank, else MF_ERR_ARGUMENT) */
} mf_cg_params;

typedef struct {
  int32_t iterations;        /* applications of A in the CG loop (not counting the eigenvalue estimate / preconditioner) */
  double final_rel_residual; /* ||r_N|| / ||b|| */
  double lambda_max;         /* safety * Ritz estimate used by the Chebyshev preconditioner */
} mf_cg_result;

/* Solve A x = b from x0 = 0 with Chebyshev(cheb_degree)-Jacobi PCG (§8(a) a10,
 * S:500-508).  b, x: device buffers of n_local doubles.  Optional residual
 * history: if history != NULL it receives ||r_j|| after each apply (up to
 * history_cap entries).  Blocks (the host reads 2-3 scalars per iteration). */
mf_status mf_cg_solve(mf_op *op, const double *b, double *x, int64_t n, const mf_cg_params *params,
                      mf_cg_result *result, double *history, int32_t history_cap);

/* Introspection for tests and the benchmark. */
typedef struct {
  int32_t dim, degree, geometry, coeff_kind;
  int32_t apply_variant;      /* kernel family chosen for mf_apply */
  int64_t n_cells_local;
  int64_t kernel_launches;    /* cumulative count of this library's kernel launches on this op */
  int64_t bytes_algorithmic;  /* algorithmic HBM bytes of one apply: 16 B/DoF + stored geometry */
  double flops_algorithmic;   /* FP64 flops of one apply for the chosen variant */
} mf_info;
mf_status mf_get_info(const mf_op *op, mf_info *info);

/* Force a kernel family for mf_apply (0 = automatic).  Unknown or unsupported
 * choices return MF_ERR_ARGUMENT. */
mf_status mf_set_apply_variant(mf_op *op, int32_t variant);

/* Live timing of the dominant cell kernel of mf_apply with CUDA events recorded
 * on the op's stream around each launch (enable != 0 starts a new window).
 * mf_kernel_timing synchronises those events and returns the summed
 * milliseconds and the number of timed launches since the window started. */
mf_status mf_set_kernel_timing(mf_op *op, int32_t enable);
mf_status mf_kernel_timing(mf_op *op, double *ms_total, int64_t *count);

/* ---- Geometric multigrid (§6.1;
 * SPEC S:602-695) ------------------------------------------------------------
 * A hierarchy of globally refined bricks: level L-1 is `finest`, level l has
 * finest.n_cells / 2^(L-1-l) cells per direction, the same degree, geometry,
 * coefficient and Dirichlet faces on every level.  Level operators are mf_op's.
 * Transfer: prolongation = interpolation of the coarse Q_k function at the fine
 * GLL support points (tensor product of 1D interpolations), restriction = its
 * exact transpose; constrained DoFs are 0 on every level.  Smoother: the
 * Chebyshev(degree) polynomial of mf_chebyshev on [lam_l/range, lam_l],
 * lam_l = safety * Ritz(eig_steps) of the level (pre: x = Cheb(b); post:
 * x += Cheb(b - A x)).  Coarse solver: the dense inverse of level 0 (built once on
 * the GPU by Gauss-Jordan elimination), so one V-cycle is a fixed symmetric linear
 * operator.  Single GPU (world_size 1).  Ownership: the hierarchy owns its level
 * ops and scratch vectors; every vector argument is a caller-owned device buffer
 * of the stated level's n_local doubles. */
typedef struct mf_mg mf_mg; /* opaque */
typedef struct {
  int32_t n_levels;        /* 0: halve while every direction is even and the coarser level has > max_coarse_dofs DoFs */
  int64_t max_coarse_dofs; /* e.g. 1000; MF_ERR_ARGUMENT if the coarse level would exceed 2048 DoFs */
  int32_t smooth_degree;   /* Chebyshev degree of pre- and post-smoothing, 6 */
  double smooth_range;     /* 20 */
  double smooth_safety;    /* 1.2 */
  int32_t eig_cg_steps;    /* 12 */
  int32_t precision;       /* 0: FP64 V-cycle; 1: FP32 V-cycle (level operators, smoothers, transfers and
                              coarse solve in single precision) inside the FP64 CG -- the paper's production
                              setting, "run in single precision ... with some double-precision
                              correction" */
} mf_mg_params;
/* Errors: MF_ERR_ARGUMENT (n_cells not divisible by 2^(levels-1), bad parameters),
 * plus every error of mf_create. */
mf_status mf_mg_create(const mf_mesh *finest, int32_t degree, const mf_coeff *coeff, const mf_mg_params *params,
                       mf_mg **out);
void mf_mg_destroy(mf_mg *mg);
/* number of levels; n_local of level l (0 = coarsest); the level's operator
 * (borrowed, valid until mf_mg_destroy); lambda_l (with the safety factor) */
mf_status mf_mg_levels(const mf_mg *mg, int32_t *n_levels);
mf_status mf_mg_level_size(const mf_mg *mg, int32_t level, int64_t *n_local);
mf_status mf_mg_level_op(mf_mg *mg, int32_t level, mf_op **op);
mf_status mf_mg_level_lambda(const mf_mg *mg, int32_t level, double *lambda);
/* fine(level) = P coarse(level - 1); coarse(level - 1) = P^T fine(level); 1 <= level < L.  Asynchronous. */
mf_status mf_mg_prolongate(mf_mg *mg, int32_t level, const double *coarse, double *fine);
mf_status mf_mg_restrict(mf_mg *mg, int32_t level, const double *fine, double *coarse);
/* x = V(b): one V-cycle on the finest level, from x = 0.  Asynchronous, no host syncs. */
mf_status mf_mg_vcycle(mf_mg *mg, const double *b, double *x, int64_t n);
/* CG on the finest level with one V-cycle as preconditioner; same
 * stopping rule, history and errors as mf_cg_solve (result->lambda_max = lambda of
 * the finest level).  Blocks. */
mf_status mf_mg_cg_solve(mf_mg *mg, const double *b, double *x, int64_t n, double rel_tol, int32_t max_iter,
                         mf_cg_result *result, double *history, int32_t history_cap);
mf_status mf_mg_set_stream(mf_mg *mg, void *cuda_stream);

/* ---- Hanging nodes (restricted to one 2:1 interface; PAPER.md
 * P:776-781 §3.5 "hanging node constraints"): the box [lower, upper] cut at
 * z = z_mid into a coarse lower brick of n_cells_coarse cells and an upper brick
 * refined once more (2 nx, 2 ny, nz_fine cells), Q_k on both, constant coefficient,
 * Dirichlet (identity rows) on every outer face.  The fine interface nodes hang:
 * u_f = (P_y (x) P_x) u_c on the interface (coarse face function interpolated at the
 * fine nodes), applied in the gather and transposed in the scatter of the matrix-free
 * apply.  Global vector (R20): every coarse-grid node (x-fastest, plane by
 * plane), then the fine grid's nodes above the interface plane; n = nC + nF - one
 * fine plane.  Device buffers of n doubles; asynchronous on the stream; single GPU. */
typedef struct mf_hng mf_hng;
mf_status mf_hng_create(const double *lower3, const double *upper3, double z_mid, const int64_t *n_cells_coarse3,
                        int64_t nz_fine, int32_t degree, const mf_coeff *coeff, mf_hng **out);
void mf_hng_destroy(mf_hng *h);
mf_status mf_hng_sizes(const mf_hng *h, int64_t *n, int64_t *n_coarse);
mf_status mf_hng_apply(mf_hng *h, const double *src, int64_t n_src, double *dst, int64_t n_dst);
mf_status mf_hng_set_stream(mf_hng *h, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* MF_B200_H */
