/* oracle.h -- the plain CPU oracle for the matrix-free Laplace hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path in
 * paper_1910_13247_b200/ (see DESIGN.md "Oracle independence").
 *
 * What it computes is the plain definition of the operator of PAPER.md
 * Eq. (1) (§2.4, a(u,v) = (grad u, grad v)_Omega) discretised with
 * continuous Q_k Lagrange elements on Gauss-Lobatto support points (P:802-813
 * §3.4) and assembled with the step-4 loop of P:341-348 §2.4:
 *     A_c(i,j) = sum_q c(x_q) grad phi_i(x_q) . grad phi_j(x_q) JxW(q),
 * scattered to a global CSR matrix, then y = A x by sparse matrix-vector
 * product.  No sum factorisation, no blocking, no fusion.
 *
 * Readings of the paper (DESIGN.md "Readings" R1-R15):
 *   R1 Gauss-Legendre quadrature with k+1 points per direction;
 *   R2 GLL support points, x-fastest lexicographic numbering;
 *   R3 Dirichlet rows/cols zeroed with a unit diagonal (identity);
 *   R4 curved geometry Phi(x) = x + eps*(hi-lo)*prod_d sin(pi xt_d), isoparametric;
 *   R5 variable coefficient c(x) = 1/(0.05 + 2|x|^2) at the mapped x_q.
 * Parity status per function: see oracle/README.md and DESIGN.md.
 */
#ifndef MF_ORACLE_H
#define MF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The oracle's own description of a problem (independent of include/mf.h). */
typedef struct {
  int32_t dim;          /* 1, 2 or 3 */
  int64_t nc[3];        /* cells per direction */
  double lo[3], hi[3];  /* brick [lo, hi] */
  int32_t degree;       /* k >= 1 */
  int32_t geom;         /* 0 = affine brick, 1 = sine-deformed (R4) */
  double eps;           /* deformation amplitude for geom = 1 */
  int32_t coeff_kind;   /* 0 = constant coeff_value, 1 = c(x) of R5 */
  double coeff_value;
  uint32_t dirichlet;   /* bit f for face f = x-,x+,y-,y+,z-,z+  */
} or_problem;

/* 1D rules on [0,1] (O1). Return 0 on success. */
int or_gauss(int n, double *x, double *w);
int or_gll(int k, double *x);
/* Lagrange basis on `nodes` (O2): value and derivative of l_i at x. */
double or_lagrange(const double *nodes, int n, int i, double x);
double or_lagrange_d(const double *nodes, int n, int i, double x);

/* Sizes (O3). */
int64_t or_n_dofs(const or_problem *p);
int64_t or_n_cells(const or_problem *p);
/* 1 if global DoF g sits on a Dirichlet face. */
int or_is_constrained(const or_problem *p, int64_t g);
/* global DoF indices of the (k+1)^dim local nodes of cell `cell` (lexicographic) */
int or_cell_dofs(const or_problem *p, int64_t cell, int64_t *dofs);
/* Phi applied to a point of the brick (R4). */
void or_phi(const or_problem *p, const double *x, double *out);

/* Element matrices (O4-O5): A (stiffness with coefficient) and/or M (mass),
 * each (k+1)^dim squared, row-major, with nq Gauss points per direction.
 * Returns 0, or -3 if det J <= 0 at a quadrature point. */
int or_cell_matrix(const or_problem *p, int64_t cell, int nq, double *A, double *M);

/* Global CSR (O6). which = 0 stiffness, 1 mass. apply_dirichlet = 1 applies R3.
 * nnz from or_csr_nnz; rowptr has n+1 entries. */
int64_t or_csr_nnz(const or_problem *p);
int or_assemble_csr(const or_problem *p, int which, int apply_dirichlet,
                    int64_t *rowptr, int32_t *col, double *val);
void or_spmv(int64_t n, const int64_t *rowptr, const int32_t *col,
             const double *val, const double *x, double *y);
void or_csr_diagonal(int64_t n, const int64_t *rowptr, const int32_t *col,
                     const double *val, double *diag);

/* (A x)_g for selected rows only, by element-matrix rows of the cells that
 * contain g (same definition, no global matrix).  Dirichlet convention R3. */
int or_apply_rows(const or_problem *p, const int64_t *rows, int64_t m,
                  const double *x, double *out);

/* RHS (O8): f_kind 0 -> f = 1; 1 -> f = dim pi^2 prod sin(pi x_e).
 * nq Gauss points per direction (R14: k+1).  Dirichlet entries are 0. */
int or_rhs(const or_problem *p, int f_kind, int nq, double *b);
/* L2 error of the FE function u against prod sin(pi x_e) with nq points (R14: k+3). */
double or_l2_error(const or_problem *p, const double *u, int nq);

/* Kronecker-sum oracle (O12), affine bricks with constant coefficient only:
 * A = c (K_x (x) M_y (x) M_z + M_x (x) K_y (x) M_z + M_x (x) M_y (x) K_z)
 * with 1D matrices assembled by or_assemble_csr on 1D meshes; R3 for Dirichlet. */
int or_kron_apply(const or_problem *p, const double *x, double *y);

int or_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
