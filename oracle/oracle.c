/* oracle.c -- plain CPU oracle (C11 + OpenMP, fp64).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with the
 * CUDA path.  Every routine below is the textbook definition written out; the
 * citations name the passage each one follows (P: = PAPER.md, S: = SPEC.md
 * line numbers; readings R1-R15 are listed in DESIGN.md).
 *
 * Parity pins for each routine live in tests/test_oracle_*.py (closed forms,
 * exact polynomial integration, invariants, brute force).  The variable-
 * coefficient operator on the deformed mesh has no closed form; it is pinned
 * by the Neumann kernel, symmetry, or_assemble_csr = or_apply_rows, and the
 * energy of the physical linears (u_a^T A u_b = delta_ab int c dx against a
 * mesh-free quadrature of int c; tests/test_oracle_operator.py).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* O1: 1D rules on [0,1] (R1: Gauss-Legendre, k+1 points; R2: Gauss-Lobatto   */
/* support points).  Newton iteration on the Legendre polynomial P_n (Gauss)  */
/* and on P_k' (interior Lobatto nodes), three-term recurrence for P_j.       */
/* ------------------------------------------------------------------------- */
static void legendre(int n, double t, double *p, double *pm1) {
  /* P_n(t) and P_{n-1}(t) by (j+1) P_{j+1} = (2j+1) t P_j - j P_{j-1} */
  double a = 1.0, b = t; /* P_0, P_1 */
  if (n == 0) { *p = 1.0; *pm1 = 0.0; return; }
  for (int j = 1; j < n; ++j) {
    double c = ((2.0 * j + 1.0) * t * b - j * a) / (j + 1.0);
    a = b;
    b = c;
  }
  *p = b;
  *pm1 = a;
}

int or_gauss(int n, double *x, double *w) {
  if (n < 1) return -1;
  for (int i = 0; i < n; ++i) {
    double t = cos(OR_PI * (i + 0.75) / (n + 0.5));
    double p, pm1, dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      legendre(n, t, &p, &pm1);
      dp = n * (t * p - pm1) / (t * t - 1.0); /* P_n'(t) */
      double dt = p / dp;
      t -= dt;
      if (fabs(dt) < 1e-17) break;
    }
    legendre(n, t, &p, &pm1);
    dp = n * (t * p - pm1) / (t * t - 1.0);
    /* map t in [-1,1] (descending in i) to x in [0,1] (ascending) */
    x[i] = 0.5 * (1.0 - t);
    w[i] = 0.5 * 2.0 / ((1.0 - t * t) * dp * dp);
  }
  return 0;
}

int or_gll(int k, double *x) {
  if (k < 1) return -1;
  x[0] = 0.0;
  x[k] = 1.0;
  for (int j = 1; j < k; ++j) {
    double t = cos(OR_PI * j / k);
    for (int it = 0; it < 100; ++it) {
      double p, pm1;
      legendre(k, t, &p, &pm1);
      double dp = k * (t * p - pm1) / (t * t - 1.0);          /* P_k'  */
      double ddp = (2.0 * t * dp - k * (k + 1.0) * p) / (1.0 - t * t); /* P_k'' (Legendre ODE) */
      double dt = dp / ddp;
      t -= dt;
      if (fabs(dt) < 1e-17) break;
    }
    x[j] = 0.5 * (1.0 - t);
  }
  return 0;
}

/* O2: Lagrange polynomials by the product formula. */
double or_lagrange(const double *nodes, int n, int i, double x) {
  double v = 1.0;
  for (int j = 0; j < n; ++j)
    if (j != i) v *= (x - nodes[j]) / (nodes[i] - nodes[j]);
  return v;
}

double or_lagrange_d(const double *nodes, int n, int i, double x) {
  double s = 0.0;
  for (int m = 0; m < n; ++m) {
    if (m == i) continue;
    double v = 1.0 / (nodes[i] - nodes[m]);
    for (int j = 0; j < n; ++j)
      if (j != i && j != m) v *= (x - nodes[j]) / (nodes[i] - nodes[j]);
    s += v;
  }
  return s;
}

/* ------------------------------------------------------------------------- */
/* O3: structured brick, x-fastest lexicographic numbering.                   */
/* ------------------------------------------------------------------------- */
static int64_t n1d(const or_problem *p, int e) {
  return e < p->dim ? (int64_t)p->degree * p->nc[e] + 1 : 1;
}
static int64_t nc1d(const or_problem *p, int e) { return e < p->dim ? p->nc[e] : 1; }

int64_t or_n_dofs(const or_problem *p) { return n1d(p, 0) * n1d(p, 1) * n1d(p, 2); }
int64_t or_n_cells(const or_problem *p) { return nc1d(p, 0) * nc1d(p, 1) * nc1d(p, 2); }

int or_is_constrained(const or_problem *p, int64_t g) {
  int64_t N[3] = {n1d(p, 0), n1d(p, 1), n1d(p, 2)};
  int64_t m[3];
  m[0] = g % N[0];
  m[1] = (g / N[0]) % N[1];
  m[2] = g / (N[0] * N[1]);
  for (int e = 0; e < p->dim; ++e) {
    if ((p->dirichlet >> (2 * e)) & 1u && m[e] == 0) return 1;
    if ((p->dirichlet >> (2 * e + 1)) & 1u && m[e] == N[e] - 1) return 1;
  }
  return 0;
}

static void cell_coords(const or_problem *p, int64_t cell, int64_t c[3]) {
  c[0] = cell % nc1d(p, 0);
  c[1] = (cell / nc1d(p, 0)) % nc1d(p, 1);
  c[2] = cell / (nc1d(p, 0) * nc1d(p, 1));
}

static int pow_int(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

int or_cell_dofs(const or_problem *p, int64_t cell, int64_t *dofs) {
  int k = p->degree, n = k + 1, nv = pow_int(n, p->dim);
  int64_t c[3];
  cell_coords(p, cell, c);
  int64_t Nx = n1d(p, 0), Ny = n1d(p, 1);
  for (int i = 0; i < nv; ++i) {
    int l[3] = {i % n, p->dim > 1 ? (i / n) % n : 0, p->dim > 2 ? i / (n * n) : 0};
    int64_t gx = k * c[0] + l[0], gy = k * c[1] + l[1], gz = k * c[2] + l[2];
    dofs[i] = (gz * Ny + gy) * Nx + gx;
  }
  return nv;
}

/* R4: Phi(x) = x + eps (hi - lo) prod_d sin(pi xt_d), xt = (x - lo)/(hi - lo). */
void or_phi(const or_problem *p, const double *x, double *out) {
  double s = 1.0;
  for (int d = 0; d < p->dim; ++d) s *= sin(OR_PI * (x[d] - p->lo[d]) / (p->hi[d] - p->lo[d]));
  for (int d = 0; d < p->dim; ++d)
    out[d] = x[d] + (p->geom == 1 ? p->eps * (p->hi[d] - p->lo[d]) * s : 0.0);
}

/* R5 */
static double coeff(const or_problem *p, const double *x) {
  if (p->coeff_kind == 0) return p->coeff_value;
  double r2 = 0.0;
  for (int d = 0; d < p->dim; ++d) r2 += x[d] * x[d];
  return 1.0 / (0.05 + 2.0 * r2);
}

/* ------------------------------------------------------------------------- */
/* O4: FEValues-like evaluation on one cell at a tensor Gauss rule of nq      */
/* points per direction: shape values, physical gradients J^{-T} grad phi_i,  */
/* JxW and mapped points.  Isoparametric mapping of degree k through the      */
/* support points Phi(GLL) (§3.4).  Brute-force sums over    */
/* all (k+1)^dim support points -- no sum factorisation.                      */
/* ------------------------------------------------------------------------- */
typedef struct {
  int dim, n, nv, nq, nqv;
  double *phi;  /* [nqv][nv] */
  double *grad; /* [nqv][nv][dim] physical gradients */
  double *jxw;  /* [nqv] */
  double *xq;   /* [nqv][dim] */
} cell_eval_t;

static void cell_eval_free(cell_eval_t *ce) {
  free(ce->phi);
  free(ce->grad);
  free(ce->jxw);
  free(ce->xq);
}

static int cell_eval(const or_problem *p, int64_t cell, int nq, cell_eval_t *ce) {
  const int dim = p->dim, k = p->degree, n = k + 1;
  const int nv = pow_int(n, dim), nqv = pow_int(nq, dim);
  ce->dim = dim; ce->n = n; ce->nv = nv; ce->nq = nq; ce->nqv = nqv;
  ce->phi = (double *)malloc(sizeof(double) * nqv * nv);
  ce->grad = (double *)malloc(sizeof(double) * nqv * nv * dim);
  ce->jxw = (double *)malloc(sizeof(double) * nqv);
  ce->xq = (double *)malloc(sizeof(double) * nqv * dim);
  double gll[16], gx[32], gw[32];
  or_gll(k, gll);
  or_gauss(nq, gx, gw);
  double L[32][16], Ld[32][16]; /* 1D basis values / derivatives at Gauss points */
  for (int q = 0; q < nq; ++q)
    for (int i = 0; i < n; ++i) {
      L[q][i] = or_lagrange(gll, n, i, gx[q]);
      Ld[q][i] = or_lagrange_d(gll, n, i, gx[q]);
    }
  /* support points x_j = Phi(lo + h (c + xhat_j)) */
  int64_t c[3];
  cell_coords(p, cell, c);
  double *X = (double *)malloc(sizeof(double) * nv * dim);
  for (int j = 0; j < nv; ++j) {
    double xb[3];
    int jj = j;
    for (int d = 0; d < dim; ++d) {
      int l = jj % n;
      jj /= n;
      double h = (p->hi[d] - p->lo[d]) / (double)p->nc[d];
      xb[d] = p->lo[d] + h * ((double)c[d] + gll[l]);
    }
    or_phi(p, xb, X + j * dim);
  }
  double *rg = (double *)malloc(sizeof(double) * nv * dim); /* reference gradients */
  int status = 0;
  for (int q = 0; q < nqv; ++q) {
    int qd[3] = {0, 0, 0}, qq = q;
    double W = 1.0;
    for (int d = 0; d < dim; ++d) { qd[d] = qq % nq; qq /= nq; W *= gw[qd[d]]; }
    for (int j = 0; j < nv; ++j) {
      int jd[3] = {0, 0, 0}, jj = j;
      for (int d = 0; d < dim; ++d) { jd[d] = jj % n; jj /= n; }
      double v = 1.0;
      for (int d = 0; d < dim; ++d) v *= L[qd[d]][jd[d]];
      ce->phi[q * nv + j] = v;
      for (int b = 0; b < dim; ++b) {
        double g = 1.0;
        for (int d = 0; d < dim; ++d) g *= (d == b) ? Ld[qd[d]][jd[d]] : L[qd[d]][jd[d]];
        rg[j * dim + b] = g;
      }
    }
    double J[3][3] = {{0}}, x[3] = {0, 0, 0};
    for (int j = 0; j < nv; ++j)
      for (int a = 0; a < dim; ++a) {
        x[a] += X[j * dim + a] * ce->phi[q * nv + j];
        for (int b = 0; b < dim; ++b) J[a][b] += X[j * dim + a] * rg[j * dim + b];
      }
    double det, Ji[3][3];
    if (dim == 1) {
      det = J[0][0];
      Ji[0][0] = 1.0 / J[0][0];
    } else if (dim == 2) {
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      Ji[0][0] = J[1][1] / det; Ji[0][1] = -J[0][1] / det;
      Ji[1][0] = -J[1][0] / det; Ji[1][1] = J[0][0] / det;
    } else {
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
            J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    }
    if (!(det > 0.0)) status = -3; /* SingularTensor */
    ce->jxw[q] = det * W;
    for (int a = 0; a < dim; ++a) ce->xq[q * dim + a] = x[a];
    /* grad phi_j = J^{-T} grad-hat phi_j */
    for (int j = 0; j < nv; ++j)
      for (int a = 0; a < dim; ++a) {
        double s = 0.0;
        for (int b = 0; b < dim; ++b) s += Ji[b][a] * rg[j * dim + b];
        ce->grad[(q * nv + j) * dim + a] = s;
      }
  }
  free(X);
  free(rg);
  return status;
}

/* O5: A_c(i,j) = sum_q c(x_q) grad phi_i . grad phi_j JxW (§2.4). */
int or_cell_matrix(const or_problem *p, int64_t cell, int nq, double *A, double *M) {
  cell_eval_t ce;
  int st = cell_eval(p, cell, nq, &ce);
  const int nv = ce.nv, dim = ce.dim;
  if (A) memset(A, 0, sizeof(double) * nv * nv);
  if (M) memset(M, 0, sizeof(double) * nv * nv);
  for (int q = 0; q < ce.nqv; ++q) {
    double cj = coeff(p, ce.xq + q * dim) * ce.jxw[q];
    for (int i = 0; i < nv; ++i)
      for (int j = 0; j < nv; ++j) {
        if (A) {
          double s = 0.0;
          for (int a = 0; a < dim; ++a)
            s += ce.grad[(q * nv + i) * dim + a] * ce.grad[(q * nv + j) * dim + a];
          A[i * nv + j] += s * cj;
        }
        if (M) M[i * nv + j] += ce.phi[q * nv + i] * ce.phi[q * nv + j] * ce.jxw[q];
      }
  }
  cell_eval_free(&ce);
  return st;
}

/* ------------------------------------------------------------------------- */
/* O6: global CSR.  Row g couples with every DoF of every cell containing g:  */
/* per direction the node range [m-k, m+k] for a vertex node (m % k == 0) or  */
/* [k floor(m/k), k floor(m/k) + k] otherwise, clipped to the brick; the row  */
/* is the tensor product of the three ranges, sorted by global index.         */
/* ------------------------------------------------------------------------- */
static void range1d(const or_problem *p, int e, int64_t m, int64_t *a, int64_t *b) {
  int64_t k = p->degree, N = n1d(p, e);
  if (e >= p->dim) { *a = 0; *b = 0; return; }
  if (m % k == 0) {
    *a = m - k < 0 ? 0 : m - k;
    *b = m + k > N - 1 ? N - 1 : m + k;
  } else {
    *a = k * (m / k);
    *b = *a + k;
  }
}

int64_t or_csr_nnz(const or_problem *p) {
  int64_t nnz = 1;
  for (int e = 0; e < 3; ++e) {
    int64_t s = 0;
    for (int64_t m = 0; m < n1d(p, e); ++m) {
      int64_t a, b;
      range1d(p, e, m, &a, &b);
      s += b - a + 1;
    }
    nnz *= s;
  }
  return nnz;
}

static void decode(const or_problem *p, int64_t g, int64_t m[3]) {
  int64_t Nx = n1d(p, 0), Ny = n1d(p, 1);
  m[0] = g % Nx;
  m[1] = (g / Nx) % Ny;
  m[2] = g / (Nx * Ny);
}

/* position of column (jx,jy,jz) within row g */
static int64_t csr_pos(const or_problem *p, const int64_t *rowptr, int64_t g, const int64_t mj[3]) {
  int64_t mi[3], a[3], b[3];
  decode(p, g, mi);
  for (int e = 0; e < 3; ++e) range1d(p, e, mi[e], &a[e], &b[e]);
  int64_t Lx = b[0] - a[0] + 1, Ly = b[1] - a[1] + 1;
  return rowptr[g] + ((mj[2] - a[2]) * Ly + (mj[1] - a[1])) * Lx + (mj[0] - a[0]);
}

int or_assemble_csr(const or_problem *p, int which, int apply_dirichlet,
                    int64_t *rowptr, int32_t *col, double *val) {
  const int64_t n = or_n_dofs(p), Nx = n1d(p, 0), Ny = n1d(p, 1);
  /* structure */
  rowptr[0] = 0;
  for (int64_t g = 0; g < n; ++g) {
    int64_t m[3], a[3], b[3];
    decode(p, g, m);
    int64_t len = 1;
    for (int e = 0; e < 3; ++e) { range1d(p, e, m[e], &a[e], &b[e]); len *= b[e] - a[e] + 1; }
    rowptr[g + 1] = rowptr[g] + len;
  }
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < n; ++g) {
    int64_t m[3], a[3], b[3];
    decode(p, g, m);
    for (int e = 0; e < 3; ++e) range1d(p, e, m[e], &a[e], &b[e]);
    int64_t pos = rowptr[g];
    for (int64_t z = a[2]; z <= b[2]; ++z)
      for (int64_t y = a[1]; y <= b[1]; ++y)
        for (int64_t x = a[0]; x <= b[0]; ++x) {
          col[pos] = (int32_t)((z * Ny + y) * Nx + x);
          val[pos] = 0.0;
          ++pos;
        }
  }
  /* step-4 loop over cells; cells of equal coordinate parity share no DoF,
   * so each of the 2^dim colours is scattered in parallel. */
  const int nv = pow_int(p->degree + 1, p->dim), nq = p->degree + 1;
  const int64_t ncell = or_n_cells(p);
  int status = 0;
  for (int color = 0; color < (1 << p->dim); ++color) {
#pragma omp parallel
    {
      double *Ae = (double *)malloc(sizeof(double) * nv * nv);
      int64_t *dofs = (int64_t *)malloc(sizeof(int64_t) * nv);
#pragma omp for schedule(dynamic, 4)
      for (int64_t cell = 0; cell < ncell; ++cell) {
        int64_t c[3];
        cell_coords(p, cell, c);
        int cc = (int)((c[0] & 1) | ((c[1] & 1) << 1) | ((c[2] & 1) << 2));
        if (cc != color) continue;
        int st = which == 0 ? or_cell_matrix(p, cell, nq, Ae, NULL)
                            : or_cell_matrix(p, cell, nq, NULL, Ae);
        if (st) {
#pragma omp atomic write
          status = st;
        }
        or_cell_dofs(p, cell, dofs);
        for (int i = 0; i < nv; ++i)
          for (int j = 0; j < nv; ++j) {
            int64_t mj[3];
            decode(p, dofs[j], mj);
            val[csr_pos(p, rowptr, dofs[i], mj)] += Ae[i * nv + j];
          }
      }
      free(Ae);
      free(dofs);
    }
  }
  if (apply_dirichlet) { /* R3: constrained rows and columns zero, unit diagonal */
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < n; ++g) {
      int rc = or_is_constrained(p, g);
      for (int64_t q = rowptr[g]; q < rowptr[g + 1]; ++q) {
        int cc = or_is_constrained(p, col[q]);
        if (rc || cc) val[q] = (col[q] == g) ? 1.0 : 0.0;
      }
    }
  }
  return status;
}

void or_spmv(int64_t n, const int64_t *rowptr, const int32_t *col,
             const double *val, const double *x, double *y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q) s += val[q] * x[col[q]];
    y[i] = s;
  }
}

void or_csr_diagonal(int64_t n, const int64_t *rowptr, const int32_t *col,
                     const double *val, double *diag) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    diag[i] = 0.0;
    for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q)
      if (col[q] == i) diag[i] = val[q];
  }
}

/* (A x)_g by element-matrix rows (same definition as O5/O6, R3). */
int or_apply_rows(const or_problem *p, const int64_t *rows, int64_t mrows,
                  const double *x, double *out) {
  const int k = p->degree, n = k + 1, nv = pow_int(n, p->dim), dim = p->dim;
  int status = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < mrows; ++r) {
    int64_t g = rows[r];
    if (or_is_constrained(p, g)) { out[r] = x[g]; continue; }
    int64_t m[3];
    decode(p, g, m);
    /* cells containing g: per direction c in {m/k - 1, m/k} (vertex) or {m/k} */
    int64_t clo[3] = {0, 0, 0}, chi[3] = {0, 0, 0};
    for (int e = 0; e < dim; ++e) {
      int64_t cm = m[e] / k;
      clo[e] = (m[e] % k == 0) ? cm - 1 : cm;
      chi[e] = cm;
      if (clo[e] < 0) clo[e] = 0;
      if (chi[e] > p->nc[e] - 1) chi[e] = p->nc[e] - 1;
    }
    double s = 0.0;
    int64_t dofs[729];
    for (int64_t cz = clo[2]; cz <= chi[2]; ++cz)
      for (int64_t cy = clo[1]; cy <= chi[1]; ++cy)
        for (int64_t cx = clo[0]; cx <= chi[0]; ++cx) {
          int64_t cell = (cz * nc1d(p, 1) + cy) * nc1d(p, 0) + cx;
          int64_t cc[3] = {cx, cy, cz};
          int il = 0, stride = 1;
          for (int e = 0; e < dim; ++e) { il += (int)(m[e] - k * cc[e]) * stride; stride *= n; }
          cell_eval_t ce;
          int st = cell_eval(p, cell, n, &ce);
          if (st) {
#pragma omp atomic write
            status = st;
          }
          or_cell_dofs(p, cell, dofs);
          for (int q = 0; q < ce.nqv; ++q) {
            double cj = coeff(p, ce.xq + q * dim) * ce.jxw[q];
            for (int j = 0; j < nv; ++j) {
              if (or_is_constrained(p, dofs[j])) continue;
              double d = 0.0;
              for (int a = 0; a < dim; ++a)
                d += ce.grad[(q * nv + il) * dim + a] * ce.grad[(q * nv + j) * dim + a];
              s += d * cj * x[dofs[j]];
            }
          }
          cell_eval_free(&ce);
        }
    out[r] = s;
  }
  return status;
}

/* O8: b_i = sum_c sum_q f(x_q) phi_i(x_q) JxW (§2.4 RHS loop). */
static double f_rhs(const or_problem *p, int f_kind, const double *x) {
  if (f_kind == 0) return 1.0;
  double s = p->dim * OR_PI * OR_PI;
  for (int d = 0; d < p->dim; ++d) s *= sin(OR_PI * x[d]);
  return s;
}

int or_rhs(const or_problem *p, int f_kind, int nq, double *b) {
  const int64_t n = or_n_dofs(p), ncell = or_n_cells(p);
  const int nv = pow_int(p->degree + 1, p->dim);
  memset(b, 0, sizeof(double) * n);
  int status = 0;
  for (int color = 0; color < (1 << p->dim); ++color) {
#pragma omp parallel
    {
      int64_t *dofs = (int64_t *)malloc(sizeof(int64_t) * nv);
#pragma omp for schedule(dynamic, 4)
      for (int64_t cell = 0; cell < ncell; ++cell) {
        int64_t c[3];
        cell_coords(p, cell, c);
        int cc = (int)((c[0] & 1) | ((c[1] & 1) << 1) | ((c[2] & 1) << 2));
        if (cc != color) continue;
        cell_eval_t ce;
        int st = cell_eval(p, cell, nq, &ce);
        if (st) {
#pragma omp atomic write
          status = st;
        }
        or_cell_dofs(p, cell, dofs);
        for (int q = 0; q < ce.nqv; ++q) {
          double fj = f_rhs(p, f_kind, ce.xq + q * p->dim) * ce.jxw[q];
          for (int i = 0; i < nv; ++i) b[dofs[i]] += ce.phi[q * nv + i] * fj;
        }
        cell_eval_free(&ce);
      }
      free(dofs);
    }
  }
  for (int64_t g = 0; g < n; ++g)
    if (or_is_constrained(p, g)) b[g] = 0.0;
  return status;
}

double or_l2_error(const or_problem *p, const double *u, int nq) {
  const int64_t ncell = or_n_cells(p);
  const int nv = pow_int(p->degree + 1, p->dim);
  double err = 0.0;
#pragma omp parallel reduction(+ : err)
  {
    int64_t *dofs = (int64_t *)malloc(sizeof(int64_t) * nv);
#pragma omp for schedule(dynamic, 4)
    for (int64_t cell = 0; cell < ncell; ++cell) {
      cell_eval_t ce;
      cell_eval(p, cell, nq, &ce);
      or_cell_dofs(p, cell, dofs);
      for (int q = 0; q < ce.nqv; ++q) {
        double uh = 0.0;
        for (int j = 0; j < nv; ++j) uh += u[dofs[j]] * ce.phi[q * nv + j];
        double ue = 1.0;
        for (int d = 0; d < p->dim; ++d) ue *= sin(OR_PI * ce.xq[q * p->dim + d]);
        err += (uh - ue) * (uh - ue) * ce.jxw[q];
      }
      cell_eval_free(&ce);
    }
    free(dofs);
  }
  return sqrt(err);
}

/* ------------------------------------------------------------------------- */
/* O12: Kronecker-sum oracle.  1D stiffness K_e and mass M_e are assembled by  */
/* the 1D instance of O5/O6; the 3D operator is the sum over e of K along e    */
/* and M along the other directions, applied to x with constrained entries    */
/* zeroed, then R3 on constrained rows.                                        */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  int64_t *rowptr;
  int32_t *col;
  double *val;
} csr1d_t;

static void build1d(const or_problem *p, int e, int which, csr1d_t *m) {
  or_problem q;
  memset(&q, 0, sizeof(q));
  q.dim = 1;
  q.nc[0] = p->nc[e];
  q.lo[0] = p->lo[e];
  q.hi[0] = p->hi[e];
  q.degree = p->degree;
  q.geom = 0;
  q.coeff_kind = 0;
  q.coeff_value = 1.0;
  m->n = or_n_dofs(&q);
  int64_t nnz = or_csr_nnz(&q);
  m->rowptr = (int64_t *)malloc(sizeof(int64_t) * (m->n + 1));
  m->col = (int32_t *)malloc(sizeof(int32_t) * nnz);
  m->val = (double *)malloc(sizeof(double) * nnz);
  or_assemble_csr(&q, which, 0, m->rowptr, m->col, m->val);
}

static void free1d(csr1d_t *m) {
  free(m->rowptr);
  free(m->col);
  free(m->val);
}

/* out = (1D matrix along direction e) applied to the lexicographic array in */
static void apply_along(const csr1d_t *m, int e, const int64_t N[3], const double *in, double *out) {
  const int64_t stride = e == 0 ? 1 : (e == 1 ? N[0] : N[0] * N[1]);
  const int64_t total = N[0] * N[1] * N[2];
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < total; ++g) {
    int64_t me = (g / stride) % N[e];
    int64_t base = g - me * stride;
    double s = 0.0;
    for (int64_t q = m->rowptr[me]; q < m->rowptr[me + 1]; ++q) s += m->val[q] * in[base + m->col[q] * stride];
    out[g] = s;
  }
}

int or_kron_apply(const or_problem *p, const double *x, double *y) {
  if (p->geom != 0 || p->coeff_kind != 0) return -1;
  const int dim = p->dim;
  const int64_t N[3] = {n1d(p, 0), n1d(p, 1), n1d(p, 2)};
  const int64_t total = N[0] * N[1] * N[2];
  csr1d_t K[3], M[3];
  for (int e = 0; e < dim; ++e) { build1d(p, e, 0, &K[e]); build1d(p, e, 1, &M[e]); }
  double *xt = (double *)malloc(sizeof(double) * total);
  double *t1 = (double *)malloc(sizeof(double) * total);
  double *t2 = (double *)malloc(sizeof(double) * total);
  for (int64_t g = 0; g < total; ++g) xt[g] = or_is_constrained(p, g) ? 0.0 : x[g];
  memset(y, 0, sizeof(double) * total);
  for (int term = 0; term < dim; ++term) {
    /* term: K along `term`, M along every other direction */
    const double *src = xt;
    for (int e = 0; e < dim; ++e) {
      double *dst = (src == t1) ? t2 : t1;
      apply_along(e == term ? &K[e] : &M[e], e, N, src, dst);
      src = dst;
    }
    for (int64_t g = 0; g < total; ++g) y[g] += p->coeff_value * src[g];
  }
  for (int64_t g = 0; g < total; ++g)
    if (or_is_constrained(p, g)) y[g] = x[g];
  free(xt);
  free(t1);
  free(t2);
  for (int e = 0; e < dim; ++e) { free1d(&K[e]); free1d(&M[e]); }
  return 0;
}
