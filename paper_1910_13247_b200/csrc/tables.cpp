// tables.cpp -- 1D rules and basis tables on [0,1] for the CUDA path (§8(a) a1).
//
// Written independently of oracle/ (DESIGN.md "Oracle independence"): Gauss
// points are the roots of P_n found by long-double Newton iterations on the
// Bonnet recurrence started from the Tricomi approximation, Lobatto nodes the
// roots of (1-t^2) P_k'(t) found by Newton on P_{k-1} - P_{k+1} (proportional
// to it), and every basis table is evaluated through the barycentric form of
// Lagrange interpolation.  D = Co * S is formed by exact collocation (the
// derivative of a degree-k polynomial is reproduced by the k+1 Gauss points).
// Readings: R1 (Gauss-Legendre, k+1 points), R2 (GLL support points).
#include <cmath>
#include <cstring>

#include "internal.h"

namespace mf {
namespace {

typedef long double ld;
const ld kPi = 3.141592653589793238462643383279502884L;

// P_m(t) for m = 0..M by Bonnet's recurrence
void legendre_all(int M, ld t, ld *P) {
  P[0] = 1.0L;
  if (M >= 1) P[1] = t;
  for (int m = 1; m < M; ++m) P[m + 1] = ((2 * m + 1) * t * P[m] - m * P[m - 1]) / (m + 1);
}

void gauss_on_01(int n, ld *x, ld *w) {
  ld P[kMaxN + 3];
  for (int i = 0; i < n; ++i) {
    // Tricomi: t ~ (1 - (n-1)/(8 n^3)) cos(pi (4i+3)/(4n+2)); roots ascending in t
    ld t = -(1.0L - (n - 1.0L) / (8.0L * n * n * n)) * std::cos(kPi * (4 * i + 3) / (4.0L * n + 2.0L));
    for (int it = 0; it < 60; ++it) {
      legendre_all(n, t, P);
      ld dP = n * (P[n - 1] - t * P[n]) / (1.0L - t * t);
      ld dt = P[n] / dP;
      t -= dt;
      if (std::fabs(dt) < 1e-21L) break;
    }
    legendre_all(n, t, P);
    ld dP = n * (P[n - 1] - t * P[n]) / (1.0L - t * t);
    x[i] = 0.5L * (t + 1.0L);
    w[i] = 1.0L / ((1.0L - t * t) * dP * dP);  // (2 / ((1-t^2) P'^2)) / 2
  }
}

void lobatto_on_01(int k, ld *x) {
  ld P[kMaxN + 3];
  x[0] = 0.0L;
  x[k] = 1.0L;
  for (int j = 1; j < k; ++j) {
    // f(t) = P_{k-1}(t) - P_{k+1}(t) = (2k+1)/(k(k+1)) (1-t^2) P_k'(t)... roots = interior GLL
    ld t = -std::cos(kPi * j / k);
    for (int it = 0; it < 60; ++it) {
      legendre_all(k + 1, t, P);
      ld f = P[k - 1] - P[k + 1];
      // f'(t) = P_{k-1}'(t) - P_{k+1}'(t) = -(2k+1) P_k(t)   (standard identity)
      ld df = -(2.0L * k + 1.0L) * P[k];
      ld dt = f / df;
      t -= dt;
      if (std::fabs(dt) < 1e-21L) break;
    }
    x[j] = 0.5L * (t + 1.0L);
  }
}

// barycentric weights lambda_j = 1 / prod_{m != j} (x_j - x_m)
void bary_weights(int n, const ld *x, ld *lam) {
  for (int j = 0; j < n; ++j) {
    ld p = 1.0L;
    for (int m = 0; m < n; ++m)
      if (m != j) p *= (x[j] - x[m]);
    lam[j] = 1.0L / p;
  }
}

// values of all Lagrange polynomials on nodes x at point y (barycentric, second form)
void bary_eval(int n, const ld *x, const ld *lam, ld y, ld *out) {
  for (int j = 0; j < n; ++j)
    if (y == x[j]) {
      for (int m = 0; m < n; ++m) out[m] = (m == j) ? 1.0L : 0.0L;
      return;
    }
  ld s = 0.0L;
  for (int j = 0; j < n; ++j) s += lam[j] / (y - x[j]);
  for (int j = 0; j < n; ++j) out[j] = lam[j] / (y - x[j]) / s;
}

}  // namespace

void build_tables(int k, Tables *t) {
  std::memset(t, 0, sizeof(Tables));
  const int n = k + 1;
  ld xg[kMaxN], wg[kMaxN], xl[kMaxN], lamg[kMaxN], laml[kMaxN];
  gauss_on_01(n, xg, wg);
  lobatto_on_01(k, xl);
  bary_weights(n, xg, lamg);
  bary_weights(n, xl, laml);
  ld S[kMaxN][kMaxN], Co[kMaxN][kMaxN];
  for (int q = 0; q < n; ++q) bary_eval(n, xl, laml, xg[q], S[q]);
  // collocation differentiation matrix on the Gauss points
  for (int q = 0; q < n; ++q) {
    ld diag = 0.0L;
    for (int p = 0; p < n; ++p) {
      if (p == q) continue;
      Co[q][p] = (lamg[p] / lamg[q]) / (xg[q] - xg[p]);
      diag -= Co[q][p];
    }
    Co[q][q] = diag;
  }
  for (int q = 0; q < n; ++q) {
    t->w[q] = (double)wg[q];
    t->xi[q] = (double)xg[q];
    t->gll[q] = (double)xl[q];
    for (int i = 0; i < n; ++i) {
      t->S[q][i] = (double)S[q][i];
      t->Co[q][i] = (double)Co[q][i];
      ld d = 0.0L;
      for (int p = 0; p < n; ++p) d += Co[q][p] * S[p][i];
      t->D[q][i] = (double)d;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      ld mm = 0.0L, kk = 0.0L;
      for (int q = 0; q < n; ++q) {
        ld di = 0.0L, dj = 0.0L;
        for (int p = 0; p < n; ++p) {
          di += Co[q][p] * S[p][i];
          dj += Co[q][p] * S[p][j];
        }
        mm += wg[q] * S[q][i] * S[q][j];
        kk += wg[q] * di * dj;
      }
      t->Mr[i][j] = (double)mm;
      t->Kr[i][j] = (double)kk;
    }
  const int m = n / 2, h = (n + 1) / 2;
  auto eo = [&](const double A[kMaxN][kMaxN], double E[5][5], double O[5][5]) {
    for (int i = 0; i < h; ++i) {
      for (int j = 0; j < m; ++j) E[i][j] = 0.5 * (A[i][j] + A[i][n - 1 - j]);
      if (n & 1) E[i][m] = A[i][m];
    }
    if (n & 1)
      for (int j = 0; j < m; ++j) E[m][j] = A[m][j];
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) O[i][j] = 0.5 * (A[i][j] - A[i][n - 1 - j]);
  };
  eo(t->Mr, t->Me, t->Mo);
  eo(t->Kr, t->Ke, t->Ko);
}

}  // namespace mf
