// Host-side constant generation: reference P_k element matrices and DG(q)
// temporal matrices (setup constants, a few hundred numbers).
//
// Independent of the oracle by construction: the Lagrange basis is the
// barycentric product formula (not a Vandermonde inverse), derivatives come
// from forward-mode dual numbers, and integrals use Gauss-Legendre rules
// (collapsed/Duffy on the triangle) rather than closed-form monomial integrals.
// DESIGN.md R20: any rule exact for the integrands; these are exact to degree
// 14 on the triangle and 2*ng-1 on the interval.
//
// Eq. heatfem: (U, psi) -> mass, (grad U, grad psi) -> stiffness.
// Eq. dgintime with R1 (upwind traces) and R2 (equispaced
// Lagrange nodes incl. both end points) -> C + E0, Mt, E1.
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.h"

namespace wrmg {
namespace {

struct Dual {
  double v, dx, dy;
};
inline Dual mul(Dual a, Dual b) { return {a.v * b.v, a.dx * b.v + a.v * b.dx, a.dy * b.v + a.v * b.dy}; }

// Gauss-Legendre nodes/weights on [0, 1].
void gauss01(int n, double *x, double *w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int j = 2; j <= n; ++j) {
        double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      // p1 = P_n(z), p0 = P_{n-1}(z)
      double dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1.0, p1 = z;
    for (int j = 2; j <= n; ++j) {
      double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
      p0 = p1;
      p1 = p2;
    }
    double dp = n * (z * p1 - p0) / (z * z - 1.0);
    x[i] = 0.5 * (1.0 - z);
    w[i] = 1.0 / ((1.0 - z * z) * dp * dp);  // 2/((1-z^2)P'^2) on [-1,1], halved for [0,1]
  }
}

// Product-formula Lagrange basis function (a, b) of degree k at barycentric
// duals l0, l1, l2 (each multiplied by k).
Dual lagrange_tri(int k, int a, int b, Dual kl0, Dual kl1, Dual kl2) {
  int c = k - a - b;
  Dual r = {1.0, 0.0, 0.0};
  for (int s = 0; s < c; ++s) r = mul(r, Dual{(kl0.v - s) / (s + 1), kl0.dx / (s + 1), kl0.dy / (s + 1)});
  for (int s = 0; s < a; ++s) r = mul(r, Dual{(kl1.v - s) / (s + 1), kl1.dx / (s + 1), kl1.dy / (s + 1)});
  for (int s = 0; s < b; ++s) r = mul(r, Dual{(kl2.v - s) / (s + 1), kl2.dx / (s + 1), kl2.dy / (s + 1)});
  return r;
}

}  // namespace

void build_ref_element(int k, RefElement *E) {
  std::memset(E, 0, sizeof(*E));
  E->k = k;
  int n = 0;
  for (int b = 0; b <= k; ++b)
    for (int a = 0; a + b <= k; ++a) {
      E->a[n] = a;
      E->b[n] = b;
      ++n;
    }
  E->nloc = n;
  const int ng = 8;
  double gx[ng], gw[ng];
  gauss01(ng, gx, gw);
  for (int iu = 0; iu < ng; ++iu)
    for (int iv = 0; iv < ng; ++iv) {
      double v = gx[iv], u = gx[iu];
      double xi = u * (1.0 - v), eta = v, wt = gw[iu] * gw[iv] * (1.0 - v);
      Dual kl1 = {k * xi, (double)k, 0.0}, kl2 = {k * eta, 0.0, (double)k};
      Dual kl0 = {k * (1.0 - xi - eta), -(double)k, -(double)k};
      Dual phi[kMaxLoc];
      for (int i = 0; i < n; ++i) phi[i] = lagrange_tri(k, E->a[i], E->b[i], kl0, kl1, kl2);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          E->M[i * n + j] += wt * phi[i].v * phi[j].v;
          E->K[i * n + j] += wt * (phi[i].dx * phi[j].dx + phi[i].dy * phi[j].dy);
        }
    }
}

void eval_basis_grad(int k, double xi, double eta, double *v, double *dxi, double *deta) {
  Dual kl1 = {k * xi, (double)k, 0.0}, kl2 = {k * eta, 0.0, (double)k};
  Dual kl0 = {k * (1.0 - xi - eta), -(double)k, -(double)k};
  int n = 0;
  for (int b = 0; b <= k; ++b)
    for (int a = 0; a + b <= k; ++a) {
      Dual p = lagrange_tri(k, a, b, kl0, kl1, kl2);
      v[n] = p.v;
      dxi[n] = p.dx;
      deta[n] = p.dy;
      ++n;
    }
}

void gauss_triangle(int ng, std::vector<double> &xi, std::vector<double> &eta, std::vector<double> &w) {
  double gx[32], gw[32];
  gauss01(ng, gx, gw);
  xi.clear();
  eta.clear();
  w.clear();
  for (int iu = 0; iu < ng; ++iu)
    for (int iv = 0; iv < ng; ++iv) {
      double v = gx[iv], u = gx[iu];
      xi.push_back(u * (1.0 - v));
      eta.push_back(v);
      w.push_back(gw[iu] * gw[iv] * (1.0 - v));
    }
}

void eval_basis_klambda(int k, double kl1, double kl2, double *vals) {
  Dual d1 = {kl1, 0, 0}, d2 = {kl2, 0, 0}, d0 = {k - kl1 - kl2, 0, 0};
  int n = 0;
  for (int b = 0; b <= k; ++b)
    for (int a = 0; a + b <= k; ++a) vals[n++] = lagrange_tri(k, a, b, d0, d1, d2).v;
}

void build_temporal(int q, double dt, Temporal *T) {
  std::memset(T, 0, sizeof(*T));
  T->q = q;
  T->nq = q + 1;
  const int nq = q + 1;
  auto basis = [&](int a, double tau, double *d) {
    // Lagrange basis on nodes s/q (q >= 1); DG0 is the constant 1 (R2)
    if (q == 0) {
      *d = 0.0;
      return 1.0;
    }
    double v = 1.0, dv = 0.0;
    for (int s = 0; s <= q; ++s) {
      if (s == a) continue;
      double f = (tau - (double)s / q) / ((double)a / q - (double)s / q);
      double df = 1.0 / ((double)a / q - (double)s / q);
      dv = dv * f + v * df;
      v *= f;
    }
    *d = dv;
    return v;
  };
  const int ng = q + 3;
  double gx[16], gw[16];
  gauss01(ng, gx, gw);
  double C[16] = {0}, Mt[16] = {0}, Tr[64] = {0};
  for (int g = 0; g < ng; ++g) {
    double v[4], d[4];
    for (int a = 0; a < nq; ++a) v[a] = basis(a, gx[g], &d[a]);
    for (int a = 0; a < nq; ++a)
      for (int b = 0; b < nq; ++b) {
        C[a * nq + b] += gw[g] * d[b] * v[a];
        Mt[a * nq + b] += gw[g] * v[a] * v[b];
        for (int c = 0; c < nq; ++c) Tr[(a * nq + b) * nq + c] += gw[g] * v[a] * v[b] * v[c];
      }
  }
  double v0[4], v1[4], dd;
  for (int a = 0; a < nq; ++a) {
    v0[a] = basis(a, 0.0, &dd);
    v1[a] = basis(a, 1.0, &dd);
  }
  for (int a = 0; a < nq; ++a) T->phi0[a] = v0[a];
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b) {
      T->CE[a * nq + b] = C[a * nq + b] + v0[a] * v0[b];
      T->Mt[a * nq + b] = dt * Mt[a * nq + b];
      T->E1[a * nq + b] = v0[a] * v1[b];
      for (int c2 = 0; c2 < nq; ++c2) T->T[(a * nq + b) * nq + c2] = dt * Tr[(a * nq + b) * nq + c2];
    }
}

}  // namespace wrmg
