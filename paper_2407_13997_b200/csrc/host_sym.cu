// Symmetry-reduced Kronecker patch solves (host setup for kernels_sweep_sym.cu).
//
// The interior vertex star of the anti-diagonal P_k lattice (PAPER.md:381,
// 524-525) is invariant under the point reflection s_p: (x, y) -> (-x, -y) and
// the reflection s_d: (x, y) -> (y, x) about the vertex; both map the mesh onto
// itself, so the patch matrices M_p, K_p commute with the node permutations of
// the group G = {e, s_p, s_d, s_p s_d} ~ Z2 x Z2.  In the orthonormal
// symmetry-adapted basis U (orbit sums / differences, one column per (orbit,
// character chi of G that is trivial on the orbit's stabiliser)) both become
// block diagonal with one block per character:
//     U^T M_p U = diag(M_chi),  U^T K_p U = diag(K_chi),   chi in {++, +-, -+, --}
// (P3: blocks 7, 3, 4, 5 instead of one 19 x 19; P2: 3, 1, 1, 2 instead of 7 x 7).
// The generalised eigenproblems K_chi v = lambda M_chi v, v^T M_chi v = 1 are
// solved per block, so the patch space-time solve of kernels_kron.cu
// (ghat = V^T g, per-mode DG(q) solves and end-trace recurrence, x = V w) costs
// sum_chi d_chi^2 instead of m_p^2 FMAs per transform and time value.  It is the
// same exact solve of A_p x = g (R9); only the basis of the modes differs.
//
// Slot order (fixed, the kernel's compile-time layout): the vertex; n1 free
// orbits of size 4 as (e, s_p e, s_d e, s_p s_d e); n2 orbits of size 2 fixed by
// s_p s_d as (e, s_p e); n3 orbits of size 2 fixed by s_d as (e, s_p e).
// Coordinates y: block ++ = [vertex, n1, n2, n3 orbits], +- = [n1], -+ = [n1, n3],
// -- = [n1, n2].
#include <algorithm>
#include <cmath>
#include <map>
#include <utility>
#include <vector>

#include "plan.h"
#include "sym.h"

namespace wrmg {

namespace {

// (character chi, group element g) -> chi(g), g in (e, s_p, s_d, s_p s_d), chi in (++, +-, -+, --)
int chr(int chi, int g) {
  const int cp = (chi == 2 || chi == 3) ? -1 : 1, cd = (chi == 1 || chi == 3) ? -1 : 1;
  return g == 0 ? 1 : g == 1 ? cp : g == 2 ? cd : cp * cd;
}

// Symmetric generalised eigenproblem K v = lambda M v (M SPD), d <= kSymMaxD:
// Cholesky M = L L^T, C = L^-1 K L^-T, cyclic Jacobi C = Q diag Q^T, V = L^-T Q.
bool gen_eig(int d, const double *M, const double *K, double *V, double *lam) {
  std::vector<double> L(d * d, 0.0), C(d * d), Q(d * d, 0.0), X(d * d);
  for (int j = 0; j < d; ++j) {
    double s = M[j * d + j];
    for (int p = 0; p < j; ++p) s -= L[j * d + p] * L[j * d + p];
    if (!(s > 0.0)) return false;
    L[j * d + j] = std::sqrt(s);
    for (int i = j + 1; i < d; ++i) {
      double t = M[i * d + j];
      for (int p = 0; p < j; ++p) t -= L[i * d + p] * L[j * d + p];
      L[i * d + j] = t / L[j * d + j];
    }
  }
  // X = L^-1 K, C = L^-1 X^T  (= L^-1 K L^-T, K symmetric)
  for (int c = 0; c < d; ++c)
    for (int i = 0; i < d; ++i) {
      double s = K[i * d + c];
      for (int p = 0; p < i; ++p) s -= L[i * d + p] * X[p * d + c];
      X[i * d + c] = s / L[i * d + i];
    }
  for (int c = 0; c < d; ++c)
    for (int i = 0; i < d; ++i) {
      double s = X[c * d + i];
      for (int p = 0; p < i; ++p) s -= L[i * d + p] * C[p * d + c];
      C[i * d + c] = s / L[i * d + i];
    }
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) C[i * d + j] = C[j * d + i] = 0.5 * (C[i * d + j] + C[j * d + i]);
  for (int i = 0; i < d; ++i) Q[i * d + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) (i == j ? dia : off) += C[i * d + j] * C[i * d + j];
    if (off <= 1e-32 * dia) break;
    for (int p = 0; p < d - 1; ++p)
      for (int q = p + 1; q < d; ++q) {
        const double apq = C[p * d + q];
        if (std::fabs(apq) <= 1e-300) continue;
        const double th = (C[q * d + q] - C[p * d + p]) / (2.0 * apq);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < d; ++k) {
          const double akp = C[k * d + p], akq = C[k * d + q];
          C[k * d + p] = c * akp - s * akq;
          C[k * d + q] = s * akp + c * akq;
          const double qkp = Q[k * d + p], qkq = Q[k * d + q];
          Q[k * d + p] = c * qkp - s * qkq;
          Q[k * d + q] = s * qkp + c * qkq;
        }
        for (int k = 0; k < d; ++k) {
          const double apk = C[p * d + k], aqk = C[q * d + k];
          C[p * d + k] = c * apk - s * aqk;
          C[q * d + k] = s * apk + c * aqk;
        }
        C[p * d + q] = C[q * d + p] = 0.0;
      }
  }
  for (int i = 0; i < d; ++i) lam[i] = C[i * d + i];
  // V = L^-T Q (back substitution with L^T, column by column)
  for (int c = 0; c < d; ++c)
    for (int i = d - 1; i >= 0; --i) {
      double s = Q[i * d + c];
      for (int p = i + 1; p < d; ++p) s -= L[p * d + i] * V[p * d + c];
      V[i * d + c] = s / L[i * d + i];
    }
  return true;
}

}  // namespace

bool plan_sym_class(const PlanLevel &P, int k, int cls, std::vector<int32_t> &perm, int counts[3]) {
  perm.clear();
  if (k < 2 || k > 3 || cls < 0 || cls >= P.ntypes) return false;
  const int64_t rep = P.type_rep[cls];
  const int mp = P.psize[rep];
  if (mp != (k == 2 ? 7 : 19)) return false;
  const int v = P.pvert[rep], vi = v % (P.nx + 1), vj = v / (P.nx + 1);
  std::map<std::pair<int, int>, int> at;  // relative lattice coordinates -> patch slot
  std::vector<std::pair<int, int>> xy(mp);
  for (int j = 0; j < mp; ++j) {
    const int32_t i = P.pnodes[rep * P.mp + j];
    if (i < 0) return false;
    xy[j] = {(int)(i % P.Lx) - k * vi, (int)(i / P.Lx) - k * vj};
    at[xy[j]] = j;
  }
  auto img = [&](int j, int g) -> int {  // g in (e, s_p, s_d, s_p s_d)
    int x = xy[j].first, y = xy[j].second;
    if (g == 1 || g == 3) { x = -x; y = -y; }
    if (g == 2 || g == 3) std::swap(x, y);
    auto it = at.find({x, y});
    return it == at.end() ? -1 : it->second;
  };
  std::vector<int> seen(mp, 0), t0, t1, t2, t3;
  for (int j = 0; j < mp; ++j) {
    if (seen[j]) continue;
    int o[4];
    for (int g = 0; g < 4; ++g) {
      o[g] = img(j, g);
      if (o[g] < 0) return false;  // not closed under the group: not the interior class
    }
    std::vector<int> orb(o, o + 4);
    std::sort(orb.begin(), orb.end());
    orb.erase(std::unique(orb.begin(), orb.end()), orb.end());
    for (int s : orb) seen[s] = 1;
    if (orb.size() == 1) {
      t0.push_back(j);
    } else if (orb.size() == 4) {
      for (int g = 0; g < 4; ++g) t1.push_back(o[g]);
    } else if (orb.size() == 2 && o[3] == j) {  // fixed by s_p s_d
      t2.push_back(j);
      t2.push_back(o[1]);
    } else if (orb.size() == 2 && o[2] == j) {  // fixed by s_d
      t3.push_back(j);
      t3.push_back(o[1]);
    } else {
      return false;
    }
  }
  if (t0.size() != 1) return false;
  counts[0] = (int)t1.size() / 4;
  counts[1] = (int)t2.size() / 2;
  counts[2] = (int)t3.size() / 2;
  const int want[2][3] = {{1, 1, 0}, {3, 2, 1}};
  for (int e = 0; e < 3; ++e)
    if (counts[e] != want[k - 2][e]) return false;
  perm = t0;
  perm.insert(perm.end(), t1.begin(), t1.end());
  perm.insert(perm.end(), t2.begin(), t2.end());
  perm.insert(perm.end(), t3.begin(), t3.end());
  return true;
}

bool sym_factor(int k, const double *Mp, const double *Kp, const Temporal &tm, SymTab *out) {
  const int n1 = k == 2 ? 1 : 3, n2 = k == 2 ? 1 : 2, n3 = k == 2 ? 0 : 1;
  const int mp = 1 + 4 * n1 + 2 * n2 + 2 * n3;
  const int d[4] = {1 + n1 + n2 + n3, n1, n1 + n3, n1 + n2};
  // U: slot x coordinate, coordinates ordered by block (chi) as in the header
  std::vector<double> U(mp * mp, 0.0);
  int col = 0;
  const double h = 0.5, r = 1.0 / std::sqrt(2.0);
  for (int chi = 0; chi < 4; ++chi) {
    if (chi == 0) U[0 * mp + col++] = 1.0;  // vertex
    for (int o = 0; o < n1; ++o, ++col)
      for (int g = 0; g < 4; ++g) U[(1 + 4 * o + g) * mp + col] = h * chr(chi, g);
    if (chi == 0 || chi == 3)
      for (int o = 0; o < n2; ++o, ++col) {
        const int s0 = 1 + 4 * n1 + 2 * o;
        U[s0 * mp + col] = r;
        U[(s0 + 1) * mp + col] = r * chr(chi, 1);
      }
    if (chi == 0 || chi == 2)
      for (int o = 0; o < n3; ++o, ++col) {
        const int s0 = 1 + 4 * n1 + 2 * n2 + 2 * o;
        U[s0 * mp + col] = r;
        U[(s0 + 1) * mp + col] = r * chr(chi, 1);
      }
  }
  if (col != mp) return false;
  // B = U^T X U for X = M, K; off-block entries must vanish (the symmetry check)
  auto congr = [&](const double *X, std::vector<double> &B) {
    std::vector<double> T(mp * mp, 0.0);
    B.assign(mp * mp, 0.0);
    for (int i = 0; i < mp; ++i)
      for (int c = 0; c < mp; ++c) {
        double s = 0.0;
        for (int j = 0; j < mp; ++j) s += X[i * mp + j] * U[j * mp + c];
        T[i * mp + c] = s;
      }
    for (int a = 0; a < mp; ++a)
      for (int c = 0; c < mp; ++c) {
        double s = 0.0;
        for (int i = 0; i < mp; ++i) s += U[i * mp + a] * T[i * mp + c];
        B[a * mp + c] = s;
      }
  };
  std::vector<double> BM, BK;
  congr(Mp, BM);
  congr(Kp, BK);
  int blk[19], b0[5] = {0, 0, 0, 0, 0};
  for (int chi = 0; chi < 4; ++chi) b0[chi + 1] = b0[chi] + d[chi];
  for (int chi = 0; chi < 4; ++chi)
    for (int a = b0[chi]; a < b0[chi + 1]; ++a) blk[a] = chi;
  double mm = 0.0, mk = 0.0;
  for (int e = 0; e < mp * mp; ++e) {
    mm = std::max(mm, std::fabs(BM[e]));
    mk = std::max(mk, std::fabs(BK[e]));
  }
  for (int a = 0; a < mp; ++a)
    for (int c = 0; c < mp; ++c)
      if (blk[a] != blk[c] && (std::fabs(BM[a * mp + c]) > 1e-12 * mm || std::fabs(BK[a * mp + c]) > 1e-12 * mk))
        return false;
  *out = SymTab{};
  const int nq = tm.nq;
  int voff = 0, mode = 0;
  for (int chi = 0; chi < 4; ++chi) {
    const int dd = d[chi];
    if (dd == 0) continue;
    std::vector<double> Mb(dd * dd), Kb(dd * dd), Vb(dd * dd), lam(dd);
    for (int a = 0; a < dd; ++a)
      for (int c = 0; c < dd; ++c) {
        Mb[a * dd + c] = BM[(b0[chi] + a) * mp + b0[chi] + c];
        Kb[a * dd + c] = BK[(b0[chi] + a) * mp + b0[chi] + c];
      }
    if (!gen_eig(dd, Mb.data(), Kb.data(), Vb.data(), lam.data())) return false;
    for (int e = 0; e < dd * dd; ++e) out->V[voff + e] = Vb[e];
    voff += dd * dd;
    for (int i = 0; i < dd; ++i, ++mode) {  // S_i = (CE + lambda_i Mt)^-1, Gauss-Jordan with partial pivoting
      double a[16], inv[16];
      for (int p = 0; p < nq; ++p)
        for (int q = 0; q < nq; ++q) {
          a[p * nq + q] = tm.CE[p * nq + q] + lam[i] * tm.Mt[p * nq + q];
          inv[p * nq + q] = p == q ? 1.0 : 0.0;
        }
      for (int c = 0; c < nq; ++c) {
        int pr = c;
        for (int p = c + 1; p < nq; ++p)
          if (std::fabs(a[p * nq + c]) > std::fabs(a[pr * nq + c])) pr = p;
        for (int q = 0; q < nq; ++q) {
          std::swap(a[c * nq + q], a[pr * nq + q]);
          std::swap(inv[c * nq + q], inv[pr * nq + q]);
        }
        const double dg = a[c * nq + c];
        if (dg == 0.0) return false;
        for (int q = 0; q < nq; ++q) {
          a[c * nq + q] /= dg;
          inv[c * nq + q] /= dg;
        }
        for (int p = 0; p < nq; ++p)
          if (p != c) {
            const double f = a[p * nq + c];
            for (int q = 0; q < nq; ++q) {
              a[p * nq + q] -= f * a[c * nq + q];
              inv[p * nq + q] -= f * inv[c * nq + q];
            }
          }
      }
      for (int e = 0; e < nq * nq; ++e) out->S[mode * 16 + e] = inv[e];
      out->sig[mode] = inv[(nq - 1) * nq + 0];
      double pp = out->sig[mode];  // the squarings the scan would form in-kernel, bit for bit
      for (int k2 = 0; k2 < 5; ++k2) {
        out->sig2[k2][mode] = pp;
        pp *= pp;
      }
    }
  }
  return true;
}

}  // namespace wrmg
