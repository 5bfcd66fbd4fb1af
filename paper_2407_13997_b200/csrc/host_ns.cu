// Host-side setup of the Navier-Stokes path (integer plans and a few hundred
// reference constants; no per-DoF arithmetic):
//   * Taylor-Hood reference integrals (eq. nsfem) by collapsed
//     Gauss quadrature of the product-formula basis (host_fem.cu), exact for the
//     polynomial integrands (R20);
//   * sid numbering, Dirichlet/lid data (R5), the sid CSR pattern;
//   * Vanka+star patches (Fig. patches right; R8): both velocity
//     components on the closure of each vertex star, pressure on the open star;
//   * block-diagonal interpolation diag(Pu, Pu, Pp) (R12).
#include <algorithm>
#include <vector>

#include "lattice.h"
#include "ns.h"
#include "plan.h"

namespace wrmg {

void build_th_element(int k, THElement *E) {
  *E = THElement{};
  const int ku = k + 1, kp = k;
  E->ku = ku;
  E->kp = kp;
  E->nu = (ku + 1) * (ku + 2) / 2;
  E->np = (kp + 1) * (kp + 2) / 2;
  const int nu = E->nu, np = E->np;
  std::vector<double> X, Y, W;
  gauss_triangle(8, X, Y, W);  // exact to degree 14 (integrands here: <= 3 ku - 1 = 11)
  for (size_t g = 0; g < W.size(); ++g) {
    double v[kMaxLocU], vx[kMaxLocU], vy[kMaxLocU], p[kMaxLocU], px[kMaxLocU], py[kMaxLocU];
    eval_basis_grad(ku, X[g], Y[g], v, vx, vy);
    eval_basis_grad(kp, X[g], Y[g], p, px, py);
    const double w = W[g];
    const double *dv[2] = {vx, vy};
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nu; ++j) {
        E->Mh[i * nu + j] += w * v[i] * v[j];
        E->Kh[i * nu + j] += w * (vx[i] * vx[j] + vy[i] * vy[j]);
      }
    for (int d = 0; d < 2; ++d)
      for (int i = 0; i < nu; ++i) {
        for (int j = 0; j < np; ++j) E->Gh[(d * nu + i) * np + j] += w * p[j] * dv[d][i];
        for (int l = 0; l < nu; ++l)
          for (int j = 0; j < nu; ++j) E->Th[((d * nu + i) * nu + l) * nu + j] += w * v[i] * v[l] * dv[d][j];
      }
  }
}

namespace {

// All lattice nodes (degree kk) of the cells containing lattice node (I, J) of degree kn.
void cell_neighbours(int kn, int kk, int nx, int ny, int I, int J, int Lxk, std::vector<int32_t> &out) {
  int ci[6], cj[6], t[6], la[6], lb[6];
  const int nc = cells_of_node(kn, nx, ny, I, J, ci, cj, t, la, lb);
  out.clear();
  for (int c = 0; c < nc; ++c)
    for (int b = 0; b <= kk; ++b)
      for (int a = 0; a + b <= kk; ++a) {
        int I2, J2;
        loc_to_lattice(kk, ci[c], cj[c], t[c], a, b, &I2, &J2);
        out.push_back(J2 * Lxk + I2);
      }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

}  // namespace

void plan_ns_level(int nx, int ny, double h, int k, int bc, double lid_speed, NSPlan *P) {
  *P = NSPlan{};
  const int ku = k + 1, kp = k;
  P->nx = nx;
  P->ny = ny;
  P->h = h;
  P->ku = ku;
  P->kp = kp;
  P->Lux = ku * nx + 1;
  P->Luy = ku * ny + 1;
  P->Lpx = kp * nx + 1;
  P->Lpy = kp * ny + 1;
  P->Lu = (int64_t)P->Lux * P->Luy;
  P->Lp = (int64_t)P->Lpx * P->Lpy;
  P->ns = 2 * P->Lu + P->Lp;
  const int64_t Lu = P->Lu, Lp = P->Lp;
  // Dirichlet velocity on the whole boundary; lid (lid_speed, 0) on y = Y without the corners (R5)
  P->con.assign(P->ns, 0);
  P->g.assign(P->ns, 0.0);
  int64_t ncon = 0;
  for (int J = 0; J < P->Luy; ++J)
    for (int I = 0; I < P->Lux; ++I) {
      const bool b = (I == 0 || J == 0 || I == P->Lux - 1 || J == P->Luy - 1);
      const int64_t i = (int64_t)J * P->Lux + I;
      P->con[i] = P->con[Lu + i] = b;
      ncon += 2 * b;
      if (bc == WRMG_BC_LID && J == P->Luy - 1 && I > 0 && I < P->Lux - 1) P->g[i] = lid_speed;
    }
  P->nfree = P->ns - ncon;
  // sid CSR pattern: velocity columns (u_x block, then u_y block) before pressure columns
  P->rowptr.assign(P->ns + 1, 0);
  P->vvptr.assign(2 * Lu + 1, 0);
  P->col.clear();
  std::vector<int32_t> nu, np;
  std::vector<std::vector<int32_t>> vrow(Lu);
  std::vector<int32_t> vnnz(Lu);
  for (int J = 0; J < P->Luy; ++J)
    for (int I = 0; I < P->Lux; ++I) {
      const int64_t i = (int64_t)J * P->Lux + I;
      cell_neighbours(ku, ku, nx, ny, I, J, P->Lux, nu);
      // pressure nodes of the same cells: node (I, J) of degree ku lies in the cells found above
      int ci[6], cj[6], t[6], la[6], lb[6];
      const int nc = cells_of_node(ku, nx, ny, I, J, ci, cj, t, la, lb);
      np.clear();
      for (int c = 0; c < nc; ++c)
        for (int b = 0; b <= kp; ++b)
          for (int a = 0; a + b <= kp; ++a) {
            int I2, J2;
            loc_to_lattice(kp, ci[c], cj[c], t[c], a, b, &I2, &J2);
            np.push_back(J2 * P->Lpx + I2);
          }
      std::sort(np.begin(), np.end());
      np.erase(std::unique(np.begin(), np.end()), np.end());
      std::vector<int32_t> &row = vrow[i];
      for (int32_t j : nu) row.push_back(j);
      for (int32_t j : nu) row.push_back((int32_t)(Lu + j));
      for (int32_t j : np) row.push_back((int32_t)(2 * Lu + j));
      vnnz[i] = 2 * (int32_t)nu.size();
    }
  for (int d = 0; d < 2; ++d)
    for (int64_t i = 0; i < Lu; ++i) {
      const int64_t r = d * Lu + i;
      P->col.insert(P->col.end(), vrow[i].begin(), vrow[i].end());
      P->rowptr[r + 1] = (int32_t)P->col.size();
      P->vvptr[r + 1] = P->vvptr[r] + vnnz[i];
    }
  for (int Jp = 0; Jp < P->Lpy; ++Jp)
    for (int Ip = 0; Ip < P->Lpx; ++Ip) {
      const int64_t j = (int64_t)Jp * P->Lpx + Ip;
      cell_neighbours(kp, ku, nx, ny, Ip, Jp, P->Lux, nu);
      for (int32_t v : nu) P->col.push_back(v);
      for (int32_t v : nu) P->col.push_back((int32_t)(Lu + v));
      P->rowptr[2 * Lu + j + 1] = (int32_t)P->col.size();
    }
  (void)Lp;
  // Vanka+star patches, one per mesh vertex (R8)
  const int nv = (nx + 1) * (ny + 1);
  std::vector<std::vector<int32_t>> pre(nv);
  for (int Jp = 0; Jp < P->Lpy; ++Jp)
    for (int Ip = 0; Ip < P->Lpx; ++Ip) {
      int vi[3], vj[3];
      const int ne = entity_vertices(kp, Ip, Jp, vi, vj);
      for (int e = 0; e < ne; ++e) pre[vj[e] * (nx + 1) + vi[e]].push_back(Jp * P->Lpx + Ip);
    }
  std::vector<std::vector<int32_t>> pat;
  pat.reserve(nv);
  P->mu.assign(P->ns, 0);
  for (int vj = 0; vj <= ny; ++vj)
    for (int vi = 0; vi <= nx; ++vi) {
      cell_neighbours(ku, ku, nx, ny, ku * vi, ku * vj, P->Lux, nu);  // closure of the star
      std::vector<int32_t> s;
      for (int d = 0; d < 2; ++d)
        for (int32_t i : nu)
          if (!P->con[d * Lu + i]) s.push_back((int32_t)(d * Lu + i));
      std::vector<int32_t> &pv = pre[vj * (nx + 1) + vi];
      std::sort(pv.begin(), pv.end());
      for (int32_t j : pv) s.push_back((int32_t)(2 * Lu + j));
      if (s.empty()) continue;  // empty patches dropped (R8)
      for (int32_t x : s) P->mu[x] += 1;
      P->mp = std::max<int>(P->mp, (int)s.size());
      pat.push_back(std::move(s));
    }
  P->npatch = (int64_t)pat.size();
  P->pnodes.assign(P->npatch * P->mp, -1);
  P->psize.resize(P->npatch);
  for (int64_t p = 0; p < P->npatch; ++p) {
    P->psize[p] = (int32_t)pat[p].size();
    std::copy(pat[p].begin(), pat[p].end(), P->pnodes.begin() + p * P->mp);
  }
}

void plan_ns_interpolation(const NSPlan &C, const NSPlan &F, std::vector<int32_t> &rowptr,
                           std::vector<int32_t> &col, std::vector<double> &val) {
  auto scalar = [](const NSPlan &Q, bool vel) {
    PlanLevel S;
    S.nx = Q.nx;
    S.ny = Q.ny;
    S.Lx = vel ? Q.Lux : Q.Lpx;
    S.Ly = vel ? Q.Luy : Q.Lpy;
    S.nnode = (int64_t)S.Lx * S.Ly;
    S.con.assign(S.nnode, 0);
    if (vel)
      for (int64_t i = 0; i < S.nnode; ++i) S.con[i] = Q.con[i];
    return S;
  };
  std::vector<int32_t> urp, uci, prp, pci;
  std::vector<double> uv, pv;
  plan_interpolation(scalar(C, true), scalar(F, true), F.ku, urp, uci, uv);
  plan_interpolation(scalar(C, false), scalar(F, false), F.kp, prp, pci, pv);
  rowptr.assign(F.ns + 1, 0);
  col.clear();
  val.clear();
  int64_t r = 0;
  for (int blk = 0; blk < 3; ++blk) {
    const bool vel = blk < 2;
    const std::vector<int32_t> &rp = vel ? urp : prp, &ci = vel ? uci : pci;
    const std::vector<double> &vv = vel ? uv : pv;
    const int64_t off = blk * C.Lu;  // coarse sid offset (pressure block starts at 2 C.Lu)
    const int64_t nrow = vel ? F.Lu : F.Lp;
    for (int64_t i = 0; i < nrow; ++i, ++r) {
      for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
        col.push_back((int32_t)(off + ci[e]));
        val.push_back(vv[e]);
      }
      rowptr[r + 1] = (int32_t)col.size();
    }
  }
}

}  // namespace wrmg
