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
#include <stdexcept>
#include <vector>

#include "lattice.h"
#include "ns.h"
#include "plan.h"
#include "strip.h"

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
  P->pvert.clear();
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
      P->pvert.push_back(vj * (nx + 1) + vi);
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

namespace {

// Column bookkeeping of one lattice (degree k) of a strip whose local mesh starts at cell cx0.
void strip_columns(int k, int gnx, int x0, int nx, int cx0, int nxl, int rank, int nranks, StripInfo *S) {
  StripInfo &s = *S;
  s = StripInfo{};
  s.rank = rank;
  s.nranks = nranks;
  s.gnx = gnx;
  s.x0 = x0;
  s.nx = nx;
  s.cx0 = cx0;
  s.nxl = nxl;
  s.G0 = k * cx0;
  s.own0 = (rank == 0 ? 0 : k * x0 + 1) - s.G0;
  s.own1 = k * (x0 + nx) - s.G0;
  if (rank > 0) {
    s.nlg = k;
    s.lg0 = k * x0 - k + 1 - s.G0;
    s.nsl = k;
    s.sl0 = k * x0 + 1 - s.G0;
  }
  if (rank < nranks - 1) {
    s.nrg = k;
    s.rg0 = k * (x0 + nx) + 1 - s.G0;
    s.nsr = k;
    s.sr0 = k * (x0 + nx) - k + 1 - s.G0;
  }
}

// Scalar lattice view (Lx, Ly, nnode) of one NS field for plan_strip_interpolation.
PlanLevel scalar_view(const NSPlan &Q, bool vel) {
  PlanLevel S;
  S.nx = Q.nx;
  S.ny = Q.ny;
  S.Lx = vel ? Q.Lux : Q.Lpx;
  S.Ly = vel ? Q.Luy : Q.Lpy;
  S.nnode = (int64_t)S.Lx * S.Ly;
  return S;
}

}  // namespace

void plan_ns_strip_level(int gnx, int gny, int x0, int nx, double h, int k, int bc, double lid_speed, int rank,
                         int nranks, NSPlan *P, StripInfo *su, StripInfo *sp) {
  NSPlan G;
  plan_ns_level(gnx, gny, h, k, bc, lid_speed, &G);
  const int cx0 = std::max(0, x0 - 1), cx1 = std::min(gnx, x0 + nx + 2), nxl = cx1 - cx0;
  const int ku = k + 1, kp = k;
  plan_ns_level(nxl, gny, h, k, bc, lid_speed, P);  // CSR pattern of the local mesh (edge rows truncated)
  strip_columns(ku, gnx, x0, nx, cx0, nxl, rank, nranks, su);
  strip_columns(kp, gnx, x0, nx, cx0, nxl, rank, nranks, sp);
  const int G0u = su->G0, G0p = sp->G0;
  // local sid of a global sid (-1 outside the local lattices)
  auto loc = [&](int64_t g) -> int64_t {
    if (g < 2 * G.Lu) {
      const int64_t d = g / G.Lu, i = g - d * G.Lu;
      const int I = (int)(i % G.Lux) - G0u, J = (int)(i / G.Lux);
      if (I < 0 || I >= P->Lux) return -1;
      return d * P->Lu + (int64_t)J * P->Lux + I;
    }
    const int64_t j = g - 2 * G.Lu;
    const int I = (int)(j % G.Lpx) - G0p, J = (int)(j / G.Lpx);
    if (I < 0 || I >= P->Lpx) return -1;
    return 2 * P->Lu + (int64_t)J * P->Lpx + I;
  };
  // global sid of a local sid
  auto glob = [&](int64_t l) -> int64_t {
    if (l < 2 * P->Lu) {
      const int64_t d = l / P->Lu, i = l - d * P->Lu;
      const int I = (int)(i % P->Lux) + G0u, J = (int)(i / P->Lux);
      return d * G.Lu + (int64_t)J * G.Lux + I;
    }
    const int64_t j = l - 2 * P->Lu;
    const int I = (int)(j % P->Lpx) + G0p, J = (int)(j / P->Lpx);
    return 2 * G.Lu + (int64_t)J * G.Lpx + I;
  };
  int64_t ncon = 0;
  for (int64_t l = 0; l < P->ns; ++l) {
    const int64_t g = glob(l);
    P->con[l] = G.con[g];
    P->g[l] = G.g[g];
    P->mu[l] = G.mu[g];
    ncon += P->con[l];
  }
  P->nfree = P->ns - ncon;
  const int vlo = rank == 0 ? 0 : x0 + 1, vhi = x0 + nx;
  std::vector<std::vector<int32_t>> pat;
  std::vector<int32_t> pv;
  int mp = 0;
  for (int64_t p = 0; p < G.npatch; ++p) {
    const int vi = G.pvert[p] % (gnx + 1);
    if (vi < vlo || vi > vhi) continue;
    std::vector<int32_t> s;
    for (int e = 0; e < G.psize[p]; ++e) {
      const int64_t l = loc(G.pnodes[p * G.mp + e]);
      if (l < 0) throw std::runtime_error("plan_ns_strip_level: patch outside the local lattice");
      s.push_back((int32_t)l);
    }
    mp = std::max<int>(mp, (int)s.size());
    pv.push_back(G.pvert[p]);
    pat.push_back(std::move(s));
  }
  P->mp = mp;
  P->npatch = (int64_t)pat.size();
  P->pvert.swap(pv);
  P->pnodes.assign(P->npatch * P->mp, -1);
  P->psize.resize(P->npatch);
  for (int64_t p = 0; p < P->npatch; ++p) {
    P->psize[p] = (int32_t)pat[p].size();
    std::copy(pat[p].begin(), pat[p].end(), P->pnodes.begin() + p * P->mp);
  }
  (void)ku;
  (void)kp;
}

void plan_ns_strip_interpolation(const NSPlan &C, const StripInfo &Scu, const StripInfo &Scp, const NSPlan &F,
                                 const StripInfo &Sfu, const StripInfo &Sfp, int gny_f, std::vector<int32_t> &rowptr,
                                 std::vector<int32_t> &col, std::vector<double> &val) {
  std::vector<int32_t> urp, uci, prp, pci;
  std::vector<double> uv, pv;
  plan_strip_interpolation(scalar_view(C, true), Scu, scalar_view(F, true), Sfu, F.ku, gny_f, urp, uci, uv, false);
  plan_strip_interpolation(scalar_view(C, false), Scp, scalar_view(F, false), Sfp, F.kp, gny_f, prp, pci, pv, true);
  rowptr.assign(F.ns + 1, 0);
  col.clear();
  val.clear();
  int64_t r = 0;
  for (int blk = 0; blk < 3; ++blk) {
    const bool vel = blk < 2;
    const std::vector<int32_t> &rp = vel ? urp : prp, &ci = vel ? uci : pci;
    const std::vector<double> &vv = vel ? uv : pv;
    const int64_t off = blk * C.Lu;
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
