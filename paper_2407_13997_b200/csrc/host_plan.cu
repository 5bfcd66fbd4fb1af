// Host-side integer setup (H3 and CSR structure): lattice maps, sparsity
// patterns, Dirichlet masks, vertex-star patch tables, translation classes of
// patches, and the finite-element interpolation P_h between nested lattices.
// Runs once per wrmg_setup; no floating-point method arithmetic except the
// P_h basis evaluations (R12).
#include <algorithm>
#include <map>
#include <vector>

#include "lattice.h"
#include "plan.h"

namespace wrmg {

void plan_level(int nx, int ny, double h, int k, PlanLevel *P, bool neumann) {
  P->nx = nx;
  P->ny = ny;
  P->h = h;
  P->Lx = k * nx + 1;
  P->Ly = k * ny + 1;
  const int Lx = P->Lx, Ly = P->Ly;
  const int64_t nn = (int64_t)Lx * Ly;
  P->nnode = nn;
  // Dirichlet mask: every boundary lattice node (R5)
  P->con.assign(nn, 0);
  int64_t nfree = 0;
  for (int J = 0; J < Ly; ++J)
    for (int I = 0; I < Lx; ++I) {
      bool c = !neumann && (I == 0 || J == 0 || I == Lx - 1 || J == Ly - 1);  // Neumann: no constrained DoF
      P->con[(int64_t)J * Lx + I] = c;
      nfree += !c;
    }
  P->nfree = nfree;
  // CSR pattern: j ~ i iff they share a triangle
  P->rowptr.assign(nn + 1, 0);
  P->col.clear();
  P->col.reserve(nn * (k == 1 ? 7 : k == 2 ? 12 : 18));
  std::vector<int32_t> nb;
  for (int J = 0; J < Ly; ++J)
    for (int I = 0; I < Lx; ++I) {
      int ci[6], cj[6], t[6], la[6], lb[6];
      int nc = cells_of_node(k, nx, ny, I, J, ci, cj, t, la, lb);
      nb.clear();
      for (int c = 0; c < nc; ++c)
        for (int b = 0; b <= k; ++b)
          for (int a = 0; a + b <= k; ++a) {
            int I2, J2;
            loc_to_lattice(k, ci[c], cj[c], t[c], a, b, &I2, &J2);
            nb.push_back(J2 * Lx + I2);
          }
      std::sort(nb.begin(), nb.end());
      nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
      int64_t i = (int64_t)J * Lx + I;
      P->col.insert(P->col.end(), nb.begin(), nb.end());
      P->rowptr[i + 1] = (int32_t)P->col.size();
    }
  // vertex-star patches (R8): node -> vertices of its entity
  const int nv = (nx + 1) * (ny + 1);
  std::vector<std::vector<int32_t>> star(nv);
  for (int J = 0; J < Ly; ++J)
    for (int I = 0; I < Lx; ++I) {
      int64_t i = (int64_t)J * Lx + I;
      if (P->con[i]) continue;
      int vi[3], vj[3];
      int ne = entity_vertices(k, I, J, vi, vj);
      for (int e = 0; e < ne; ++e) star[vj[e] * (nx + 1) + vi[e]].push_back((int32_t)i);
    }
  P->mp = (k == 1) ? 1 : (k == 2) ? 7 : 19;
  int mpmax = 0;
  for (auto &s : star) mpmax = std::max<int>(mpmax, (int)s.size());
  if (mpmax > P->mp) P->mp = mpmax;  // cannot happen on this lattice; defensive
  P->pnodes.clear();
  P->psize.clear();
  P->pvert.clear();
  P->ptype.clear();
  P->type_rep.clear();
  std::map<std::vector<int32_t>, int> types;
  std::vector<int32_t> mu(nn, 0);
  for (int v = 0; v < nv; ++v) {
    auto &s = star[v];
    if (s.empty()) continue;  // empty patches dropped (R8)
    int64_t p = (int64_t)P->psize.size();
    int vi = v % (nx + 1), vj = v / (nx + 1);
    std::vector<int32_t> sig;
    sig.reserve(2 * s.size() + 20);
    for (int32_t i : s) {
      sig.push_back((int32_t)(i % Lx) - k * vi);
      sig.push_back((int32_t)(i / Lx) - k * vj);
      mu[i] += 1;
    }
    {  // the cells of the star enter the block too (P1 stars are one node; Neumann boundary stars differ)
      int ci[6], cj[6], t[6], la[6], lb[6];
      const int nc = cells_of_node(k, nx, ny, k * vi, k * vj, ci, cj, t, la, lb);
      sig.push_back(-1000 - nc);
      for (int c = 0; c < nc; ++c) {
        sig.push_back(ci[c] - vi);
        sig.push_back(cj[c] - vj);
        sig.push_back(t[c]);
      }
    }
    auto it = types.find(sig);
    int ty;
    if (it == types.end()) {
      ty = (int)types.size();
      types.emplace(sig, ty);
      P->type_rep.push_back((int32_t)p);
    } else {
      ty = it->second;
    }
    P->ptype.push_back(ty);
    P->pvert.push_back(v);
    P->psize.push_back((int32_t)s.size());
    for (int j = 0; j < P->mp; ++j) P->pnodes.push_back(j < (int)s.size() ? s[j] : -1);
  }
  P->npatch = (int64_t)P->psize.size();
  P->ntypes = (int)types.size();
  P->mu = mu;
  // stencil classes of free rows: (I mod k, J mod k, which of the candidate cells exist)
  std::map<std::vector<int32_t>, int> cls;
  P->rcls.assign(nn, kRowConstrained);
  P->cls_rep.clear();
  for (int J = 0; J < Ly; ++J)
    for (int I = 0; I < Lx; ++I) {
      int64_t i = (int64_t)J * Lx + I;
      if (P->con[i]) continue;
      int ci[6], cj[6], t[6], la[6], lb[6];
      int nc = cells_of_node(k, nx, ny, I, J, ci, cj, t, la, lb);
      std::vector<int32_t> sig = {I % k, J % k};
      for (int c = 0; c < nc; ++c) {
        sig.push_back(ci[c] * k - I);
        sig.push_back(cj[c] * k - J);
        sig.push_back(t[c]);
      }
      auto it = cls.find(sig);
      int id;
      if (it == cls.end()) {
        id = (int)cls.size();
        cls.emplace(sig, id);
        P->cls_rep.push_back((int32_t)i);
      } else {
        id = it->second;
      }
      P->rcls[i] = id < (int)kRowGeneric ? (uint8_t)id : kRowGeneric;
    }
}

void plan_sweep_ctas(const PlanLevel &P, int pp, std::vector<int32_t> &cta_patch, std::vector<int32_t> &cta_type,
                     int exclude, const std::vector<uint8_t> *colour, int want) {
  cta_patch.clear();
  cta_type.clear();
  std::vector<std::vector<int32_t>> by(P.ntypes);
  for (int64_t p = 0; p < P.npatch; ++p)
    if (!colour || (*colour)[p] == want) by[P.ptype[p]].push_back((int32_t)p);
  for (int t = 0; t < P.ntypes; ++t)
    if (t != exclude)
    for (size_t s = 0; s < by[t].size(); s += pp) {
      cta_type.push_back(t);
      for (int j = 0; j < pp; ++j) cta_patch.push_back(s + j < by[t].size() ? by[t][s + j] : -1);
    }
}

// P_h from coarse (ncx x ncy, lattice Lxc) to fine (2ncx x 2ncy): row i (fine
// node) holds the coarse basis functions evaluated at node i (R12).  Correction
// form: constrained fine rows and constrained coarse columns dropped (R5).
void plan_interpolation(const PlanLevel &C, const PlanLevel &F, int k, std::vector<int32_t> &rowptr,
                        std::vector<int32_t> &col, std::vector<double> &val) {
  rowptr.assign(F.nnode + 1, 0);
  col.clear();
  val.clear();
  double phi[16];
  const int twok = 2 * k;
  for (int J = 0; J < F.Ly; ++J)
    for (int I = 0; I < F.Lx; ++I) {
      int64_t i = (int64_t)J * F.Lx + I;
      if (!F.con[i]) {
        // coarse square containing the fine node; lattice units of the coarse mesh scaled by 2k
        int ci = std::min(I / twok, C.nx - 1), cj = std::min(J / twok, C.ny - 1);
        int ra = I - twok * ci, rb = J - twok * cj;  // 0..2k
        int t = 0;
        // k * lambda = (2k*xi) / 2: exact halves
        double kl1 = 0.5 * ra, kl2 = 0.5 * rb;
        if (ra + rb > twok) {  // upper triangle: xi' = 1 - xi, eta' = 1 - eta
          t = 1;
          kl1 = 0.5 * (twok - ra);
          kl2 = 0.5 * (twok - rb);
        }
        eval_basis_klambda(k, kl1, kl2, phi);
        std::vector<std::pair<int32_t, double>> ent;
        for (int b = 0; b <= k; ++b)
          for (int a = 0; a + b <= k; ++a) {
            double v = phi[loc_index(k, a, b)];
            if (v == 0.0 || std::abs(v) < 1e-14) continue;
            int I2, J2;
            loc_to_lattice(k, ci, cj, t, a, b, &I2, &J2);
            int32_t jc = J2 * C.Lx + I2;
            if (C.con[jc]) continue;
            ent.push_back({jc, v});
          }
        std::sort(ent.begin(), ent.end());
        for (auto &e : ent) {
          col.push_back(e.first);
          val.push_back(e.second);
        }
      }
      rowptr[i + 1] = (int32_t)col.size();
    }
}

void transpose_csr(int64_t nrow, int64_t ncol, const std::vector<int32_t> &rp, const std::vector<int32_t> &ci,
                   const std::vector<double> &v, std::vector<int32_t> &trp, std::vector<int32_t> &tci,
                   std::vector<double> &tv) {
  trp.assign(ncol + 1, 0);
  for (int32_t c : ci) trp[c + 1]++;
  for (int64_t j = 0; j < ncol; ++j) trp[j + 1] += trp[j];
  tci.assign(ci.size(), 0);
  tv.assign(v.size(), 0.0);
  std::vector<int32_t> pos(trp.begin(), trp.end() - 1);
  for (int64_t i = 0; i < nrow; ++i)
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
      int32_t d = pos[ci[e]]++;
      tci[d] = (int32_t)i;
      tv[d] = v[e];  // identical doubles: R = P^T bitwise (R12)
    }
}

std::vector<int> level_sizes(int gnx, int gny, int ncoarse, std::vector<int> *nys) {
  std::vector<int> nxs;
  nys->clear();
  int nx = gnx, ny = gny;
  nxs.push_back(nx);
  nys->push_back(ny);
  while (std::min(nx, ny) > ncoarse && nx % 2 == 0 && ny % 2 == 0) {
    nx /= 2;
    ny /= 2;
    nxs.push_back(nx);
    nys->push_back(ny);
  }
  std::reverse(nxs.begin(), nxs.end());
  std::reverse(nys->begin(), nys->end());
  return nxs;
}

}  // namespace wrmg
