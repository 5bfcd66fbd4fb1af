// Host plan of the spatial strip partition (strip.h).
#include <algorithm>
#include <map>
#include <vector>

#include "lattice.h"
#include "strip.h"

namespace wrmg {

void plan_strip_level(int gnx, int gny, int x0, int nx, double h, int k, int rank, int nranks, PlanLevel *P,
                      StripInfo *S, bool neumann) {
  StripInfo &s = *S;
  s = StripInfo{};
  s.rank = rank;
  s.nranks = nranks;
  s.gnx = gnx;
  s.x0 = x0;
  s.nx = nx;
  s.cx0 = x0 > 0 ? x0 - 1 : 0;
  const int cx1 = std::min(gnx, x0 + nx + 1);
  s.nxl = cx1 - s.cx0;
  s.G0 = k * s.cx0;
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
  plan_level(s.nxl, gny, h, k, P, neumann);
  // keep the patches of owned vertices only; renumber the translation classes
  const int vlo = (rank == 0 ? 0 : x0 + 1) - s.cx0, vhi = x0 + nx - s.cx0;
  const int nvx = s.nxl + 1;
  std::vector<int32_t> pn, ps, pv, pt, rep;
  std::map<int32_t, int32_t> remap;
  int64_t np = 0;
  for (int64_t p = 0; p < P->npatch; ++p) {
    const int vc = P->pvert[p] % nvx;
    if (vc < vlo || vc > vhi) continue;
    auto it = remap.find(P->ptype[p]);
    int32_t t;
    if (it == remap.end()) {
      t = (int32_t)remap.size();
      remap.emplace(P->ptype[p], t);
      rep.push_back((int32_t)np);
    } else {
      t = it->second;
    }
    pt.push_back(t);
    pv.push_back(P->pvert[p]);
    ps.push_back(P->psize[p]);
    pn.insert(pn.end(), P->pnodes.begin() + p * P->mp, P->pnodes.begin() + (p + 1) * P->mp);
    ++np;
  }
  P->pnodes.swap(pn);
  P->psize.swap(ps);
  P->pvert.swap(pv);
  P->ptype.swap(pt);
  P->type_rep.swap(rep);
  P->npatch = np;
  P->ntypes = (int)remap.size();
}

void plan_strip_interpolation(const PlanLevel &C, const StripInfo &Sc, const PlanLevel &F, const StripInfo &Sf, int k,
                              int gny_f, std::vector<int32_t> &rowptr, std::vector<int32_t> &col,
                              std::vector<double> &val, bool neumann) {
  rowptr.assign(F.nnode + 1, 0);
  col.clear();
  val.clear();
  double phi[16];
  const int twok = 2 * k;
  const int gLxf = k * Sf.gnx + 1, gLy = k * gny_f + 1;
  const int gncx = Sc.gnx, gncy = gny_f / 2;
  for (int J = 0; J < F.Ly; ++J)
    for (int I = 0; I < F.Lx; ++I) {
      const int64_t i = (int64_t)J * F.Lx + I;
      const int Ig = I + Sf.G0;
      const bool owned = I >= Sf.own0 && I <= Sf.own1;
      const bool gcon = !neumann && (Ig == 0 || Ig == gLxf - 1 || J == 0 || J == gLy - 1);  // Dirichlet (R5)
      if (owned && !gcon) {
        const int ci = std::min(Ig / twok, gncx - 1), cj = std::min(J / twok, gncy - 1);
        const int ra = Ig - twok * ci, rb = J - twok * cj;
        int t = 0;
        double kl1 = 0.5 * ra, kl2 = 0.5 * rb;
        if (ra + rb > twok) {
          t = 1;
          kl1 = 0.5 * (twok - ra);
          kl2 = 0.5 * (twok - rb);
        }
        eval_basis_klambda(k, kl1, kl2, phi);
        std::vector<std::pair<int32_t, double>> ent;
        for (int b = 0; b <= k; ++b)
          for (int a = 0; a + b <= k; ++a) {
            const double v = phi[loc_index(k, a, b)];
            if (v == 0.0 || std::abs(v) < 1e-14) continue;
            int I2, J2;
            loc_to_lattice(k, ci, cj, t, a, b, &I2, &J2);  // global coarse lattice
            const int gLxc = k * gncx + 1, gLyc = k * gncy + 1;
            if (!neumann && (I2 == 0 || I2 == gLxc - 1 || J2 == 0 || J2 == gLyc - 1)) continue;  // constrained
            const int Il = I2 - Sc.G0;
            ent.push_back({J2 * C.Lx + Il, v});
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

}  // namespace wrmg
