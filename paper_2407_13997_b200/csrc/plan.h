// Host-side plan of one multigrid level (integer setup data).
#pragma once
#include <cstdint>
#include <vector>

#include "internal.h"

namespace wrmg {

struct PlanLevel {
  int nx = 0, ny = 0, Lx = 0, Ly = 0;
  double h = 0;
  int64_t nnode = 0, nfree = 0;
  std::vector<uint8_t> con;
  std::vector<int32_t> rowptr, col;  // spatial sparsity (all nodes)
  int mp = 0;                        // padded patch size
  int64_t npatch = 0;
  int ntypes = 0;
  std::vector<int32_t> pnodes, psize, pvert, ptype, type_rep, mu;
  // residual stencil classes: rows with identical geometry share (offsets, values)
  std::vector<uint8_t> rcls;         // per row: class id, kRowConstrained, kRowGeneric
  std::vector<int32_t> cls_rep;      // representative row per class
};

constexpr uint8_t kRowConstrained = 255;
constexpr uint8_t kRowGeneric = 254;

// Type-grouped CTA work list for the Kronecker sweep: ncta x pp patch ids (-1 pad).
// Patches of class `exclude` (>= 0) are left out (they run in the symmetry-reduced sweep).
// colour: only patches whose (*colour)[p] == want.
void plan_sweep_ctas(const PlanLevel &P, int pp, std::vector<int32_t> &cta_patch, std::vector<int32_t> &cta_type,
                     int exclude = -1, const std::vector<uint8_t> *colour = nullptr, int want = -1);

void plan_level(int nx, int ny, double h, int k, PlanLevel *P, bool neumann = false);
void plan_interpolation(const PlanLevel &C, const PlanLevel &F, int k, std::vector<int32_t> &rowptr,
                        std::vector<int32_t> &col, std::vector<double> &val);
void transpose_csr(int64_t nrow, int64_t ncol, const std::vector<int32_t> &rp, const std::vector<int32_t> &ci,
                   const std::vector<double> &v, std::vector<int32_t> &trp, std::vector<int32_t> &tci,
                   std::vector<double> &tv);
std::vector<int> level_sizes(int gnx, int gny, int ncoarse, std::vector<int> *nys);

}  // namespace wrmg
