// Spatial strip partition of the heat hierarchy across ranks (
// DESIGN.md section 7).  Integer setup only.
//
// Rank r owns the cell columns [x0, x0 + nx) of a level's global mesh (gnx x gny
// cells) and the lattice node columns
//     rank 0:  [0, k (x0 + nx)]            rank r > 0:  (k x0, k (x0 + nx)]
// (an interface node column belongs to the left rank), the vertex-star patches
// of its vertex columns (same rule in cell units), and every slab of those DoFs.
// Its local lattice is the node lattice of the cells [x0 - 1, x0 + nx + 1)
// clipped to [0, gnx): one cell of overlap per interior side.  Local column c is
// global column G0 + c.  Ghost columns (k each, filled from the neighbour):
//     left  (r > 0):      global (k x0 - k, k x0]
//     right (r < P - 1):  global (k (x0 + nx), k (x0 + nx) + k]
// The residual of an owned row reads u only on owned and ghost columns; an owned
// patch touches owned and right-ghost columns; restriction from owned fine rows
// touches owned and left-ghost coarse columns; prolongation to owned fine rows
// reads owned and left-ghost coarse columns.
#pragma once
#include <cstdint>
#include <vector>

#include "plan.h"

namespace wrmg {

// StripInfo: internal.h.

// Plan one level's strip: the local PlanLevel (patches restricted to owned vertices,
// translation classes renumbered) and the column bookkeeping.
void plan_strip_level(int gnx, int gny, int x0, int nx, double h, int k, int rank, int nranks, PlanLevel *P,
                      StripInfo *S, bool neumann = false);

// P_h (correction form, R5, R12) with rows only for owned fine nodes; columns are
// local coarse lattice indices (Sc = a whole-lattice strip with G0 = 0: global ids,
// used for the hand-over to the replicated coarse levels).
void plan_strip_interpolation(const PlanLevel &C, const StripInfo &Sc, const PlanLevel &F, const StripInfo &Sf, int k,
                              int gny_f, std::vector<int32_t> &rowptr, std::vector<int32_t> &col,
                              std::vector<double> &val, bool neumann = false);

}  // namespace wrmg
