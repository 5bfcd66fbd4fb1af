// Symmetry-reduced Kronecker patch solves of the interior vertex-star class
// (host_sym.cu: setup; kernels_sweep_sym.cu: the sweep).
#pragma once
#include <cstdint>
#include <vector>

#include "internal.h"

namespace wrmg {

struct PlanLevel;

// Slot order of the interior class (perm[slot] = position in the class's pnodes row)
// and the orbit counts (n1, n2, n3); false if the class is not the symmetric interior star.
bool plan_sym_class(const PlanLevel &P, int k, int cls, std::vector<int32_t> &perm, int counts[3]);
// Block-diagonalise M_p, K_p (slot order, mp x mp row-major) and solve the per-block
// generalised eigenproblems and the per-mode temporal inverses.  false if the blocks
// are not exactly decoupled (relative 1e-12) or a block is not positive definite.
bool sym_factor(int k, const double *Mp, const double *Kp, const Temporal &tm, SymTab *out);

}  // namespace wrmg
