// Navier-Stokes (Taylor-Hood P_{k+1}-P_k x DG(q)) host plan and constants.
//
// Spatial unknown ids ("sids", R4, field order u_x, u_y, p):
//     u_x node i -> i,   u_y node i -> Lu + i,   p node j -> 2 Lu + j,
// i on the (ku nx + 1) x (ku ny + 1) velocity lattice (ku = k + 1), j on the
// (kp nx + 1) x (kp ny + 1) pressure lattice (kp = k).  Vectors are
// waveform-major over sids: v[(sid * N + n) (q + 1) + a].
#pragma once
#include <cstdint>
#include <vector>

#include "internal.h"

namespace wrmg {

constexpr int kMaxLocU = 10;  // P3 velocity
constexpr int kMaxLocP = 6;   // P2 pressure

// Reference-triangle integrals of the Taylor-Hood pair (x = v0 + h xi; the
// physical values follow from the scalings in kernels_ns.cu):
//   Mh[i][j]       = int v_i v_j              Kh[i][j] = int grad v_i . grad v_j
//   Gh[d][i][j]    = int chi_j d_d v_i        (i velocity, j pressure)
//   Th[d][i][l][j] = int v_i v_l d_d v_j      (convection, eq. nsfem)
struct THElement {
  int ku = 0, kp = 0, nu = 0, np = 0;
  double Mh[kMaxLocU * kMaxLocU];
  double Kh[kMaxLocU * kMaxLocU];
  double Gh[2 * kMaxLocU * kMaxLocP];
  double Th[2 * kMaxLocU * kMaxLocU * kMaxLocU];
};
void build_th_element(int k, THElement *E);

struct NSPlan {
  int nx = 0, ny = 0, ku = 0, kp = 0;
  double h = 0;
  int Lux = 0, Luy = 0, Lpx = 0, Lpy = 0;
  int64_t Lu = 0, Lp = 0, ns = 0, nfree = 0;
  std::vector<uint8_t> con;      // per sid: Dirichlet velocity (R5)
  std::vector<double> g;         // per sid: boundary value (lid, R5)
  std::vector<int32_t> rowptr, col;  // sid CSR pattern; velocity columns first in every row
  std::vector<int32_t> vvptr;    // 2 Lu + 1: compact index of the velocity-velocity entries of each velocity row
  int mp = 0;                    // largest Vanka+star patch
  int64_t npatch = 0;
  std::vector<int32_t> pnodes, psize, mu;  // [npatch][mp] sids (-1 pad), sizes, multiplicity per sid
};

void plan_ns_level(int nx, int ny, double h, int k, int bc, double lid_speed, NSPlan *P);
// Block-diagonal P_h = diag(Pu, Pu, Pp) in correction form (R5, R12).
void plan_ns_interpolation(const NSPlan &C, const NSPlan &F, std::vector<int32_t> &rowptr,
                           std::vector<int32_t> &col, std::vector<double> &val);

}  // namespace wrmg
