// Structured P_k lattice of the anti-diagonal triangulation (PAPER.md:524-525:
// squares "cut into 2 triangles each from bottom-right to top-left").
//
// Cells.  Square (ci, cj) has a lower triangle (t = 0) with vertices
// (ci,cj), (ci+1,cj), (ci,cj+1) and an upper triangle (t = 1) with vertices
// (ci+1,cj+1), (ci,cj+1), (ci+1,cj).  With that vertex order both are the image
// of the reference triangle under x = v0 +/- h xi, so they share the reference
// matrices: M_e = h^2 M^, K_e = K^.
// Local node (a, b) (a + b <= k) of triangle t sits at lattice point
//     t = 0: (k ci + a, k cj + b)        t = 1: (k (ci+1) - a, k (cj+1) - b).
// Local index: b outer, a inner: idx(a, b) = b (k + 1) - b (b - 1) / 2 + a.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define WRMG_HD __host__ __device__ __forceinline__
#else
#define WRMG_HD inline
#endif

namespace wrmg {

WRMG_HD int loc_index(int k, int a, int b) { return b * (k + 1) - b * (b - 1) / 2 + a; }

// Lattice point of local node (a, b) of triangle t in square (ci, cj).
WRMG_HD void loc_to_lattice(int k, int ci, int cj, int t, int a, int b, int *I, int *J) {
  if (t == 0) {
    *I = k * ci + a;
    *J = k * cj + b;
  } else {
    *I = k * (ci + 1) - a;
    *J = k * (cj + 1) - b;
  }
}

// Enumerate the (at most 6) triangles containing lattice node (I, J) in a fixed
// order (cj, ci ascending; lower before upper).  For each, writes the square,
// the triangle and the node's local (a, b).  Returns the count.
WRMG_HD int cells_of_node(int k, int nx, int ny, int I, int J, int *ci, int *cj, int *t, int *la, int *lb) {
  int n = 0;
  int ci0 = (I - 1) / k, cj0 = (J - 1) / k;  // I >= 1 ... candidate range below
  if (I == 0) ci0 = 0;
  if (J == 0) cj0 = 0;
  for (int y = cj0; y <= J / k && y < ny; ++y) {
    if (y < 0) continue;
    for (int x = ci0; x <= I / k && x < nx; ++x) {
      if (x < 0) continue;
      int a = I - k * x, b = J - k * y;
      if (a >= 0 && b >= 0 && a + b <= k) {
        ci[n] = x; cj[n] = y; t[n] = 0; la[n] = a; lb[n] = b; ++n;
      }
      a = k * (x + 1) - I;
      b = k * (y + 1) - J;
      if (a >= 0 && b >= 0 && a + b <= k) {
        ci[n] = x; cj[n] = y; t[n] = 1; la[n] = a; lb[n] = b; ++n;
      }
    }
  }
  return n;
}

// Vertices (in cell units) of the smallest closed mesh entity containing
// lattice node (I, J): a vertex (1), an edge (2) or a triangle (3).  The node
// belongs to the open vertex star of exactly these vertices.
WRMG_HD int entity_vertices(int k, int I, int J, int *vi, int *vj) {
  int ci = I / k, a = I % k, cj = J / k, b = J % k;
  if (a == 0 && b == 0) {
    vi[0] = ci; vj[0] = cj;
    return 1;
  }
  if (b == 0) {  // horizontal edge
    vi[0] = ci; vj[0] = cj; vi[1] = ci + 1; vj[1] = cj;
    return 2;
  }
  if (a == 0) {  // vertical edge
    vi[0] = ci; vj[0] = cj; vi[1] = ci; vj[1] = cj + 1;
    return 2;
  }
  if (a + b == k) {  // diagonal, bottom-right to top-left
    vi[0] = ci + 1; vj[0] = cj; vi[1] = ci; vj[1] = cj + 1;
    return 2;
  }
  if (a + b < k) {  // lower triangle interior
    vi[0] = ci; vj[0] = cj; vi[1] = ci + 1; vj[1] = cj; vi[2] = ci; vj[2] = cj + 1;
    return 3;
  }
  vi[0] = ci + 1; vj[0] = cj + 1; vi[1] = ci; vj[1] = cj + 1; vi[2] = ci + 1; vj[2] = cj;
  return 3;
}

}  // namespace wrmg
