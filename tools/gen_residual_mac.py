"""Generate paper_2407_13997_b200/csrc/residual_mac_gen.h: the compile-time
stencil geometry of the macro-block space-time residual (kernels_residual_mac.cu).

Pure lattice geometry, no arithmetic of the method: on the anti-diagonal mesh of
PAPER.md:524-525 (square [i, i+1] x [j, j+1] cut from (i+1, j) to (i, j+1)) the
P_k nodes are the lattice points (k i + a, k j + b); two nodes are coupled by the
mass and stiffness matrices (eq. heatfem) iff they lie in a
common triangle.  A macro block is the k x k nodes (k i + a, k j + b), 0 <= a, b
< k; its k^2 rows have 7 (P1), 46 (P2: 19 + 3 * 9) and 153 (P3) stencil entries
on the interior lattice but touch only 7 / 22 / 43 distinct nodes, so the kernel
loads each of those once per (macro, time chunk) and feeds every row that uses it.

Emitted per k:
  kMacCnt<k>[t]        entries of row type t = b k + a (interior stencil)
  kMacOff<k>[t][e]     (dx, dy) of entry e of type t, ordered by (dy, dx)
  kMacBase<k>[t]       offset of type t in the flat coefficient arrays
  mac_accum_k<k>(...)  fully unrolled: for each union node (dx, dy) relative to the
                       macro origin, one shared-memory load and the FMAs of every
                       (row, entry) that uses it.  Group g = (dy + k) / k selects the
                       staged line group (three groups of k node lines), line l =
                       (dy + k) % k, column x = dx + k of the staged window.
Usage: python tools/gen_residual_mac.py > paper_2407_13997_b200/csrc/residual_mac_gen.h
"""
import sys


def tri_nodes(k, i, j, up):
    s = set()
    for a in range(k + 1):
        for b in range(k + 1):
            if (not up and a + b <= k) or (up and a + b >= k):
                s.add((k * i + a, k * j + b))
    return s


def stencil(k, X, Y):
    nb = set()
    for i in range(X // k - 2, X // k + 3):
        for j in range(Y // k - 2, Y // k + 3):
            for up in (0, 1):
                t = tri_nodes(k, i, j, up)
                if (X, Y) in t:
                    nb |= t
    return sorted(((x - X, y - Y) for x, y in nb), key=lambda d: (d[1], d[0]))


def emit(k, out):
    types = [(a, b) for b in range(k) for a in range(k)]
    st = [stencil(k, k * 10 + a, k * 10 + b) for (a, b) in types]
    base, acc = [], 0
    for s in st:
        base.append(acc)
        acc += len(s)
    maxe = max(len(s) for s in st)
    out.append(f"// ---- P{k}: {k * k} row types, {acc} stencil entries")
    out.append(f"constexpr int kMacTypes{k} = {k * k};")
    out.append(f"constexpr int kMacEntries{k} = {acc};")
    out.append(f"constexpr int kMacMaxE{k} = {maxe};")
    out.append(f"constexpr int kMacCnt{k}[{k * k}] = {{{', '.join(str(len(s)) for s in st)}}};")
    out.append(f"constexpr int kMacBase{k}[{k * k}] = {{{', '.join(map(str, base))}}};")
    rows = []
    for s in st:
        cells = ", ".join(f"{{{dx}, {dy}}}" for dx, dy in s)
        pad = ", ".join(["{0, 0}"] * (maxe - len(s)))
        rows.append("{" + cells + (", " + pad if pad else "") + "}")
    out.append(f"constexpr int8_t kMacOff{k}[{k * k}][{maxe}][2] = {{")
    out.append(",\n".join("    " + r for r in rows))
    out.append("};")
    # union nodes relative to the macro origin, and who uses them
    users = {}
    for t, ((a, b), s) in enumerate(zip(types, st)):
        for e, (dx, dy) in enumerate(s):
            users.setdefault((a + dx, b + dy), []).append((t, base[t] + e))
    order = sorted(users, key=lambda p: (p[1], p[0]))
    out.append(f"// {len(order)} distinct nodes feed the {acc} entries")
    out.append(f"template <int RWX, int VPC, class Coef>")
    out.append(f"__device__ __forceinline__ void mac_accum_k{k}(const double *__restrict__ g0, "
               f"const double *__restrict__ g1, const double *__restrict__ g2, const Coef &C, "
               f"double (&am)[{k * k}], double (&ak)[{k * k}]) {{")
    for (x, y) in order:
        g, l = (y + k) // k, (y + k) % k
        assert 0 <= g <= 2 and -k <= x < 2 * k
        out.append(f"  {{ const double v = g{g}[({l} * RWX + {x + k}) * VPC];")
        for (t, idx) in users[(x, y)]:
            out.append(f"    am[{t}] = fma(C.m[{idx}], v, am[{t}]); ak[{t}] = fma(C.k[{idx}], v, ak[{t}]);")
        out.append("  }")
    out.append("}")
    out.append("")
    # L1 variant: values through a loader functor ld(line, column) of the (3k lines) x (3k columns)
    # window around the macro (line = dy + k, column = dx + k), any value type V with vfma
    out.append("template <class LD, class Coef, class V>")
    out.append(f"__device__ __forceinline__ void mac_accum_ld_k{k}(const LD &ld, const Coef &C, "
               f"V (&am)[{k * k}], V (&ak)[{k * k}]) {{")
    for (x, y) in order:
        out.append(f"  {{ const V v = ld({y + k}, {x + k});")
        for (t, idx) in users[(x, y)]:
            out.append(f"    vfma(am[{t}], C.m[{idx}], v); vfma(ak[{t}], C.k[{idx}], v);")
        out.append("  }")
    out.append("}")
    out.append("")
    # row-split variant: part 0 = the rows of macro line b = 0, part 1 = lines b >= 1 (two
    # warps share a macro block; each loads only the union of its own rows' stencils)
    if k > 1:
        for part in (0, 1):
            rows = [t for t, (a, b) in enumerate(types) if (b == 0) == (part == 0)]
            sub = {}
            for t in rows:
                a, b = types[t]
                for e, (dx, dy) in enumerate(st[t]):
                    sub.setdefault((a + dx, b + dy), []).append((t, base[t] + e))
            sorder = sorted(sub, key=lambda p: (p[1], p[0]))
            out.append(f"// part {part}: rows {rows}, {len(sorder)} distinct nodes")
            out.append("template <class LD, class Coef, class V>")
            out.append(f"__device__ __forceinline__ void mac_accum_ld_k{k}_p{part}(const LD &ld, const Coef &C, "
                       f"V (&am)[{k * k}], V (&ak)[{k * k}]) {{")
            for (x, y) in sorder:
                out.append(f"  {{ const V v = ld({y + k}, {x + k});")
                for (t, idx) in sub[(x, y)]:
                    out.append(f"    vfma(am[{t}], C.m[{idx}], v); vfma(ak[{t}], C.k[{idx}], v);")
                out.append("  }")
            out.append("}")
            out.append("")


def main():
    out = ["// GENERATED by tools/gen_residual_mac.py -- do not edit.",
           "// Interior P_k stencils of the anti-diagonal lattice (PAPER.md:524-525) and the",
           "// unrolled macro-block accumulation of kernels_residual_mac.cu.",
           "#pragma once", "#include <cstdint>", "", "namespace wrmg {", ""]
    for k in (1, 2, 3):
        emit(k, out)
    out.append("}  // namespace wrmg")
    sys.stdout.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
