// Eigenvalues of a real upper Hessenberg matrix by the Francis double-shift QR
// iteration (the classical EISPACK hqr algorithm), host side: the Chebyshev
// smoother's largest-eigenvalue estimate takes the largest |Ritz value| of the
// Arnoldi Hessenberg (DESIGN.md R-cheb).
#include <cmath>
#include <vector>

namespace wrmg {

// a: n x n row-major upper Hessenberg (destroyed).  Returns false if an
// eigenvalue failed to converge in 60 iterations.
bool hessenberg_eigenvalues(std::vector<double> &a, int n, std::vector<double> &wr, std::vector<double> &wi) {
  auto A = [&](int i, int j) -> double & { return a[(size_t)i * n + j]; };
  auto sgn = [](double x, double y) { return y >= 0.0 ? std::fabs(x) : -std::fabs(x); };
  wr.assign(n, 0.0);
  wi.assign(n, 0.0);
  double anorm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::fabs(A(i, j));
  int nn = n - 1;
  double t = 0.0;
  while (nn >= 0) {
    int its = 0, l;
    do {
      for (l = nn; l >= 1; --l) {
        double s = std::fabs(A(l - 1, l - 1)) + std::fabs(A(l, l));
        if (s == 0.0) s = anorm;
        if (std::fabs(A(l, l - 1)) + s == s) {
          A(l, l - 1) = 0.0;
          break;
        }
      }
      double x = A(nn, nn);
      if (l == nn) {  // one root
        wr[nn] = x + t;
        wi[nn] = 0.0;
        --nn;
      } else {
        double y = A(nn - 1, nn - 1), w = A(nn, nn - 1) * A(nn - 1, nn);
        if (l == nn - 1) {  // two roots
          double p = 0.5 * (y - x), q = p * p + w, z = std::sqrt(std::fabs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sgn(z, p);
            wr[nn - 1] = wr[nn] = x + z;
            if (z != 0.0) wr[nn] = x - w / z;
            wi[nn - 1] = wi[nn] = 0.0;
          } else {
            wr[nn - 1] = wr[nn] = x + p;
            wi[nn - 1] = -z;
            wi[nn] = z;
          }
          nn -= 2;
        } else {  // no roots yet: double-shift QR sweep on rows l .. nn
          if (its == 60) return false;
          if (its == 10 || its == 20) {  // exceptional shift
            t += x;
            for (int i = 0; i <= nn; ++i) A(i, i) -= x;
            const double s = std::fabs(A(nn, nn - 1)) + std::fabs(A(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          int m;
          double p = 0, q = 0, r = 0, z;
          for (m = nn - 2; m >= l; --m) {
            z = A(m, m);
            r = x - z;
            double s = y - z;
            p = (r * s - w) / A(m + 1, m) + A(m, m + 1);
            q = A(m + 1, m + 1) - z - r - s;
            r = A(m + 2, m + 1);
            s = std::fabs(p) + std::fabs(q) + std::fabs(r);
            p /= s;
            q /= s;
            r /= s;
            if (m == l) break;
            const double u = std::fabs(A(m, m - 1)) * (std::fabs(q) + std::fabs(r));
            const double v = std::fabs(p) * (std::fabs(A(m - 1, m - 1)) + std::fabs(z) + std::fabs(A(m + 1, m + 1)));
            if (u + v == v) break;
          }
          for (int i = m + 2; i <= nn; ++i) {
            A(i, i - 2) = 0.0;
            if (i != m + 2) A(i, i - 3) = 0.0;
          }
          for (int k = m; k <= nn - 1; ++k) {
            if (k != m) {
              p = A(k, k - 1);
              q = A(k + 1, k - 1);
              r = 0.0;
              if (k != nn - 1) r = A(k + 2, k - 1);
              if ((x = std::fabs(p) + std::fabs(q) + std::fabs(r)) != 0.0) {
                p /= x;
                q /= x;
                r /= x;
              }
            }
            const double s = sgn(std::sqrt(p * p + q * q + r * r), p);
            if (s != 0.0) {
              if (k == m) {
                if (l != m) A(k, k - 1) = -A(k, k - 1);
              } else {
                A(k, k - 1) = -s * x;
              }
              p += s;
              x = p / s;
              y = q / s;
              z = r / s;
              q /= p;
              r /= p;
              for (int j = k; j <= nn; ++j) {
                p = A(k, j) + q * A(k + 1, j);
                if (k != nn - 1) {
                  p += r * A(k + 2, j);
                  A(k + 2, j) -= p * z;
                }
                A(k + 1, j) -= p * y;
                A(k, j) -= p * x;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; ++i) {
                p = x * A(i, k) + y * A(i, k + 1);
                if (k != nn - 1) {
                  p += z * A(i, k + 2);
                  A(i, k + 2) -= p * r;
                }
                A(i, k + 1) -= p * q;
                A(i, k) -= p;
              }
            }
          }
        }
      }
    } while (l < nn - 1);
  }
  return true;
}

}  // namespace wrmg
