// Gaunt coefficients for the Helmholtz translations (csrc/cuda/helm.cu):
//   G(n,m;n',m';l) = int Y_n^m conj(Y_n'^m') conj(Y_l^{m-m'}) dOmega
// for orthonormal Y without the Condon-Shortley phase, by Gauss-Legendre quadrature
// in cos(theta) -- exact, since the integrand is a polynomial of degree n+n'+l.
// Layout: G[(kin * KP + iout) * GL + li], kin = n^2+n+m, iout = n'^2+n'+m',
// l = |n - n'| + 2 li (the parity rule n+n'+l even), GL = P + 1.
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.hpp"

namespace qbxg {

namespace {
constexpr double kPi = 3.14159265358979323846;
inline int fidx(int n, int m) { return n * n + n + m; }

void pbar(int P, double x, std::vector<double>& T) {
  T.assign(size_t((P + 1) * (P + 1)), 0.0);
  const double s = std::sqrt(std::max(0.0, 1.0 - x * x));
  double mm = 1.0 / std::sqrt(4.0 * kPi);
  for (int m = 0; m <= P; ++m) {
    if (m > 0) mm *= std::sqrt((2.0 * m + 1.0) / (2.0 * m)) * s;
    double a = mm;
    T[fidx(m, m)] = a;
    if (m + 1 > P) continue;
    double b = std::sqrt(2.0 * m + 3.0) * x * a;
    T[fidx(m + 1, m)] = b;
    for (int n = m + 2; n <= P; ++n) {
      const double an = std::sqrt((4.0 * n * n - 1.0) / (double(n) * n - double(m) * m));
      const double bn = std::sqrt(((n - 1.0) * (n - 1.0) - double(m) * m) / (4.0 * (n - 1.0) * (n - 1.0) - 1.0));
      const double c = an * (x * b - bn * a);
      T[fidx(n, m)] = c;
      a = b;
      b = c;
    }
  }
}
}  // namespace

std::vector<double> helm_gaunt_table(int P) {
  const int KP = (P + 1) * (P + 1), GL = P + 1, ng = 2 * P + 4;
  std::vector<double> x(ng), w(ng);
  for (int i = 0; i < ng; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (ng + 0.5)), pn = 0, dpn = 1;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int n = 2; n <= ng; ++n) {
        const double p2 = ((2.0 * n - 1.0) * z * p1 - (n - 1.0) * p0) / n;
        p0 = p1;
        p1 = p2;
      }
      pn = p1;
      dpn = ng * (z * p1 - p0) / (z * z - 1.0);
      const double dz = pn / dpn;
      z -= dz;
      if (std::fabs(dz) < 1e-15) break;
    }
    double p0 = 1.0, p1 = z;
    for (int n = 2; n <= ng; ++n) {
      const double p2 = ((2.0 * n - 1.0) * z * p1 - (n - 1.0) * p0) / n;
      p0 = p1;
      p1 = p2;
    }
    dpn = ng * (z * p1 - p0) / (z * z - 1.0);
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dpn * dpn);
  }
  std::vector<std::vector<double>> pb(ng);
  for (int i = 0; i < ng; ++i) pbar(2 * P, x[i], pb[i]);
  std::vector<double> G(size_t(KP) * KP * GL, 0.0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int kin = 0; kin < KP; ++kin) {
    int n = int(std::sqrt(double(kin)));
    while (n * n > kin) --n;
    const int m = kin - n * n - n;
    for (int iout = 0; iout < KP; ++iout) {
      int n2 = int(std::sqrt(double(iout)));
      while (n2 * n2 > iout) --n2;
      const int m2 = iout - n2 * n2 - n2;
      const int mu = m - m2;
      for (int li = 0; li < GL; ++li) {
        const int l = std::abs(n - n2) + 2 * li;
        if (l > n + n2) break;
        if (std::abs(mu) > l) continue;
        double s = 0.0;
        for (int i = 0; i < ng; ++i)
          s += w[i] * pb[i][fidx(n, std::abs(m))] * pb[i][fidx(n2, std::abs(m2))] * pb[i][fidx(l, std::abs(mu))];
        G[(size_t(kin) * KP + iout) * GL + li] = 2.0 * kPi * s;
      }
    }
  }
  return G;
}

}  // namespace qbxg
