// TEST INFRASTRUCTURE ONLY -- CPU oracle for the Helmholtz single layer (BASELINE
// config 3).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline may load this library; the product path never does.
//
// Parity is UNPINNED: the reference excludes Helmholtz
// and the paper's FMMLIB3D operators are not available, so the
// anchors are analytic: the Gegenbauer addition theorem, the three translation
// theorems (checked against scipy in tests/test_helmholtz.py), direct sums, and the
// FMM converging to direct QBX as p grows.
//
// Formulation (orthonormal spherical harmonics without the Condon-Shortley phase,
// Y_n^{-m} = conj(Y_n^m)):
//   G_k(x,y) = e^{ik|x-y|}/(4 pi |x-y|) = ik sum_{n,m} j_n(k|y|) h_n(k|x|) Y_n^m(x) conj(Y_n^m(y))
//   multipole  phi(x) = sum M_n^m h_n(k|x-c|) Y_n^m(x-c),  M_n^m = ik sum_s w_s j_n(k|s-c|) conj(Y_n^m(s-c))
//   local      phi(x) = sum L_n^m j_n(k|x-c|) Y_n^m(x-c),  L_n^m = ik sum_s w_s h_n(k|s-c|) conj(Y_n^m(s-c))
//   translations with R_n^m = j_n Y_n^m, S_n^m = h_n Y_n^m and
//     E_n^m(x + t) = sum_{n',m'} [4 pi sum_l i^{n'+l-n} G(n,m;n',m';l) F_l^{m-m'}(t)] E'_{n'}^{m'}(x),
//     G = int Y_n^m conj(Y_{n'}^{m'}) conj(Y_l^{m-m'}) dOmega,
//   (S|S): E = S, F = R, E' = S (M2M);  (S|R): E = S, F = S, E' = R (M2L, |x| < |t|);
//   (R|R): E = R, F = R, E' = R (L2L).
// Full complex tables, index n^2 + n + m.  Plain loops; a different code shape from
// any GPU kernel.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qbxg.h"

namespace {

using cd = std::complex<double>;
const cd I1(0.0, 1.0);
constexpr double kPi = 3.14159265358979323846;

inline int ix(int n, int m) { return n * n + n + m; }
inline int nf(int p) { return (p + 1) * (p + 1); }

std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return QBXG_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QBXG_ERR_INTERNAL;
  }
}

// fully normalised associated Legendre Pbar_n^m(x), m >= 0, no Condon-Shortley phase:
// Y_n^m = Pbar_n^|m|(cos t) e^{i m phi}
void pbar_table(int P, double x, std::vector<double>& T) {
  T.assign(size_t(nf(P)), 0.0);
  const double s = std::sqrt(std::max(0.0, 1.0 - x * x));
  std::vector<double> mm(P + 1);
  mm[0] = 1.0 / std::sqrt(4.0 * kPi);
  for (int m = 1; m <= P; ++m) mm[m] = std::sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * mm[m - 1];
  for (int m = 0; m <= P; ++m) {
    double a = mm[m];
    T[ix(m, m)] = a;
    if (m + 1 > P) continue;
    double b = std::sqrt(2.0 * m + 3.0) * x * a;
    T[ix(m + 1, m)] = b;
    for (int n = m + 2; n <= P; ++n) {
      const double an = std::sqrt((4.0 * n * n - 1.0) / (double(n) * n - double(m) * m));
      const double bn = std::sqrt(((n - 1.0) * (n - 1.0) - double(m) * m) / (4.0 * (n - 1.0) * (n - 1.0) - 1.0));
      const double c = an * (x * b - bn * a);
      T[ix(n, m)] = c;
      a = b;
      b = c;
    }
  }
}

// Y_n^m(v/|v|) for all n <= P, |m| <= n
void ylm(int P, const double* v, std::vector<cd>& Y) {
  const double r = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  const double ct = r > 0 ? v[2] / r : 1.0;
  const double ph = std::atan2(v[1], v[0]);
  std::vector<double> T;
  pbar_table(P, ct, T);
  Y.assign(size_t(nf(P)), cd(0));
  for (int n = 0; n <= P; ++n)
    for (int m = 0; m <= n; ++m) {
      const cd e = std::polar(1.0, m * ph);
      Y[ix(n, m)] = T[ix(n, m)] * e;
      Y[ix(n, -m)] = std::conj(Y[ix(n, m)]);
    }
}

// spherical Bessel j_n(x), n <= P: series for x < 1, Miller's downward recurrence otherwise
void sph_j(int P, double x, std::vector<double>& J) {
  J.assign(size_t(P + 1), 0.0);
  if (x < 1.0) {
    double pre = 1.0;  // x^n / (2n+1)!!
    for (int n = 0; n <= P; ++n) {
      if (n > 0) pre *= x / (2.0 * n + 1.0);
      double term = 1.0, sum = 1.0;
      for (int k = 1; k < 40; ++k) {
        term *= -0.5 * x * x / (k * (2.0 * n + 2.0 * k + 1.0));
        sum += term;
        if (std::fabs(term) < 1e-18 * std::fabs(sum)) break;
      }
      J[n] = pre * sum;
    }
    return;
  }
  const int N = P + 30 + int(x);
  std::vector<double> t(N + 2, 0.0);
  t[N + 1] = 0.0;
  t[N] = 1e-280;
  for (int n = N; n >= 1; --n) {
    t[n - 1] = (2.0 * n + 1.0) / x * t[n] - t[n + 1];
    if (std::fabs(t[n - 1]) > 1e250)  // rescale to stay in range
      for (int k = n - 1; k <= N + 1; ++k) t[k] *= 1e-250;
  }
  const double j0 = std::sin(x) / x, j1 = std::sin(x) / (x * x) - std::cos(x) / x;
  const double f = std::fabs(j0) > std::fabs(j1) ? j0 / t[0] : j1 / t[1];
  for (int n = 0; n <= P; ++n) J[n] = t[n] * f;
}

// spherical Hankel h_n^(1)(x) = j_n + i y_n, y_n by the (stable) upward recurrence
void sph_h(int P, double x, std::vector<cd>& H) {
  std::vector<double> J;
  sph_j(P, x, J);
  std::vector<double> Yn(P + 1);
  Yn[0] = -std::cos(x) / x;
  if (P >= 1) Yn[1] = -std::cos(x) / (x * x) - std::sin(x) / x;
  for (int n = 1; n < P; ++n) Yn[n + 1] = (2.0 * n + 1.0) / x * Yn[n] - Yn[n - 1];
  H.resize(size_t(P + 1));
  for (int n = 0; n <= P; ++n) H[n] = cd(J[n], Yn[n]);
}

// regular / singular wave functions of v for all n <= P
void wave_R(double k, int P, const double* v, std::vector<cd>& R) {
  std::vector<cd> Y;
  ylm(P, v, Y);
  std::vector<double> J;
  sph_j(P, k * std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]), J);
  R.resize(Y.size());
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) R[ix(n, m)] = J[n] * Y[ix(n, m)];
}
void wave_S(double k, int P, const double* v, std::vector<cd>& S) {
  std::vector<cd> Y;
  ylm(P, v, Y);
  std::vector<cd> H;
  sph_h(P, k * std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]), H);
  S.resize(Y.size());
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) S[ix(n, m)] = H[n] * Y[ix(n, m)];
}

// Gaunt coefficients G(n,m;n',m';l) = int Y_n^m conj(Y_n'^m') conj(Y_l^{m-m'}) by
// Gauss-Legendre quadrature in cos(theta) (exact: polynomial degree <= n+n'+l).
struct Gaunt {
  int P = -1;
  std::vector<double> x, w;                // nodes, weights
  std::vector<std::vector<double>> pb;     // per node: Pbar table to degree 2P
  void build(int Pmax) {
    if (Pmax <= P) return;
    P = Pmax;
    const int ng = 2 * P + 4;  // 2 ng - 1 >= 4P
    x.assign(ng, 0.0);
    w.assign(ng, 0.0);
    auto legendre = [&](double z, double& pn, double& dpn) {
      double p0 = 1.0, p1 = z;
      for (int n = 2; n <= ng; ++n) {
        const double p2 = ((2.0 * n - 1.0) * z * p1 - (n - 1.0) * p0) / n;
        p0 = p1;
        p1 = p2;
      }
      pn = p1;
      dpn = ng * (z * p1 - p0) / (z * z - 1.0);
    };
    for (int i = 0; i < ng; ++i) {  // Newton on P_ng from the usual asymptotic guess
      double z = std::cos(kPi * (i + 0.75) / (ng + 0.5)), pn, dpn;
      for (int it = 0; it < 100; ++it) {
        legendre(z, pn, dpn);
        const double dz = pn / dpn;
        z -= dz;
        if (std::fabs(dz) < 1e-15) break;
      }
      legendre(z, pn, dpn);
      x[i] = z;
      w[i] = 2.0 / ((1.0 - z * z) * dpn * dpn);
    }
    pb.resize(ng);
    for (int i = 0; i < ng; ++i) pbar_table(2 * P, x[i], pb[i]);
    // memo of every value (the same quadrature sum, evaluated once): (P+1)^4 x (2P+1)
    const int K = nf(P);
    tab.assign(size_t(K) * K * (2 * P + 1), 0.0);
#pragma omp parallel for schedule(dynamic, 4)
    for (int a = 0; a < K; ++a) {
      const int n = int(std::sqrt(double(a))), m = a - n * n - n;
      for (int n2 = 0; n2 <= P; ++n2)
        for (int m2 = -n2; m2 <= n2; ++m2)
          for (int l = 0; l <= 2 * P; ++l) tab[(size_t(a) * K + ix(n2, m2)) * (2 * P + 1) + l] = quad(n, m, n2, m2, l);
    }
  }
  double quad(int n, int m, int n2, int m2, int l) const {
    const int mu = m - m2;
    if (std::abs(m) > n || std::abs(m2) > n2 || std::abs(mu) > l) return 0.0;
    if ((n + n2 + l) & 1) return 0.0;
    double s = 0.0;
    for (size_t i = 0; i < x.size(); ++i)
      s += w[i] * pb[i][ix(n, std::abs(m))] * pb[i][ix(n2, std::abs(m2))] * pb[i][ix(l, std::abs(mu))];
    return 2.0 * kPi * s;
  }
  double operator()(int n, int m, int n2, int m2, int l) const {
    if (n > P || n2 > P || l > 2 * P || l < 0) return quad(n, m, n2, m2, l);
    if (std::abs(m) > n || std::abs(m2) > n2) return 0.0;
    return tab[(size_t(ix(n, m)) * nf(P) + ix(n2, m2)) * (2 * P + 1) + l];
  }
  std::vector<double> tab;
};
Gaunt g_gaunt;

cd ipow(int e) {
  switch (((e % 4) + 4) % 4) {
    case 0: return cd(1, 0);
    case 1: return cd(0, 1);
    case 2: return cd(-1, 0);
    default: return cd(0, -1);
  }
}

// out_{n'}^{m'} += sum_{n<=Pin, m} in_n^m [4 pi sum_l i^{n'+l-n} G(n,m;n',m';l) F_l^{m-m'}(t)], n' <= Pout
// F = R (regular) when singular_t is false, S (singular) otherwise.
void translate(double k, const std::vector<cd>& in, int Pin, const double* t, bool singular_t, int Pout,
               std::vector<cd>& out) {
  const int L = Pin + Pout;
  g_gaunt.build(std::max(Pin, Pout));
  std::vector<cd> F;
  if (singular_t)
    wave_S(k, L, t, F);
  else
    wave_R(k, L, t, F);
  for (int n2 = 0; n2 <= Pout; ++n2)
    for (int m2 = -n2; m2 <= n2; ++m2) {
      cd acc(0);
      for (int n = 0; n <= Pin; ++n)
        for (int m = -n; m <= n; ++m) {
          const cd a = in[ix(n, m)];
          if (a == cd(0)) continue;
          cd c(0);
          for (int l = std::abs(n - n2); l <= n + n2; ++l) {
            if (std::abs(m - m2) > l) continue;
            const double g = g_gaunt(n, m, n2, m2, l);
            if (g != 0.0) c += ipow(n2 + l - n) * g * F[ix(l, m - m2)];
          }
          acc += a * (4.0 * kPi) * c;
        }
      out[ix(n2, m2)] += acc;
    }
}

struct Src {
  const double* pos;
  const double* w;   // interleaved complex
  const double* mu;  // null, or 3 complex dipole components per source (6 doubles)
  cd weight(int64_t s) const { return cd(w[2 * s], w[2 * s + 1]); }
  void dipole(int64_t s, cd (&m)[3]) const {
    for (int d = 0; d < 3; ++d) m[d] = cd(mu[6 * s + 2 * d], mu[6 * s + 2 * d + 1]);
  }
};

// mu . grad_v F_n^m(v) for a wave table F = f_n(k|v|) Y_n^m (f = j_n or h_n, orders
// <= PF, PF >= n + 1), by the ladder identities of the spherical wave functions in this
// normalisation (orthonormal Y without the Condon-Shortley phase; checked against
// Richardson finite differences in tests/test_helmholtz.py):
//   d_z F_n^m       = k [a_n^m F_{n-1}^m - a_{n+1}^m F_{n+1}^m],  a_n^m = sqrt((n^2 - m^2) / ((2n-1)(2n+1)))
//   (d_x + i d_y) F = s+ k [c F_{n-1}^{m+1} + e F_{n+1}^{m+1}],   s+ = -1 (m >= 0), +1 (m < 0)
//   (d_x - i d_y) F = s- k [f F_{n-1}^{m-1} + g F_{n+1}^{m-1}],   s- = +1 (m > 0), -1 (m <= 0)
// c = sqrt((n-m-1)(n-m) / ((2n-1)(2n+1))), e = sqrt((n+m+1)(n+m+2) / ((2n+1)(2n+3))),
// f = sqrt((n+m-1)(n+m) / ((2n-1)(2n+1))), g = sqrt((n-m+1)(n-m+2) / ((2n+1)(2n+3)));
// mu . grad = mu_z d_z + (mu_x - i mu_y)/2 (d_x + i d_y) + (mu_x + i mu_y)/2 (d_x - i d_y).
cd grad_dot(double k, const std::vector<cd>& F, int PF, int n, int m, const cd (&mu)[3]) {
  auto at = [&](int nn, int mm) -> cd {
    if (nn < 0 || nn > PF || std::abs(mm) > nn) return cd(0);
    return F[ix(nn, mm)];
  };
  auto sq = [](double x) { return x > 0 ? std::sqrt(x) : 0.0; };
  const double dn = n, dm = m;
  const double a0 = sq((dn * dn - dm * dm) / ((2 * dn - 1) * (2 * dn + 1)));
  const double a1 = sq(((dn + 1) * (dn + 1) - dm * dm) / ((2 * dn + 1) * (2 * dn + 3)));
  const double c = sq((dn - dm - 1) * (dn - dm) / ((2 * dn - 1) * (2 * dn + 1)));
  const double e = sq((dn + dm + 1) * (dn + dm + 2) / ((2 * dn + 1) * (2 * dn + 3)));
  const double f = sq((dn + dm - 1) * (dn + dm) / ((2 * dn - 1) * (2 * dn + 1)));
  const double g = sq((dn - dm + 1) * (dn - dm + 2) / ((2 * dn + 1) * (2 * dn + 3)));
  const cd dz = k * (a0 * at(n - 1, m) - a1 * at(n + 1, m));
  const cd dp = (m >= 0 ? -1.0 : 1.0) * k * (c * at(n - 1, m + 1) + e * at(n + 1, m + 1));
  const cd dmi = (m > 0 ? 1.0 : -1.0) * k * (f * at(n - 1, m - 1) + g * at(n + 1, m - 1));
  return mu[2] * dz + 0.5 * (mu[0] - I1 * mu[1]) * dp + 0.5 * (mu[0] + I1 * mu[1]) * dmi;
}

// P2M: M_n^m += ik [w conj(R_n^m(v)) + mu . grad_s conj(R_n^m(s - c))], conj(R_n^m) = R_n^{-m}
void p2m(double k, const Src& S, int64_t s, const double* c, int P, std::vector<cd>& M) {
  const double v[3] = {S.pos[3 * s] - c[0], S.pos[3 * s + 1] - c[1], S.pos[3 * s + 2] - c[2]};
  std::vector<cd> R;
  const int PF = S.mu ? P + 1 : P;
  wave_R(k, PF, v, R);
  const cd f = I1 * k * S.weight(s);
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) M[ix(n, m)] += f * std::conj(R[ix(n, m)]);
  if (!S.mu) return;
  cd mu[3];
  S.dipole(s, mu);
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) M[ix(n, m)] += I1 * k * grad_dot(k, R, PF, n, -m, mu);
}

// P2L: L_n^m += ik [w h_n conj(Y_n^m)(v) + mu . grad_s (h_n conj(Y_n^m))(s - c)], h_n conj(Y_n^m) = S_n^{-m}
void p2l(double k, const Src& S, int64_t s, const double* c, int P, std::vector<cd>& L) {
  const double v[3] = {S.pos[3 * s] - c[0], S.pos[3 * s + 1] - c[1], S.pos[3 * s + 2] - c[2]};
  std::vector<cd> Y;
  const int PF = S.mu ? P + 1 : P;
  ylm(PF, v, Y);
  std::vector<cd> H;
  sph_h(PF, k * std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]), H);
  const cd f = I1 * k * S.weight(s);
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) L[ix(n, m)] += f * H[n] * std::conj(Y[ix(n, m)]);
  if (!S.mu) return;
  std::vector<cd> F(Y.size());
  for (int n = 0; n <= PF; ++n)
    for (int m = -n; m <= n; ++m) F[ix(n, m)] = H[n] * Y[ix(n, m)];
  cd mu[3];
  S.dipole(s, mu);
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) L[ix(n, m)] += I1 * k * grad_dot(k, F, PF, n, -m, mu);
}

cd eval_local(double k, const std::vector<cd>& L, int P, const double* c, const double* t) {
  const double v[3] = {t[0] - c[0], t[1] - c[1], t[2] - c[2]};
  std::vector<cd> R;
  wave_R(k, P, v, R);
  cd a(0);
  for (int i = 0; i < nf(P); ++i) a += L[i] * R[i];
  return a;
}

cd eval_multipole(double k, const std::vector<cd>& M, int P, const double* c, const double* t) {
  const double v[3] = {t[0] - c[0], t[1] - c[1], t[2] - c[2]};
  std::vector<cd> S;
  wave_S(k, P, v, S);
  cd a(0);
  for (int i = 0; i < nf(P); ++i) a += M[i] * S[i];
  return a;
}

// w G_k(t, s) + mu . grad_s G_k(t, s) = [w + mu . (t - s) (1 - i k r) / r^2] e^{ikr} / (4 pi r)
cd p2p(double k, const Src& S, int64_t s, const double* t) {
  const double dx = t[0] - S.pos[3 * s], dy = t[1] - S.pos[3 * s + 1], dz = t[2] - S.pos[3 * s + 2];
  const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
  if (r == 0.0) throw std::invalid_argument("helmholtz p2p: target coincides with a source");
  cd a = S.weight(s);
  if (S.mu) {
    cd mu[3];
    S.dipole(s, mu);
    a += (mu[0] * dx + mu[1] * dy + mu[2] * dz) * cd(1.0, -k * r) / (r * r);
  }
  return a * std::polar(1.0, k * r) / (4.0 * kPi * r);
}

}  // namespace

extern "C" {

const char* qbxo_helm_last_error(void) { return g_err.c_str(); }

// Y_n^m (orthonormal, no Condon-Shortley phase) at direction v.
int qbxo_helm_ylm(int n, int m, const double* v, double* out) {
  return guard([&] {
    if (n < 0 || std::abs(m) > n) throw std::invalid_argument("bad (n, m)");
    std::vector<cd> Y;
    ylm(n, v, Y);
    out[0] = Y[ix(n, m)].real();
    out[1] = Y[ix(n, m)].imag();
  });
}

// j_n(x) and h_n(x) for n <= P: out_j[P+1], out_h[2(P+1)]
int qbxo_helm_bessel(int P, double x, double* out_j, double* out_h) {
  return guard([&] {
    std::vector<double> J;
    sph_j(P, x, J);
    std::vector<cd> H;
    sph_h(P, x, H);
    for (int n = 0; n <= P; ++n) {
      out_j[n] = J[n];
      out_h[2 * n] = H[n].real();
      out_h[2 * n + 1] = H[n].imag();
    }
  });
}

// Gaunt coefficient G(n,m;n',m';l)
int qbxo_helm_gaunt(int n, int m, int n2, int m2, int l, double* out) {
  return guard([&] {
    g_gaunt.build(std::max(std::max(n, n2), (l + 1) / 2 + 1));
    *out = g_gaunt(n, m, n2, m2, l);
  });
}

// kind 0: P2M (multipole about c), 1: P2L (local about c); weights interleaved complex.
int qbxo_helm_form(int kind, double k, int64_t ns, const double* pos, const double* w, const double* mu,
                   const double* c, int P, double* out) {
  return guard([&] {
    Src S{pos, w, mu};
    std::vector<cd> E(size_t(nf(P)), cd(0));
    for (int64_t s = 0; s < ns; ++s) {
      if (kind == 0)
        p2m(k, S, s, c, P, E);
      else
        p2l(k, S, s, c, P, E);
    }
    for (int i = 0; i < nf(P); ++i) {
      out[2 * i] = E[i].real();
      out[2 * i + 1] = E[i].imag();
    }
  });
}

// kind 0: multipole, 1: local; value at t
int qbxo_helm_eval(int kind, double k, const double* coeffs, int P, const double* c, const double* t, double* out) {
  return guard([&] {
    std::vector<cd> E(size_t(nf(P)));
    for (int i = 0; i < nf(P); ++i) E[i] = cd(coeffs[2 * i], coeffs[2 * i + 1]);
    const cd v = kind == 0 ? eval_multipole(k, E, P, c, t) : eval_local(k, E, P, c, t);
    out[0] = v.real();
    out[1] = v.imag();
  });
}

// kind 0: M2M (c -> C), 1: M2L (multipole at c -> local at C), 2: L2L (c -> C)
int qbxo_helm_translate(int kind, double k, const double* in, int Pin, const double* c, const double* C, int Pout,
                        double* out) {
  return guard([&] {
    std::vector<cd> A(size_t(nf(Pin))), B(size_t(nf(Pout)), cd(0));
    for (int i = 0; i < nf(Pin); ++i) A[i] = cd(in[2 * i], in[2 * i + 1]);
    const double t[3] = {C[0] - c[0], C[1] - c[1], C[2] - c[2]};
    translate(k, A, Pin, t, kind == 1, Pout, B);
    for (int i = 0; i < nf(Pout); ++i) {
      out[2 * i] = B[i].real();
      out[2 * i + 1] = B[i].imag();
    }
  });
}

// potentials (complex, interleaved) at targets from all sources
int qbxo_helm_direct_sum(double k, int64_t ns, const double* pos, const double* w, const double* mu, int64_t nt,
                         const double* tpos, double* out) {
  return guard([&] {
    Src S{pos, w, mu};
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nt; ++t) {
      cd a(0);
      for (int64_t s = 0; s < ns; ++s) a += p2p(k, S, s, &tpos[3 * t]);
      out[2 * t] = a.real();
      out[2 * t + 1] = a.imag();
    }
  });
}

// unaccelerated QBX: each associated target gets its centre's order-q local from ALL
// sources; conventional targets (association -1) the direct sum.
int qbxo_helm_direct_qbx(double k, int64_t ns, const double* pos, const double* w, const double* mu, int64_t nc,
                         const double* cpos, int64_t nt, const double* tpos, const int32_t* assoc, int q,
                         double* out) {
  return guard([&] {
    Src S{pos, w, mu};
    std::vector<std::vector<cd>> Lc{size_t(nc)};
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t c = 0; c < nc; ++c) {
      Lc[c].assign(size_t(nf(q)), cd(0));
      for (int64_t s = 0; s < ns; ++s) p2l(k, S, s, &cpos[3 * c], q, Lc[c]);
    }
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nt; ++t) {
      cd v(0);
      const int32_t a = assoc[t];
      if (a >= 0)
        v = eval_local(k, Lc[a], q, &cpos[3 * int64_t(a)], &tpos[3 * t]);
      else
        for (int64_t s = 0; s < ns; ++s) v += p2p(k, S, s, &tpos[3 * t]);
      out[2 * t] = v.real();
      out[2 * t + 1] = v.imag();
    }
  });
}

// Stages 2-9 of Algorithm 4 for G_k on the host plan (same tree and lists as the
// Laplace path).  Outputs: complex potentials (interleaved) in target order and,
// optionally, the centres' order-q locals (nc x (q+1)^2 complex, index n^2+n+m).
int qbxo_helm_execute(const qbxg_plan_view* V, double k, int p, int q, const double* src_pos,
                      const double* center_pos, const double* target_pos, const int32_t* association,
                      const double* weights, const double* dipoles, double* out_pot, double* out_center_coeffs) {
  return guard([&] {
    const int nb = V->n_boxes;
    const int KP = nf(p), KQ = nf(q);
    Src S{src_pos, weights, dipoles};
    g_gaunt.build(p);
    auto src_of = [&](int64_t sorted) { return int64_t(V->src_perm[sorted]); };
    // Stage 2: P2M at leaves, M2M in postorder
    std::vector<std::vector<cd>> M(nb, std::vector<cd>(KP, cd(0)));
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b) {
      if (V->child_starts[b + 1] != V->child_starts[b]) continue;
      for (int i = 0; i < V->src_own_count[b]; ++i)
        p2m(k, S, src_of(V->src_own_start[b] + i), &V->box_center[3 * b], p, M[b]);
    }
    for (int l = V->n_levels - 2; l >= 0; --l) {
#pragma omp parallel for schedule(dynamic, 16)
      for (int i = V->level_starts[l]; i < V->level_starts[l + 1]; ++i) {
        const int b = V->level_boxes[i];
        for (int kk = V->child_starts[b]; kk < V->child_starts[b + 1]; ++kk) {
          const int c = V->children[kk];
          if (V->src_sub_count[c] == 0) continue;
          const double t[3] = {V->box_center[3 * b] - V->box_center[3 * c],
                               V->box_center[3 * b + 1] - V->box_center[3 * c + 1],
                               V->box_center[3 * b + 2] - V->box_center[3 * c + 2]};
          // (S|S): multipole about the child re-expanded about the parent
          std::vector<cd> out(size_t(KP), cd(0));
          {
            // S_n^m(y + t) = sum (S|S)(t) S_n'^m'(y), y = x - parent, t = parent - child
            translate(k, M[c], p, t, false, p, out);
          }
          for (int j = 0; j < KP; ++j) M[b][j] += out[j];
        }
      }
    }
    const int64_t nc = V->n_centers;
    std::vector<std::vector<cd>> Lc(nc, std::vector<cd>(KQ, cd(0)));
    const int64_t nconv = V->n_conv_targets;
    std::vector<cd> phi(nconv, cd(0));
    // Stages 3, 5a, 6a: near field
    const int near_lists[3] = {QBXG_LIST_U, QBXG_LIST_W_CLOSE, QBXG_LIST_X_CLOSE};
#pragma omp parallel for schedule(dynamic, 4)
    for (int b = 0; b < nb; ++b) {
      if (!(V->box_flags[b] & QBXG_BOX_TARGET)) continue;
      for (int li : near_lists)
        for (int64_t e = V->list_starts[li][b]; e < V->list_starts[li][b + 1]; ++e) {
          const int d = V->list_boxes[li][e];
          for (int i = 0; i < V->src_own_count[d]; ++i) {
            const int64_t s = src_of(V->src_own_start[d] + i);
            for (int j = 0; j < V->ctr_own_count[b]; ++j) {
              const int64_t cs = V->ctr_own_start[b] + j;
              p2l(k, S, s, &center_pos[3 * int64_t(V->ctr_perm[cs])], q, Lc[cs]);
            }
            for (int j = 0; j < V->tgt_own_count[b]; ++j) {
              const int64_t ts = V->tgt_own_start[b] + j;
              phi[ts] += p2p(k, S, s, &target_pos[3 * int64_t(V->tgt_perm[ts])]);
            }
          }
        }
    }
    // Stage 4: M2L
    std::vector<std::vector<cd>> Lb(nb, std::vector<cd>(KP, cd(0)));
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int64_t e = V->list_starts[QBXG_LIST_V][b]; e < V->list_starts[QBXG_LIST_V][b + 1]; ++e) {
        const int d = V->list_boxes[QBXG_LIST_V][e];
        const double t[3] = {V->box_center[3 * b] - V->box_center[3 * d],
                             V->box_center[3 * b + 1] - V->box_center[3 * d + 1],
                             V->box_center[3 * b + 2] - V->box_center[3 * d + 2]};
        translate(k, M[d], p, t, true, p, Lb[b]);
      }
    // Stage 5b: List 3 far
#pragma omp parallel for schedule(dynamic, 4)
    for (int b = 0; b < nb; ++b) {
      if (!(V->box_flags[b] & QBXG_BOX_TARGET)) continue;
      for (int64_t e = V->list_starts[QBXG_LIST_W_FAR][b]; e < V->list_starts[QBXG_LIST_W_FAR][b + 1]; ++e) {
        const int d = V->list_boxes[QBXG_LIST_W_FAR][e];
        for (int j = 0; j < V->ctr_own_count[b]; ++j) {
          const int64_t cs = V->ctr_own_start[b] + j;
          const double* cp = &center_pos[3 * int64_t(V->ctr_perm[cs])];
          const double t[3] = {cp[0] - V->box_center[3 * d], cp[1] - V->box_center[3 * d + 1],
                               cp[2] - V->box_center[3 * d + 2]};
          translate(k, M[d], p, t, true, q, Lc[cs]);
        }
        for (int j = 0; j < V->tgt_own_count[b]; ++j) {
          const int64_t ts = V->tgt_own_start[b] + j;
          phi[ts] += eval_multipole(k, M[d], p, &V->box_center[3 * d], &target_pos[3 * int64_t(V->tgt_perm[ts])]);
        }
      }
    }
    // Stage 6b: List 4 far
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int64_t e = V->list_starts[QBXG_LIST_X_FAR][b]; e < V->list_starts[QBXG_LIST_X_FAR][b + 1]; ++e) {
        const int d = V->list_boxes[QBXG_LIST_X_FAR][e];
        for (int i = 0; i < V->src_own_count[d]; ++i)
          p2l(k, S, src_of(V->src_own_start[d] + i), &V->box_center[3 * b], p, Lb[b]);
      }
    // Stage 7: L2L
    for (int l = 1; l < V->n_levels; ++l) {
#pragma omp parallel for schedule(dynamic, 16)
      for (int i = V->level_starts[l]; i < V->level_starts[l + 1]; ++i) {
        const int b = V->level_boxes[i];
        if (!(V->box_flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR))) continue;
        const int a = V->box_parent[b];
        const double t[3] = {V->box_center[3 * b] - V->box_center[3 * a],
                             V->box_center[3 * b + 1] - V->box_center[3 * a + 1],
                             V->box_center[3 * b + 2] - V->box_center[3 * a + 2]};
        translate(k, Lb[a], p, t, false, p, Lb[b]);
      }
    }
    // Stage 8: L2QBXL
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < V->ctr_own_count[b]; ++j) {
        const int64_t cs = V->ctr_own_start[b] + j;
        const double* cp = &center_pos[3 * int64_t(V->ctr_perm[cs])];
        const double t[3] = {cp[0] - V->box_center[3 * b], cp[1] - V->box_center[3 * b + 1],
                             cp[2] - V->box_center[3 * b + 2]};
        translate(k, Lb[b], p, t, false, q, Lc[cs]);
      }
    // Stage 9: evaluate
    std::vector<int64_t> pos_of(nc);
    for (int64_t cs = 0; cs < nc; ++cs) pos_of[V->ctr_perm[cs]] = cs;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < V->n_targets; ++i) {
      const int32_t a = association[i];
      if (a < 0) continue;
      const cd v = eval_local(k, Lc[pos_of[a]], q, &center_pos[3 * int64_t(a)], &target_pos[3 * i]);
      out_pot[2 * i] = v.real();
      out_pot[2 * i + 1] = v.imag();
    }
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < V->tgt_own_count[b]; ++j) {
        const int64_t ts = V->tgt_own_start[b] + j;
        const int64_t ti = V->tgt_perm[ts];
        const cd v = phi[ts] + eval_local(k, Lb[b], p, &V->box_center[3 * b], &target_pos[3 * ti]);
        out_pot[2 * ti] = v.real();
        out_pot[2 * ti + 1] = v.imag();
      }
    if (out_center_coeffs)
      for (int64_t cs = 0; cs < nc; ++cs) {
        const int64_t c = V->ctr_perm[cs];
        for (int i = 0; i < KQ; ++i) {
          out_center_coeffs[2 * (c * KQ + i)] = Lc[cs][i].real();
          out_center_coeffs[2 * (c * KQ + i) + 1] = Lc[cs][i].imag();
        }
      }
  });
}

}  // extern "C"
