// Host construction of the real-DOF rotation blocks used by the GPU
// point-and-shoot M2L (see rotation.hpp).  Wigner small-d from the explicit
// factorial sum in long double (p <= 21 keeps ~14 significant digits).
//
// Basis relation (this code's unnormalised solid harmonics vs. the standard
// Condon-Shortley Y): X_n^k = (-1)^k c_{n|k|} Y_n^k, so with
// A_{n,a} = sqrt((n-a)!(n+a)!) and v = rho (sin t cos f, sin t sin f, cos t),
// Q = Ry(-t) Rz(-f) (maps v to +z):
//   I_n^k(Q^T y) = sum_k' W_{k k'} I_n^k'(y),  W_{k k'} = (-1)^{k+k'} A_{n|k|}/A_{n|k'|} d^n_{k'k}(-t) e^{ikf}
//   R_n^k(Q s)   = sum_k' V_{k k'} R_n^k'(s),  V_{k k'} = (-1)^{k+k'} A_{n|k'|}/A_{n|k|} e^{-ik'f} d^n_{k'k}(t)
// Rotated multipole M'_k' = sum_k M_k W_{kk'}; original local L_k' = sum_k L'_k V_{kk'}.
#include "rotation.hpp"

#include <cmath>
#include <complex>
#include <vector>

namespace qbxg {

namespace {

using ld = long double;
using cld = std::complex<long double>;

struct Fact {
  ld f[100];
  Fact() {
    f[0] = 1;
    for (int i = 1; i < 100; ++i) f[i] = f[i - 1] * i;
  }
};
const Fact kF;

ld ipow(ld x, int e) {
  ld r = 1;
  for (int i = 0; i < e; ++i) r *= x;
  return r;
}

ld wigner_d(int l, int mp, int m, ld c, ld s) {  // c = cos(b/2), s = sin(b/2)
  ld sum = 0;
  const int k0 = std::max(0, m - mp), k1 = std::min(l + m, l - mp);
  const ld num = std::sqrt(kF.f[l + m] * kF.f[l - m] * kF.f[l + mp] * kF.f[l - mp]);
  for (int k = k0; k <= k1; ++k) {
    const ld den = kF.f[l + m - k] * kF.f[k] * kF.f[l - k - mp] * kF.f[k - m + mp];
    const ld t = num / den * ipow(c, 2 * l - 2 * k + m - mp) * ipow(s, 2 * k - m + mp);
    sum += ((k - m + mp) & 1) ? -t : t;
  }
  return sum;
}

// Real-DOF block from a complex map Y_k' = sum_k X_k T[k][k'] on conjugate-symmetric
// data (X_{-k} = (-1)^k conj(X_k)): A = T[k][k'], B = (-1)^k T[-k][k'] (k > 0).
void real_block(int n, const std::vector<cld>& T, double* out) {
  const int d = 2 * n + 1;
  auto Tk = [&](int k, int kp) { return T[size_t(k + n) * d + (kp + n)]; };
  for (int kp = 0; kp <= n; ++kp)
    for (int po = 0; po < (kp == 0 ? 1 : 2); ++po)
      for (int k = 0; k <= n; ++k)
        for (int pi = 0; pi < (k == 0 ? 1 : 2); ++pi) {
          const cld A = Tk(k, kp);
          const cld B = k > 0 ? ((k & 1) ? -Tk(-k, kp) : Tk(-k, kp)) : cld(0);
          ld v;
          if (po == 0)
            v = pi == 0 ? (A + B).real() : -(A - B).imag();
          else
            v = pi == 0 ? (A + B).imag() : (A - B).real();
          const int ro = kp == 0 ? 0 : 2 * kp - 1 + po, ri = k == 0 ? 0 : 2 * k - 1 + pi;
          out[size_t(ro) * d + ri] = double(v);
        }
}

}  // namespace

void m2l_rotation_blocks(int p, const double v[3], double* Rf, double* Rb) {
  const ld x = v[0], y = v[1], z = v[2];
  const ld rho = std::sqrt(x * x + y * y + z * z);
  const ld th = std::acos(std::max<ld>(-1, std::min<ld>(1, z / rho)));
  const ld ph = (x == 0 && y == 0) ? 0 : std::atan2(y, x);
  const ld cp = std::cos(th / 2), sp = std::sin(th / 2);  // d(theta)
  const ld cm = cp, sm = -sp;                             // d(-theta)
  for (int n = 0; n <= p; ++n) {
    const int d = 2 * n + 1;
    std::vector<cld> W(size_t(d) * d), V(size_t(d) * d);
    for (int k = -n; k <= n; ++k)
      for (int kp = -n; kp <= n; ++kp) {
        const ld sg = ((k + kp) & 1) ? -1 : 1;
        const ld ak = std::sqrt(kF.f[n - std::abs(k)] * kF.f[n + std::abs(k)]);
        const ld akp = std::sqrt(kF.f[n - std::abs(kp)] * kF.f[n + std::abs(kp)]);
        W[size_t(k + n) * d + (kp + n)] = sg * ak / akp * wigner_d(n, kp, k, cm, sm) * std::polar<ld>(1, k * ph);
        V[size_t(k + n) * d + (kp + n)] = sg * akp / ak * std::polar<ld>(1, -kp * ph) * wigner_d(n, kp, k, cp, sp);
      }
    real_block(n, W, Rf + rot_block_offset(n));
    real_block(n, V, Rb + rot_block_offset(n));
  }
}

}  // namespace qbxg
