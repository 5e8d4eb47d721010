// Device math shared by the Helmholtz kernels (helm.cu, helm_fmm.cu): spherical
// Bessel j_n (series below 1, Miller's downward recurrence above), orthonormal
// Y_n^m without the Condon-Shortley phase, complex helpers.  Full tables, index
// n^2 + n + m.
#pragma once

#include <cuda_runtime.h>

namespace qbxg {
namespace dev {
namespace hm {

constexpr double kPi = 3.14159265358979323846;
constexpr int kHQmax = 8;
__device__ __forceinline__ int fi(int n, int m) { return n * n + n + m; }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// j_n(x): power series for x < 1, Miller's downward recurrence otherwise
__device__ inline double sph_j1(int n, double x) {
  if (x < 1.0) {
    double pre = 1.0;
    for (int i = 1; i <= n; ++i) pre *= x / (2.0 * i + 1.0);
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 40; ++k) {
      term *= -0.5 * x * x / (k * (2.0 * n + 2.0 * k + 1.0));
      sum += term;
      if (fabs(term) < 1e-18 * fabs(sum)) break;
    }
    return pre * sum;
  }
  const int N = n + 30 + int(x);
  double t2 = 0.0, t1 = 1e-280, tn = 0.0, tone = 0.0;
  for (int i = N; i >= 1; --i) {  // t_{i-1} = (2i+1)/x t_i - t_{i+1}
    const double tm = (2.0 * i + 1.0) / x * t1 - t2;
    t2 = t1;
    t1 = tm;
    if (i - 1 == n) tn = tm;
    if (i - 1 == 1) tone = tm;
    if (fabs(t1) > 1e250) {
      t1 *= 1e-250;
      t2 *= 1e-250;
      tn *= 1e-250;
      tone *= 1e-250;
    }
  }
  const double t0 = t1;
  if (n == 0) tn = t0;
  const double j0 = sin(x) / x, j1 = sin(x) / (x * x) - cos(x) / x;
  return fabs(j0) > fabs(j1) ? tn * (j0 / t0) : tn * (j1 / tone);
}

// normalised Y_n^m(v), n <= P, |m| <= n
__device__ inline void ylm_all(int P, double vx, double vy, double vz, double2* Y) {
  const double r = sqrt(vx * vx + vy * vy + vz * vz);
  const double ct = r > 0 ? vz / r : 1.0, st = sqrt(fmax(0.0, 1.0 - ct * ct));
  const double ph = atan2(vy, vx);
  double mm = 1.0 / sqrt(4.0 * kPi);
  for (int m = 0; m <= P; ++m) {
    if (m > 0) mm *= sqrt((2.0 * m + 1.0) / (2.0 * m)) * st;
    double s, c;
    sincos(m * ph, &s, &c);
    double a = mm;
    Y[fi(m, m)] = make_double2(a * c, a * s);
    Y[fi(m, -m)] = make_double2(a * c, -a * s);
    if (m + 1 > P) continue;
    double b = sqrt(2.0 * m + 3.0) * ct * a;
    Y[fi(m + 1, m)] = make_double2(b * c, b * s);
    Y[fi(m + 1, -m)] = make_double2(b * c, -b * s);
    for (int n = m + 2; n <= P; ++n) {
      const double an = sqrt((4.0 * n * n - 1.0) / (double(n) * n - double(m) * m));
      const double bn = sqrt(((n - 1.0) * (n - 1.0) - double(m) * m) / (4.0 * (n - 1.0) * (n - 1.0) - 1.0));
      const double cc = an * (ct * b - bn * a);
      Y[fi(n, m)] = make_double2(cc * c, cc * s);
      Y[fi(n, -m)] = make_double2(cc * c, -cc * s);
      a = b;
      b = cc;
    }
  }
}


__device__ __forceinline__ double2 ipow(int e) {
  switch (e & 3) {
    case 0: return make_double2(1, 0);
    case 1: return make_double2(0, 1);
    case 2: return make_double2(-1, 0);
    default: return make_double2(0, -1);
  }
}

}  // namespace hm
}  // namespace dev
}  // namespace qbxg
