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

// j_0 .. j_Q at x >= 1 from ONE downward Miller recurrence (sph_j1 per degree ran Q + 1
// of them, each with a division per step): t_{i-1} = (2i+1)/x t_i - t_{i+1} from
// i = Q + 30 + int(x), normalised by j_0 or j_1, whichever is larger.
template <int Q>
__device__ __forceinline__ void sph_j_upto(double x, double (&j)[Q + 1]) {
  const int N = Q + 30 + int(x);
  const double ix = 1.0 / x;
  double t2 = 0.0, t1 = 1e-280, t[Q + 1];
#pragma unroll
  for (int n = 0; n <= Q; ++n) t[n] = 0.0;
  for (int i = N; i >= 1; --i) {
    const double tm = (2.0 * i + 1.0) * ix * t1 - t2;
    t2 = t1;
    t1 = tm;
#pragma unroll
    for (int n = 0; n <= Q; ++n)
      if (i - 1 == n) t[n] = tm;
    if (fabs(t1) > 1e250) {
      t1 *= 1e-250;
      t2 *= 1e-250;
#pragma unroll
      for (int n = 0; n <= Q; ++n) t[n] *= 1e-250;
    }
  }
  double sn, cs;
  sincos(x, &sn, &cs);
  const double j0 = sn * ix, j1 = (sn * ix - cs) * ix;
  const double sc = (Q == 0 || fabs(j0) > fabs(j1)) ? j0 / t[0] : j1 / t[Q == 0 ? 0 : 1];
#pragma unroll
  for (int n = 0; n <= Q; ++n) j[n] = t[n] * sc;
}
// the same for a runtime degree, into the real parts of out[0 .. P] times r^-n
__device__ inline void sph_j_upto_rt(int P, double x, double ir, double2* out) {
  const int N = P + 30 + int(x);
  const double ix = 1.0 / x;
  double t2 = 0.0, t1 = 1e-280;
  for (int n = 0; n <= P; ++n) out[n].x = 0.0;
  for (int i = N; i >= 1; --i) {
    const double tm = (2.0 * i + 1.0) * ix * t1 - t2;
    t2 = t1;
    t1 = tm;
    if (i - 1 <= P) out[i - 1].x = tm;
    if (fabs(t1) > 1e250) {
      t1 *= 1e-250;
      t2 *= 1e-250;
      for (int n = i - 1; n <= P; ++n) out[n].x *= 1e-250;
    }
  }
  double sn, cs;
  sincos(x, &sn, &cs);
  const double j0 = sn * ix, j1 = (sn * ix - cs) * ix;
  double sc = (P == 0 || fabs(j0) > fabs(j1)) ? j0 / out[0].x : j1 / out[P == 0 ? 0 : 1].x;
  for (int n = 0; n <= P; ++n) {
    out[n].x *= sc;
    sc *= ir;
  }
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


// j_n(x), n = 0..N in one pass (series below 1, one Miller recurrence above)
template <int N>
__device__ inline void sph_j_all(double x, double (&J)[N + 1]) {
  if (x < 1.0) {
#pragma unroll
    for (int n = 0; n <= N; ++n) J[n] = sph_j1(n, x);
    return;
  }
  const int M = N + 30 + int(x);
  double t2 = 0.0, t1 = 1e-280, t0 = 0.0;
#pragma unroll
  for (int n = 0; n <= N; ++n) J[n] = 0.0;
  double tone = 0.0;
  for (int i = M; i >= 1; --i) {  // t_{i-1} = (2i+1)/x t_i - t_{i+1}
    const double tm = (2.0 * i + 1.0) / x * t1 - t2;
    t2 = t1;
    t1 = tm;
#pragma unroll
    for (int n = 0; n <= N; ++n)
      if (i - 1 == n) J[n] = tm;
    if (i - 1 == 1) tone = tm;
    if (fabs(t1) > 1e250) {
      t1 *= 1e-250;
      t2 *= 1e-250;
      tone *= 1e-250;
#pragma unroll
      for (int n = 0; n <= N; ++n) J[n] *= 1e-250;
    }
  }
  t0 = t1;
  const double j0 = sin(x) / x, j1 = sin(x) / (x * x) - cos(x) / x;
  const double f = fabs(j0) > fabs(j1) ? j0 / t0 : j1 / tone;
#pragma unroll
  for (int n = 0; n <= N; ++n) J[n] *= f;
}

// Double layer: acc[fi(n, m)] += fk * (mu . grad_v F_n^{-m}(v)), n <= N, for the wave
// functions F_n^m = f_n(k|v|) Y_n^m(v) (f = h_n when SING, else j_n), by the ladder
// identities of oracle/helm_oracle.cpp grad_dot (mu complex: m_x, m_y, m_z):
//   mu . grad = mu_z d_z + (mu_x - i mu_y)/2 (d_x + i d_y) + (mu_x + i mu_y)/2 (d_x - i d_y).
// The P2M / P2L / P2QBXL dipole coefficient of a source s about c is ik times this at
// v = s - c (conj(F_n^m) of the monopole formula is F_n^{-m} up to the radial conjugate,
// which the identities never touch).  Per-thread, generic; used by the double-layer
// passes and the unaccelerated paths, not by the single-layer hot kernels.
__device__ __forceinline__ double lad_sq(double x) { return x > 0.0 ? sqrt(x) : 0.0; }

template <int N, bool SING>
__device__ inline void dipole_terms(double k, double vx, double vy, double vz, const double2 (&mu)[3], double2 fk,
                                   double2* acc) {
  constexpr int N1 = N + 1;
  double2 Y[(N1 + 1) * (N1 + 1)];
  ylm_all(N1, vx, vy, vz, Y);
  const double x = k * sqrt(vx * vx + vy * vy + vz * vz);
  double J[N1 + 1];
  sph_j_all<N1>(x, J);
  double yv[N1 + 1];
  if (SING) {
    double ym = -cos(x) / x, y0 = -cos(x) / (x * x) - sin(x) / x;
#pragma unroll
    for (int n = 0; n <= N1; ++n) {
      if (n == 0) {
        yv[n] = ym;
      } else if (n == 1) {
        yv[n] = y0;
      } else {
        const double yn = (2.0 * n - 1.0) / x * y0 - ym;
        ym = y0;
        y0 = yn;
        yv[n] = yn;
      }
    }
  }
  auto F = [&](int n, int m) -> double2 {
    if (n < 0 || n > N1 || m > n || -m > n) return make_double2(0.0, 0.0);
    const double2 y = Y[fi(n, m)];
    if (!SING) return make_double2(J[n] * y.x, J[n] * y.y);
    return cmul(make_double2(J[n], yv[n]), y);
  };
  // (mu_x - i mu_y) / 2 and (mu_x + i mu_y) / 2
  const double2 hp = make_double2(0.5 * (mu[0].x + mu[1].y), 0.5 * (mu[0].y - mu[1].x));
  const double2 hm = make_double2(0.5 * (mu[0].x - mu[1].y), 0.5 * (mu[0].y + mu[1].x));
#pragma unroll
  for (int n = 0; n <= N; ++n)
#pragma unroll
    for (int mo = -n; mo <= n; ++mo) {
      const int m = -mo;  // gradient of F_n^{-mo}
      const double dn = n, dm = m;
      const double a0 = lad_sq((dn * dn - dm * dm) / ((2 * dn - 1) * (2 * dn + 1)));
      const double a1 = lad_sq(((dn + 1) * (dn + 1) - dm * dm) / ((2 * dn + 1) * (2 * dn + 3)));
      const double c = lad_sq((dn - dm - 1) * (dn - dm) / ((2 * dn - 1) * (2 * dn + 1)));
      const double e = lad_sq((dn + dm + 1) * (dn + dm + 2) / ((2 * dn + 1) * (2 * dn + 3)));
      const double f = lad_sq((dn + dm - 1) * (dn + dm) / ((2 * dn - 1) * (2 * dn + 1)));
      const double g = lad_sq((dn - dm + 1) * (dn - dm + 2) / ((2 * dn + 1) * (2 * dn + 3)));
      const double2 Fa = F(n - 1, m), Fb = F(n + 1, m);
      const double2 dz = make_double2(k * (a0 * Fa.x - a1 * Fb.x), k * (a0 * Fa.y - a1 * Fb.y));
      const double sp = m >= 0 ? -k : k, sm = m > 0 ? k : -k;
      const double2 Fc = F(n - 1, m + 1), Fe = F(n + 1, m + 1), Ff = F(n - 1, m - 1), Fg = F(n + 1, m - 1);
      const double2 dp = make_double2(sp * (c * Fc.x + e * Fe.x), sp * (c * Fc.y + e * Fe.y));
      const double2 dmi = make_double2(sm * (f * Ff.x + g * Fg.x), sm * (f * Ff.y + g * Fg.y));
      double2 t = cmul(mu[2], dz);
      t = cfma(hp, dp, t);
      t = cfma(hm, dmi, t);
      acc[fi(n, mo)] = cfma(fk, t, acc[fi(n, mo)]);
    }
}

// the closed-form double-layer kernel: m . grad_y G_k(x, y) = m.(x - y) (1 - i k r) e^{ikr} / (4 pi r^3)
__device__ __forceinline__ double2 dipole_kernel(double k, double dx, double dy, double dz, double r,
                                                 const double2 (&mu)[3]) {
  const double2 md = make_double2(mu[0].x * dx + mu[1].x * dy + mu[2].x * dz, mu[0].y * dx + mu[1].y * dy + mu[2].y * dz);
  double s, c;
  sincos(k * r, &s, &c);
  const double f = 1.0 / (4.0 * kPi * r * r * r);
  // (1 - i k r)(c + i s) = (c + k r s) + i (s - k r c)
  const double2 e = make_double2((c + k * r * s) * f, (s - k * r * c) * f);
  return cmul(md, e);
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
