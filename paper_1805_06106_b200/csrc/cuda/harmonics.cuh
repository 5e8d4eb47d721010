// Device-side solid harmonics on half tables (0 <= m <= n), fp64.
//
// Basis (same as the CPU oracle; a rescaling of the paper's Eq. (3)-(4),
// PAPER.md:263-280):
//   R_n^m(x) = r^n P_n^m(cos t) e^{i m phi} / (n+m)!          (regular)
//   I_n^m(x) = (n-m)! P_n^m(cos t) e^{i m phi} / r^{n+1}       (irregular)
//   X_n^{-m} = (-1)^m conj(X_n^m)
// evaluated with the Cartesian recurrences (no trig):
//   R_m^m = R_{m-1}^{m-1} (x+iy)/(2m),  R_{m+1}^m = z R_m^m,
//   R_n^m = ((2n-1) z R_{n-1}^m - r^2 R_{n-2}^m) / ((n-m)(n+m))
//   I_0^0 = 1/r,  I_m^m = (2m-1)(x+iy)/r^2 I_{m-1}^{m-1},  I_{m+1}^m = (2m+1) z/r^2 I_m^m,
//   I_n^m = ((2n-1) z I_{n-1}^m - (n-1+m)(n-1-m) I_{n-2}^m) / r^2
// Half-table index hidx(n, m) = n(n+1)/2 + m (n-major).
#pragma once

#include <cuda_runtime.h>

namespace qbxg {
namespace dev {

constexpr int kMaxOrder = 48;  // tables sized for p + q + 1 <= kMaxOrder
constexpr double kInv4Pi = 0.07957747154594766788;

__host__ __device__ constexpr int hidx(int n, int m) { return n * (n + 1) / 2 + m; }
__host__ __device__ constexpr int hsize(int p) { return (p + 1) * (p + 2) / 2; }

// 1 / ((n-m)(n+m)) for the regular recurrence, indexed hidx(n, m) (n >= m+2).
// Without -rdc every translation unit owns its copy: each TU that calls a
// regular_* helper must call upload_inv_nm() (host) before launching.
__constant__ double c_inv_nm[hsize(kMaxOrder)];
// the same table in global memory, for loops whose lanes index different orders m (the
// constant cache serialises divergent addresses)
__device__ double g_inv_nm[hsize(kMaxOrder)];

static inline void upload_inv_nm() {
  static bool done = false;  // per translation unit
  if (done) return;
  double h[hsize(kMaxOrder)];
  for (int n = 0; n <= kMaxOrder; ++n)
    for (int m = 0; m <= n; ++m) h[hidx(n, m)] = (n >= m + 2) ? 1.0 / double((n - m) * (n + m)) : 0.0;
  cudaMemcpyToSymbol(c_inv_nm, h, sizeof(h));
  cudaMemcpyToSymbol(g_inv_nm, h, sizeof(h));
  done = true;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// Full-index access into a half table: X_n^m for |m| <= n, zero outside.
__device__ __forceinline__ double2 hget(const double2* T, int n, int m) {
  if (m >= 0) return T[hidx(n, m)];
  const double2 v = T[hidx(n, -m)];
  return (m & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
}

// Regular harmonics up to order P into T (half table), runtime order.
__device__ inline void regular_table(double x, double y, double z, int P, double2* T) {
  const double r2 = x * x + y * y + z * z;
  double2 rmm = make_double2(1.0, 0.0);
  for (int m = 0; m <= P; ++m) {
    if (m > 0) {
      const double s = 1.0 / (2.0 * m);
      rmm = make_double2((rmm.x * x - rmm.y * y) * s, (rmm.x * y + rmm.y * x) * s);
    }
    T[hidx(m, m)] = rmm;
    if (m + 1 > P) break;
    double2 a = rmm, b = make_double2(z * rmm.x, z * rmm.y);
    T[hidx(m + 1, m)] = b;
    for (int n = m + 2; n <= P; ++n) {
      const double f = c_inv_nm[hidx(n, m)];
      const double c1 = (2 * n - 1) * z;
      const double2 c = make_double2((c1 * b.x - r2 * a.x) * f, (c1 * b.y - r2 * a.y) * f);
      T[hidx(n, m)] = c;
      a = b;
      b = c;
    }
  }
}

// Regular harmonics of one column m (n = m..P), into col[n - m].
__device__ inline void regular_column(double x, double y, double z, int m, int P, double2* col) {
  const double r2 = x * x + y * y + z * z;
  double2 rmm = make_double2(1.0, 0.0);
  for (int k = 1; k <= m; ++k) {
    const double s = 1.0 / (2.0 * k);
    rmm = make_double2((rmm.x * x - rmm.y * y) * s, (rmm.x * y + rmm.y * x) * s);
  }
  col[0] = rmm;
  if (m + 1 > P) return;
  double2 a = rmm, b = make_double2(z * rmm.x, z * rmm.y);
  col[1] = b;
  for (int n = m + 2; n <= P; ++n) {
    const double f = c_inv_nm[hidx(n, m)];
    const double c1 = (2 * n - 1) * z;
    const double2 c = make_double2((c1 * b.x - r2 * a.x) * f, (c1 * b.y - r2 * a.y) * f);
    col[n - m] = c;
    a = b;
    b = c;
  }
}

// Irregular harmonics up to order P into T (half table), runtime order.
__device__ inline void irregular_table(double x, double y, double z, int P, double2* T) {
  const double r2 = x * x + y * y + z * z;
  const double ir2 = 1.0 / r2;
  double2 imm = make_double2(sqrt(ir2), 0.0);
  for (int m = 0; m <= P; ++m) {
    if (m > 0) {
      const double s = (2 * m - 1) * ir2;
      imm = make_double2((imm.x * x - imm.y * y) * s, (imm.x * y + imm.y * x) * s);
    }
    T[hidx(m, m)] = imm;
    if (m + 1 > P) break;
    const double s1 = (2 * m + 1) * z * ir2;
    double2 a = imm, b = make_double2(s1 * imm.x, s1 * imm.y);
    T[hidx(m + 1, m)] = b;
    for (int n = m + 2; n <= P; ++n) {
      const double c1 = (2 * n - 1) * z;
      const double c2 = double((n - 1 + m) * (n - 1 - m));
      const double2 c = make_double2((c1 * b.x - c2 * a.x) * ir2, (c1 * b.y - c2 * a.y) * ir2);
      T[hidx(n, m)] = c;
      a = b;
      b = c;
    }
  }
}

// Irregular harmonics of one column m (n = m..P), into col[n - m].
__device__ inline void irregular_column(double x, double y, double z, int m, int P, double2* col) {
  const double r2 = x * x + y * y + z * z;
  const double ir2 = 1.0 / r2;
  double2 imm = make_double2(sqrt(ir2), 0.0);
  for (int k = 1; k <= m; ++k) {
    const double s = (2 * k - 1) * ir2;
    imm = make_double2((imm.x * x - imm.y * y) * s, (imm.x * y + imm.y * x) * s);
  }
  col[0] = imm;
  if (m + 1 > P) return;
  const double s1 = (2 * m + 1) * z * ir2;
  double2 a = imm, b = make_double2(s1 * imm.x, s1 * imm.y);
  col[1] = b;
  for (int n = m + 2; n <= P; ++n) {
    const double c1 = (2 * n - 1) * z;
    const double c2 = double((n - 1 + m) * (n - 1 - m));
    const double2 c = make_double2((c1 * b.x - c2 * a.x) * ir2, (c1 * b.y - c2 * a.y) * ir2);
    col[n - m] = c;
    a = b;
    b = c;
  }
}

// Compile-time-order irregular table (fully unrolled, lives in registers).
template <int P>
__device__ __forceinline__ void irregular_regs(double x, double y, double z, double2 (&T)[hsize(P)]) {
  const double r2 = x * x + y * y + z * z;
  const double ir2 = 1.0 / r2;
  double2 imm = make_double2(sqrt(ir2), 0.0);
#pragma unroll
  for (int m = 0; m <= P; ++m) {
    if (m > 0) {
      const double s = (2 * m - 1) * ir2;
      imm = make_double2((imm.x * x - imm.y * y) * s, (imm.x * y + imm.y * x) * s);
    }
    T[hidx(m, m)] = imm;
    if (m + 1 <= P) {
      const double s1 = (2 * m + 1) * z * ir2;
      T[hidx(m + 1, m)] = make_double2(s1 * imm.x, s1 * imm.y);
#pragma unroll
      for (int n = m + 2; n <= P; ++n) {
        const double c1 = (2 * n - 1) * z;
        const double c2 = double((n - 1 + m) * (n - 1 - m));
        const double2 a = T[hidx(n - 2, m)], b = T[hidx(n - 1, m)];
        T[hidx(n, m)] = make_double2((c1 * b.x - c2 * a.x) * ir2, (c1 * b.y - c2 * a.y) * ir2);
      }
    }
  }
}

template <int P>
__device__ __forceinline__ void regular_regs(double x, double y, double z, double2 (&T)[hsize(P)]) {
  const double r2 = x * x + y * y + z * z;
  double2 rmm = make_double2(1.0, 0.0);
#pragma unroll
  for (int m = 0; m <= P; ++m) {
    if (m > 0) {
      const double s = 1.0 / (2.0 * m);
      rmm = make_double2((rmm.x * x - rmm.y * y) * s, (rmm.x * y + rmm.y * x) * s);
    }
    T[hidx(m, m)] = rmm;
    if (m + 1 <= P) {
      T[hidx(m + 1, m)] = make_double2(z * rmm.x, z * rmm.y);
#pragma unroll
      for (int n = m + 2; n <= P; ++n) {
        const double f = 1.0 / double((n - m) * (n + m));
        const double c1 = (2 * n - 1) * z;
        const double2 a = T[hidx(n - 2, m)], b = T[hidx(n - 1, m)];
        T[hidx(n, m)] = make_double2((c1 * b.x - r2 * a.x) * f, (c1 * b.y - r2 * a.y) * f);
      }
    }
  }
}

}  // namespace dev
}  // namespace qbxg
