// Host tables of the Helmholtz point-and-shoot M2L (csrc/cuda/helm_fmm.cu, k_h_m2l_pas;
// PAPER.md:3485-3500).  In the azimuthally rotated frame of the split
// M2L the offset v' = (rho, 0, z) lies in the xz-plane; Q = R_y(-theta) takes it to +z.
// For the orthonormal basis of the Helmholtz path (Y_n^m = Pbar_n^|m|(cos t) e^{i m phi},
// no Condon-Shortley phase):
//   multipole into the rotated frame:  M~_k' = sum_k M'_k W_kk',  Y_k(Q^T u) = sum_k' W_kk' Y_k'(u)
//   local back from the rotated frame: L'_k' = sum_k L~_k V_kk',  Y_k(Q u)   = sum_k' V_kk' Y_k'(u)
// W and V are computed by exact quadrature on the sphere (Gauss-Legendre in cos t with
// P+1 nodes x 2P+2 equispaced azimuths: exact for the degree-2n integrands), so no
// rotation-matrix sign convention has to be trusted.  Rotations about y commute with the
// reflection y -> -y (k <-> -k), so each degree splits into the even / odd blocks of the
// split M2L (A = y_k + y_-k, B = y_k - y_-k, A_0 = y_0), written here as real DMMA
// A-fragments (8 x 4 tiles, fragment (ks, mt) = 32 doubles, lane l holding element
// (8 mt + l / 4, 4 ks + l % 4)).
#include "helm_rot.hpp"

#include <cmath>
#include <complex>
#include <stdexcept>
#include <vector>

namespace qbxg {

namespace {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;

// Gauss-Legendre nodes / weights on [-1, 1]
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), pp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      const double dz = p1 / pp;
      z -= dz;
      if (std::fabs(dz) < 1e-15) break;
    }
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

// Y_n^m(u) for |u| = 1, n <= P, index n^2 + n + m
void ylm(int P, const double u[3], std::vector<cd>& Y) {
  const int K = (P + 1) * (P + 1);
  Y.assign(K, cd(0.0));
  const double x = std::max(-1.0, std::min(1.0, u[2]));
  const double s = std::sqrt(std::max(0.0, 1.0 - x * x));
  const double ph = (u[0] == 0.0 && u[1] == 0.0) ? 0.0 : std::atan2(u[1], u[0]);
  std::vector<double> Pb(K, 0.0);
  auto pi = [](int n, int m) { return n * n + n + m; };
  Pb[pi(0, 0)] = 1.0 / std::sqrt(4.0 * kPi);
  for (int m = 1; m <= P; ++m) Pb[pi(m, m)] = std::sqrt((2.0 * m + 1) / (2.0 * m)) * s * Pb[pi(m - 1, m - 1)];
  for (int m = 0; m < P; ++m) Pb[pi(m + 1, m)] = std::sqrt(2.0 * m + 3) * x * Pb[pi(m, m)];
  for (int m = 0; m <= P; ++m)
    for (int n = m + 2; n <= P; ++n) {
      const double a = std::sqrt((4.0 * n * n - 1) / (double(n) * n - double(m) * m));
      const double b = std::sqrt(((n - 1.0) * (n - 1) - double(m) * m) / (4.0 * (n - 1) * (n - 1) - 1));
      Pb[pi(n, m)] = a * (x * Pb[pi(n - 1, m)] - b * Pb[pi(n - 2, m)]);
    }
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) Y[pi(n, m)] = Pb[pi(n, std::abs(m))] * std::polar(1.0, m * ph);
}

// rotation maps for R = R_y(a): X_op(n)[out k' + n][in k + n] = X_kk', Y_k(R u) = sum X_kk' Y_k'(u)
void rot_y(int P, double a, std::vector<std::vector<double>>& Xop) {
  std::vector<double> gx, gw;
  gauss_legendre(P + 1, gx, gw);
  const int NF = 2 * P + 2;
  const double ca = std::cos(a), sa = std::sin(a);
  std::vector<std::vector<cd>> acc(P + 1);
  for (int n = 0; n <= P; ++n) acc[n].assign(size_t(2 * n + 1) * (2 * n + 1), cd(0.0));
  std::vector<cd> Yu, Yr;
  for (int i = 0; i <= P; ++i)
    for (int j = 0; j < NF; ++j) {
      const double ct = gx[i], st = std::sqrt(std::max(0.0, 1.0 - ct * ct)), ph = 2.0 * kPi * j / NF;
      const double u[3] = {st * std::cos(ph), st * std::sin(ph), ct};
      const double r[3] = {u[0] * ca + u[2] * sa, u[1], -u[0] * sa + u[2] * ca};  // R_y(a) u
      ylm(P, u, Yu);
      ylm(P, r, Yr);
      const double wq = gw[i] * 2.0 * kPi / NF;
      for (int n = 0; n <= P; ++n) {
        const int d = 2 * n + 1;
        for (int k = -n; k <= n; ++k) {
          const cd yr = Yr[n * n + n + k] * wq;
          for (int kp = -n; kp <= n; ++kp) acc[n][size_t(kp + n) * d + (k + n)] += yr * std::conj(Yu[n * n + n + kp]);
        }
      }
    }
  Xop.assign(P + 1, {});
  for (int n = 0; n <= P; ++n) {
    const int d = 2 * n + 1;
    Xop[n].assign(size_t(d) * d, 0.0);
    for (size_t e = 0; e < acc[n].size(); ++e) {
      if (std::fabs(acc[n][e].imag()) > 1e-12)
        throw std::runtime_error("helm_rot: rotation about y is not real (basis convention)");
      Xop[n][e] = acc[n][e].real();
    }
    // orthogonality check: X X^T = I
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) s += Xop[n][size_t(i) * d + k] * Xop[n][size_t(j) * d + k];
        if (std::fabs(s - (i == j ? 1.0 : 0.0)) > 1e-12) throw std::runtime_error("helm_rot: rotation not orthogonal");
      }
  }
}

// even / odd blocks of degree n from the full op-form map, as in k_h_build_split
void split_blocks(int n, const std::vector<double>& X, std::vector<double>& E, std::vector<double>& O) {
  const int d = 2 * n + 1;
  auto x = [&](int kp, int k) { return X[size_t(kp + n) * d + (k + n)]; };  // [out][in]
  E.assign(size_t(n + 1) * (n + 1), 0.0);
  O.assign(size_t(n) * n, 0.0);
  for (int kp = 0; kp <= n; ++kp)
    for (int k = 0; k <= n; ++k) {
      double v;
      if (k == 0)
        v = x(kp, 0) * (kp > 0 ? 2.0 : 1.0);
      else
        v = (x(kp, k) + x(kp, -k)) * (kp == 0 ? 0.5 : 1.0);
      E[size_t(kp) * (n + 1) + k] = v;
    }
  for (int kp = 1; kp <= n; ++kp)
    for (int k = 1; k <= n; ++k) O[size_t(kp - 1) * n + (k - 1)] = x(kp, k) - x(kp, -k);
}

}  // namespace

size_t hpas_frag_size(int s) { return size_t((s + 7) / 8) * 8 * size_t((s + 3) / 4) * 4; }

void hpas_to_frags(int s, const double* B, double* out) {
  const int MT = (s + 7) / 8, KS = (s + 3) / 4;
  for (int ks = 0; ks < KS; ++ks)
    for (int mt = 0; mt < MT; ++mt)
      for (int l = 0; l < 32; ++l) {
        const int i = mt * 8 + l / 4, j = ks * 4 + l % 4;
        out[size_t(ks * MT + mt) * 32 + l] = (i < s && j < s) ? B[size_t(i) * s + j] : 0.0;
      }
}

HpasLayout hpas_layout(int P) {
  HpasLayout L;
  size_t o = 0;
  for (int ph = 0; ph < 2; ++ph)  // W, V
    for (int par = 0; par < 2; ++par)
      for (int n = par; n <= P; ++n) {
        L.wv_off[ph][par].push_back(o);
        o += hpas_frag_size(n + 1 - par);
      }
  L.wv_stride = o;
  o = 0;
  for (int m = 0; m <= P; ++m) {
    L.z_off.push_back(o);
    o += hpas_frag_size(2 * (P + 1 - m));
  }
  L.z_stride = o;
  return L;
}

void hpas_build_wv(int P, const std::vector<double>& thetas, std::vector<double>& out) {
  const HpasLayout L = hpas_layout(P);
  out.assign(thetas.size() * L.wv_stride, 0.0);
  int err = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
  for (long c = 0; c < long(thetas.size()); ++c) {
    try {
      for (int ph = 0; ph < 2; ++ph) {
        std::vector<std::vector<double>> X;
        rot_y(P, ph == 0 ? thetas[c] : -thetas[c], X);  // W: R = Q^T = R_y(theta); V: R = Q = R_y(-theta)
        for (int n = 0; n <= P; ++n) {
          std::vector<double> E, O;
          split_blocks(n, X[n], E, O);
          hpas_to_frags(n + 1, E.data(), &out[c * L.wv_stride + L.wv_off[ph][0][n]]);
          if (n >= 1) hpas_to_frags(n, O.data(), &out[c * L.wv_stride + L.wv_off[ph][1][n - 1]]);
        }
      }
    } catch (...) {
      err |= 1;
    }
  }
  if (err) throw std::runtime_error("hpas_build_wv: rotation blocks failed their checks");
}

}  // namespace qbxg
