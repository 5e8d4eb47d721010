// ORACLE -- test infrastructure only.  Not part of the product path.
//
// CPU restatement of the GIGAQBX evaluation path (Algorithm 4, Stages 2-9,
// PAPER.md:2316-2432), of the expansion module
// and of direct QBX.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may load this library.
//
// Pinning: sph_harm / form / eval against the SPEC golden vectors
// (SPEC.md:99-101, 108-110, 117-119), translations against the SPEC identities
// (SPEC.md:126-128), and execute against the compiled reference qbx::direct_sum
// (oracle/_ref, built from /root/reference/proj/src/kernels.cpp) and against
// direct_qbx with the Theorem-1 decay.  See tests/.
//
// Formulation (also the GPU's): unnormalised solid harmonics without the
// Condon-Shortley phase,
//   R_n^m(x) = r^n P_n^|m|(cos t) e^{i m phi} / (n+|m|)!,
//   I_n^m(x) = (n-|m|)! P_n^|m|(cos t) e^{i m phi} / r^{n+1}       (m >= 0),
//   X_n^{-m} = (-1)^m conj(X_n^m),
// so 1/|x-y| = sum_{n,m} conj(R_n^m(y)) I_n^m(x) for |y| < |x|.  This is a
// rescaling of the paper's Eq. (3)-(4); the paper's local
// coefficients of Eq. (5) are recovered by paper_from_internal() below.
// Box coefficients are box-scaled: M~ = M / |b|^n, L~ = L |b|^n (and r_c^n at
// QBX centres) so one operator per relative offset serves every level.
//
// This file deliberately uses full complex (n, m in [-n, n]) tables and plain
// loops -- a different code shape from the GPU's half-table kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qbxg.h"

namespace {

using cd = std::complex<double>;
constexpr double kInv4Pi = 0.07957747154594766788;

inline int idx(int n, int m) { return n * n + n + m; }  // paper order B_0^0, B_1^-1, B_1^0, ...
inline int nfull(int p) { return (p + 1) * (p + 1); }

double factorial(int n) {
  double f = 1;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

// Associated Legendre P_n^m(x), m >= 0, no Condon-Shortley phase.
double legendre(int n, int m, double x) {
  double pmm = 1.0;
  const double s = std::sqrt(std::max(0.0, (1.0 - x) * (1.0 + x)));
  for (int i = 1; i <= m; ++i) pmm *= (2 * i - 1) * s;
  if (n == m) return pmm;
  double pm1 = x * (2 * m + 1) * pmm;
  if (n == m + 1) return pm1;
  double pn = 0;
  for (int k = m + 2; k <= n; ++k) {
    pn = ((2 * k - 1) * x * pm1 - (k + m - 1) * pmm) / (k - m);
    pmm = pm1;
    pm1 = pn;
  }
  return pn;
}

// Y_n^m of Eq. (4).
cd sph_harm(int n, int m, double theta, double phi) {
  const int am = std::abs(m);
  const double norm = std::sqrt((2 * n + 1) / (4 * M_PI) * factorial(n - am) / factorial(n + am));
  return norm * legendre(n, am, std::cos(theta)) * std::exp(cd(0, m * phi));
}

// All P_n^m(x), 0 <= m <= n <= P (no Condon-Shortley phase), in one O(P^2)
// pass of the same recurrences as legendre(); table index idx(n, m).
void legendre_table(int P, double x, std::vector<double>& T) {
  T.assign(nfull(P), 0.0);
  const double s = std::sqrt(std::max(0.0, (1.0 - x) * (1.0 + x)));
  double pmm = 1.0;
  for (int m = 0; m <= P; ++m) {
    if (m > 0) pmm *= (2 * m - 1) * s;
    T[idx(m, m)] = pmm;
    if (m + 1 > P) break;
    double a = pmm, b = x * (2 * m + 1) * pmm;
    T[idx(m + 1, m)] = b;
    for (int k = m + 2; k <= P; ++k) {
      const double c = ((2 * k - 1) * x * b - (k + m - 1) * a) / (k - m);
      T[idx(k, m)] = c;
      a = b;
      b = c;
    }
  }
}

struct FactTable {
  double f[200];
  FactTable() {
    f[0] = 1;
    for (int i = 1; i < 200; ++i) f[i] = f[i - 1] * i;
  }
};
const FactTable kFact;

// Regular / irregular solid harmonics by explicit spherical-coordinate
// evaluation (oracle style: trig azimuth, Legendre in cos(theta); no
// Cartesian recurrences).
void regular(const double* x, int P, std::vector<cd>& R) {
  thread_local std::vector<double> Pt;
  R.assign(nfull(P), cd(0));
  const double r = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
  const double ct = r > 0 ? x[2] / r : 1.0;
  const double phi = std::atan2(x[1], x[0]);
  legendre_table(P, ct, Pt);
  const cd e1 = std::exp(cd(0, phi));
  double rn = 1;
  for (int n = 0; n <= P; ++n) {
    cd em = 1.0;
    for (int m = 0; m <= n; ++m) {
      const cd v = rn * Pt[idx(n, m)] * em / kFact.f[n + m];
      R[idx(n, m)] = v;
      R[idx(n, -m)] = (m & 1 ? -1.0 : 1.0) * std::conj(v);
      em *= e1;
    }
    rn *= r;
  }
}

void irregular(const double* x, int P, std::vector<cd>& I) {
  thread_local std::vector<double> Pt;
  I.assign(nfull(P), cd(0));
  const double r = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
  if (r == 0) throw std::domain_error("irregular harmonic at the origin (source coincides with centre)");
  const double ct = x[2] / r;
  const double phi = std::atan2(x[1], x[0]);
  legendre_table(P, ct, Pt);
  const cd e1 = std::exp(cd(0, phi));
  double rn = 1.0 / r;
  for (int n = 0; n <= P; ++n) {
    cd em = 1.0;
    for (int m = 0; m <= n; ++m) {
      const cd v = kFact.f[n - m] * Pt[idx(n, m)] * em * rn;
      I[idx(n, m)] = v;
      I[idx(n, -m)] = (m & 1 ? -1.0 : 1.0) * std::conj(v);
      em *= e1;
    }
    rn /= r;
  }
}

inline cd at(const std::vector<cd>& T, int P, int n, int m) {
  if (n < 0 || n > P || std::abs(m) > n) return cd(0);
  return T[idx(n, m)];
}

// a . grad X_n^m via the ladder identities
//   d_z R_n^m = R_{n-1}^m, (d_x - i d_y) R_n^m = R_{n-1}^{m-1}, (d_x + i d_y) R_n^m = -R_{n-1}^{m+1}
//   d_z I_n^m = -I_{n+1}^m, (d_x - i d_y) I_n^m = I_{n+1}^{m-1}, (d_x + i d_y) I_n^m = -I_{n+1}^{m+1}
// with a.grad = a_z d_z + (a_x + i a_y)/2 (d_x - i d_y) + (a_x - i a_y)/2 (d_x + i d_y).
inline cd dir_deriv_regular(const std::vector<cd>& R, int P, int n, int m, const double* a) {
  const cd ap(a[0], a[1]), amn(a[0], -a[1]);
  return a[2] * at(R, P, n - 1, m) + 0.5 * ap * at(R, P, n - 1, m - 1) - 0.5 * amn * at(R, P, n - 1, m + 1);
}
inline cd dir_deriv_irregular(const std::vector<cd>& I, int P, int n, int m, const double* a) {
  const cd ap(a[0], a[1]), amn(a[0], -a[1]);
  return -a[2] * at(I, P, n + 1, m) + 0.5 * ap * at(I, P, n + 1, m - 1) - 0.5 * amn * at(I, P, n + 1, m + 1);
}

struct Src {
  const double* pos;
  const double* w;
  const double* mu;  // may be null
};

// ---- expansion kernels on box-scaled coefficients --------------------------
// P2M: M~ += w conj(R(u)) + conj(mu . grad R(u)) / h, u = (s - c)/h   (Eq. (10))
void p2m(const Src& S, int64_t s, const double* c, double h, int P, std::vector<cd>& M) {
  double u[3] = {(S.pos[3 * s] - c[0]) / h, (S.pos[3 * s + 1] - c[1]) / h, (S.pos[3 * s + 2] - c[2]) / h};
  thread_local std::vector<cd> R;
  regular(u, P, R);
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) {
      cd v = S.w[s] * std::conj(R[idx(n, m)]);
      if (S.mu) v += std::conj(dir_deriv_regular(R, P, n, m, &S.mu[3 * s])) / h;
      M[idx(n, m)] += v;
    }
}

// P2L at a centre with scale h: L~ += (1/h)[w conj(I(u)) + conj(mu . grad I(u))/h]   (Eq. (5)/(8))
void p2l(const Src& S, int64_t s, const double* c, double h, int P, std::vector<cd>& L) {
  double u[3] = {(S.pos[3 * s] - c[0]) / h, (S.pos[3 * s + 1] - c[1]) / h, (S.pos[3 * s + 2] - c[2]) / h};
  thread_local std::vector<cd> I;
  irregular(u, P + 1, I);
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) {
      cd v = S.w[s] * std::conj(I[idx(n, m)]);
      if (S.mu) v += std::conj(dir_deriv_irregular(I, P + 1, n, m, &S.mu[3 * s])) / h;
      L[idx(n, m)] += v / h;
    }
}

// Evaluate a box-scaled local (order P, scale h, centre c) at t: sum L~ R((t-c)/h)   (Eq. (9))
double eval_local(const std::vector<cd>& L, int P, const double* c, double h, const double* t) {
  double u[3] = {(t[0] - c[0]) / h, (t[1] - c[1]) / h, (t[2] - c[2]) / h};
  thread_local std::vector<cd> R;
  regular(u, P, R);
  cd acc = 0;
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) acc += L[idx(n, m)] * R[idx(n, m)];
  return acc.real();
}

// Evaluate a box-scaled multipole at t: (1/h) sum M~ I((t-c)/h)
double eval_multipole(const std::vector<cd>& M, int P, const double* c, double h, const double* t) {
  double u[3] = {(t[0] - c[0]) / h, (t[1] - c[1]) / h, (t[2] - c[2]) / h};
  thread_local std::vector<cd> I;
  irregular(u, P, I);
  cd acc = 0;
  for (int n = 0; n <= P; ++n)
    for (int m = -n; m <= n; ++m) acc += M[idx(n, m)] * I[idx(n, m)];
  return acc.real() / h;
}

// M2M: child (scale h, centre c) -> parent (scale H, centre C):
//   M_n^m(C) = sum_{j,k} M_j^k(c) conj(R_{n-j}^{m-k}(c - C))   (Greengard thesis Thm 3.5.4)
void m2m(const std::vector<cd>& Mc, int P, const double* c, double h, const double* C, double H, std::vector<cd>& Mp) {
  double d[3] = {(c[0] - C[0]) / h, (c[1] - C[1]) / h, (c[2] - C[2]) / h};
  thread_local std::vector<cd> R;
  regular(d, P, R);
  for (int n = 0; n <= P; ++n) {
    const double s = std::pow(h / H, n);
    for (int m = -n; m <= n; ++m) {
      cd acc = 0;
      for (int j = 0; j <= n; ++j)
        for (int k = -j; k <= j; ++k) acc += Mc[idx(j, k)] * std::conj(at(R, P, n - j, m - k));
      Mp[idx(n, m)] += s * acc;
    }
  }
}

// M2L: multipole (scale h, centre c) -> local (order Q, scale H, centre C):
//   L_n^m(C) = (-1)^{n+m} sum_{j,k} M_j^k I_{j+n}^{k-m}(C - c)   (Thm 3.5.5 restated for this basis)
void m2l(const std::vector<cd>& M, int P, const double* c, double h, const double* C, double H, int Q,
         std::vector<cd>& L) {
  double d[3] = {(C[0] - c[0]) / h, (C[1] - c[1]) / h, (C[2] - c[2]) / h};
  thread_local std::vector<cd> I;
  irregular(d, P + Q, I);
  for (int n = 0; n <= Q; ++n) {
    const double s = std::pow(H / h, n) / h;
    for (int m = -n; m <= n; ++m) {
      // |k - m| <= j + n always, so every I_{j+n}^{k-m} exists: the k-row of M and the
      // shifted row of I are contiguous in the packed table (interleaved re, im)
      double ar = 0.0, ai = 0.0;
      for (int j = 0; j <= P; ++j) {
        const double* Mj = reinterpret_cast<const double*>(&M[idx(j, 0)]);
        const double* Ij = reinterpret_cast<const double*>(&I[idx(j + n, -m)]);
#pragma omp simd reduction(+ : ar, ai)
        for (int k = -j; k <= j; ++k) {
          const double mr = Mj[2 * k], mi = Mj[2 * k + 1], ir = Ij[2 * k], ii = Ij[2 * k + 1];
          ar += mr * ir - mi * ii;
          ai += mr * ii + mi * ir;
        }
      }
      const cd acc(ar, ai);
      L[idx(n, m)] += s * (((n + m) & 1) ? -1.0 : 1.0) * acc;
    }
  }
}

// L2L: local (order P, scale h, centre c) -> local (order Q, scale H, centre C):
//   L_n^m(C) = sum_{j>=n,k} L_j^k R_{j-n}^{k-m}(C - c)   (Lem. 3.2 of the thesis)
void l2l(const std::vector<cd>& Lc, int P, const double* c, double h, const double* C, double H, int Q,
         std::vector<cd>& L) {
  double d[3] = {(C[0] - c[0]) / h, (C[1] - c[1]) / h, (C[2] - c[2]) / h};
  thread_local std::vector<cd> R;
  regular(d, P, R);
  for (int n = 0; n <= Q; ++n) {
    const double s = std::pow(H / h, n);
    for (int m = -n; m <= n; ++m) {
      cd acc = 0;
      for (int j = n; j <= P; ++j)
        for (int k = -j; k <= j; ++k) acc += Lc[idx(j, k)] * at(R, P, j - n, k - m);
      L[idx(n, m)] += s * acc;
    }
  }
}

inline double p2p(const Src& S, int64_t s, const double* t) {
  const double dx = t[0] - S.pos[3 * s], dy = t[1] - S.pos[3 * s + 1], dz = t[2] - S.pos[3 * s + 2];
  const double r2 = dx * dx + dy * dy + dz * dz;
  if (r2 == 0.0) throw std::domain_error("p2p: target coincides with source " + std::to_string(s));
  const double rinv = 1.0 / std::sqrt(r2);
  double v = S.w[s] * rinv;
  if (S.mu) v += (S.mu[3 * s] * dx + S.mu[3 * s + 1] * dy + S.mu[3 * s + 2] * dz) * rinv * rinv * rinv;
  return v;
}

// Paper normalisation of a local coefficient, Eq. (5): L^paper_n^m = L_n^m / (4 pi N_nm (n+m)!),
// N_nm = sqrt((2n+1)/(4 pi) (n-m)!/(n+m)!)  (for m >= 0).
double paper_factor(int n, int m) {
  const double N = std::sqrt((2 * n + 1) / (4 * M_PI) * factorial(n - m) / factorial(n + m));
  return 1.0 / (4 * M_PI * N * factorial(n + m));
}

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // namespace

extern "C" {

const char* qbxo_last_error(void) { return g_err.c_str(); }

// ---- expansion-module entry points used by the golden-vector tests --------
int qbxo_sph_harm(int n, int m, double theta, double phi, double* out_re_im) {
  return guard([&] {
    if (std::abs(m) > n || n < 0) throw std::invalid_argument("sph_harm: |m| > n");
    cd v = sph_harm(n, m, theta, phi);
    out_re_im[0] = v.real();
    out_re_im[1] = v.imag();
  });
}

// form_expansion(kind, sources, center, p) in the paper's normalisation (Eq. (5)/(10)),
// full table (p+1)^2 complex at index n^2+n+m.  kind 0 = multipole, 1 = local.
int qbxo_form_expansion(int kind, int64_t ns, const double* pos, const double* w, const double* mu,
                        const double* center, int p, double* out /*2*(p+1)^2*/) {
  return guard([&] {
    Src S{pos, w, mu};
    std::vector<cd> T(nfull(p), cd(0));
    for (int64_t s = 0; s < ns; ++s) {
      if (kind == 0)
        p2m(S, s, center, 1.0, p, T);
      else {
        double d2 = 0;
        for (int k = 0; k < 3; ++k) d2 += (pos[3 * s + k] - center[k]) * (pos[3 * s + k] - center[k]);
        if (d2 == 0) throw std::domain_error("form_expansion: source coincides with centre");
        p2l(S, s, center, 1.0, p, T);
      }
    }
    for (int n = 0; n <= p; ++n)
      for (int m = -n; m <= n; ++m) {
        // paper multipole: M^paper = sum w/(2n+1) r^n Y_n^m = M_int * conj-normalisation ...
        cd v = T[idx(n, m)];
        const int am = std::abs(m);
        const double N = std::sqrt((2 * n + 1) / (4 * M_PI) * factorial(n - am) / factorial(n + am));
        cd pv;
        if (kind == 1) {
          // internal L = sum w conj(I_n^m) = sum w (n-|m|)! P e^{-im phi}/r^{n+1} (m>=0)
          // paper L = sum w/(2n+1) Y_n^{-m}/r^{n+1} = sum w N P e^{-im phi}/((2n+1) r^{n+1})
          pv = v * (N / ((2 * n + 1) * factorial(n - am)));
          if (m < 0 && (am & 1)) pv = -pv;
        } else {
          // internal M = sum w conj(R_n^m) = sum w r^n P e^{-im phi}/(n+|m|)!
          // paper M = sum w/(2n+1) r^n Y_n^m = sum w N r^n P e^{im phi}/(2n+1)
          pv = std::conj(v) * (N * factorial(n + am) / (2 * n + 1));
          if (m < 0 && (am & 1)) pv = -pv;
        }
        out[2 * idx(n, m)] = pv.real();
        out[2 * idx(n, m) + 1] = pv.imag();
      }
  });
}

// eval_expansion in the paper's normalisation: real part.
int qbxo_eval_expansion(int kind, const double* coeffs, int p, const double* center, const double* t,
                        double* out) {
  return guard([&] {
    double d[3] = {t[0] - center[0], t[1] - center[1], t[2] - center[2]};
    const double r = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (kind == 0 && r == 0) throw std::domain_error("eval_expansion: multipole evaluated at its centre");
    const double th = r > 0 ? std::acos(std::max(-1.0, std::min(1.0, d[2] / r))) : 0.0;
    const double ph = std::atan2(d[1], d[0]);
    cd acc = 0;
    for (int n = 0; n <= p; ++n)
      for (int m = -n; m <= n; ++m) {
        cd c(coeffs[2 * idx(n, m)], coeffs[2 * idx(n, m) + 1]);
        if (kind == 1)
          acc += c * std::pow(r, n) * sph_harm(n, m, th, ph);
        else
          acc += c / std::pow(r, n + 1) * sph_harm(n, -m, th, ph);
      }
    *out = acc.real();
  });
}

// Internal-basis translation entry points for the identity tests.
// Tables are full complex (p+1)^2, scale 1 (unscaled coefficients).
int qbxo_translate(int kind /*0 M2M, 1 M2L, 2 L2L*/, const double* in, int p, const double* c, const double* C,
                   int q, double* out) {
  return guard([&] {
    std::vector<cd> A(nfull(p)), B(nfull(q), cd(0));
    for (int i = 0; i < nfull(p); ++i) A[i] = cd(in[2 * i], in[2 * i + 1]);
    if (kind == 0) {
      if (q != p) throw std::invalid_argument("M2M: q must equal p");
      m2m(A, p, c, 1.0, C, 1.0, B);
    } else if (kind == 1) {
      m2l(A, p, c, 1.0, C, 1.0, q, B);
    } else {
      l2l(A, p, c, 1.0, C, 1.0, q, B);
    }
    for (int i = 0; i < nfull(q); ++i) {
      out[2 * i] = B[i].real();
      out[2 * i + 1] = B[i].imag();
    }
  });
}

// Internal-basis formation / evaluation (scale 1, full table, no 1/4pi).
int qbxo_form_internal(int kind, int64_t ns, const double* pos, const double* w, const double* mu,
                       const double* center, int p, double* out) {
  return guard([&] {
    Src S{pos, w, mu};
    std::vector<cd> T(nfull(p), cd(0));
    for (int64_t s = 0; s < ns; ++s) {
      if (kind == 0)
        p2m(S, s, center, 1.0, p, T);
      else
        p2l(S, s, center, 1.0, p, T);
    }
    for (int i = 0; i < nfull(p); ++i) {
      out[2 * i] = T[i].real();
      out[2 * i + 1] = T[i].imag();
    }
  });
}

int qbxo_eval_internal(int kind, const double* coeffs, int p, const double* center, const double* t, double* out) {
  return guard([&] {
    std::vector<cd> T(nfull(p));
    for (int i = 0; i < nfull(p); ++i) T[i] = cd(coeffs[2 * i], coeffs[2 * i + 1]);
    *out = kind == 0 ? eval_multipole(T, p, center, 1.0, t) : eval_local(T, p, center, 1.0, t);
  });
}

// ---- Algorithm 4, Stages 2-9 ------------------------------
// Inputs in the caller's original ordering; outputs likewise.  Potentials
// include 1/(4 pi).  out_center_coeffs (optional): n_centers x K_q complex in
// the paper normalisation, m >= 0, index n(n+1)/2+m.
// stage_seconds (optional, 8 entries): stage 2, 3+5a+6a, 4, 5b, 6b, 7, 8, 9.
// Sharded variant (test harness for the multi-rank protocol):
// mask = per-box role bits from qbxg_plan_shard (NULL: everything), phase 1 =
// upward pass of owned leaves/subtrees into Mbuf (nb x (p+1)^2 complex, other
// rows zero), phase 2 = straddling M2M from Mbuf then Stages 3-9 of the owned
// boxes (other targets/centres written as 0), phase 3 = both.
int execute_impl(const qbxg_plan_view* V, int p, int q, const double* src_pos, const double* center_pos,
                 const double* center_radius, const double* target_pos, const int32_t* association,
                 const double* weights, const double* dipoles, double* out_pot, double* out_center_coeffs,
                 double* stage_seconds, const uint8_t* mask, int phase, double* Mbuf);

int qbxo_execute(const qbxg_plan_view* V, int p, int q, double tf, const double* src_pos,
                 const double* center_pos, const double* center_radius, const double* target_pos,
                 const int32_t* association, const double* weights, const double* dipoles, double* out_pot,
                 double* out_center_coeffs, double* stage_seconds) {
  (void)tf;
  return execute_impl(V, p, q, src_pos, center_pos, center_radius, target_pos, association, weights, dipoles,
                      out_pot, out_center_coeffs, stage_seconds, nullptr, 3, nullptr);
}

int qbxo_execute_phase(const qbxg_plan_view* V, int p, int q, const double* src_pos, const double* center_pos,
                       const double* center_radius, const double* target_pos, const int32_t* association,
                       const double* weights, const double* dipoles, double* out_pot, double* out_center_coeffs,
                       const uint8_t* mask, int phase, double* Mbuf) {
  return execute_impl(V, p, q, src_pos, center_pos, center_radius, target_pos, association, weights, dipoles,
                      out_pot, out_center_coeffs, nullptr, mask, phase, Mbuf);
}

int execute_impl(const qbxg_plan_view* V, int p, int q, const double* src_pos, const double* center_pos,
                 const double* center_radius, const double* target_pos, const int32_t* association,
                 const double* weights, const double* dipoles, double* out_pot, double* out_center_coeffs,
                 double* stage_seconds, const uint8_t* mask, int phase, double* Mbuf) {
  return guard([&] {
    const int nb = V->n_boxes;
    const int KP = nfull(p), KQ = nfull(q);
    Src S{src_pos, weights, dipoles};
    auto now = [] {
      return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    auto has = [&](int b, uint8_t bit) { return mask ? (mask[b] & bit) != 0 : true; };
    auto straddle = [&](int b) { return mask ? (mask[b] & QBXG_SHARD_STRADDLE) != 0 : false; };
    double t[9];
    t[0] = now();
    // box-sorted views: source s_sorted -> original index src_perm[s_sorted]
    std::vector<std::vector<cd>> M(nb, std::vector<cd>(KP, cd(0)));
    auto src_of = [&](int64_t sorted) { return int64_t(V->src_perm[sorted]); };
    auto m2m_level = [&](int l, bool want_straddle) {
#pragma omp parallel for schedule(dynamic, 16)
      for (int i = V->level_starts[l]; i < V->level_starts[l + 1]; ++i) {
        const int b = V->level_boxes[i];
        if (want_straddle ? !straddle(b) : !has(b, QBXG_SHARD_SUBTREE)) continue;
        for (int k = V->child_starts[b]; k < V->child_starts[b + 1]; ++k) {
          const int c = V->children[k];
          if (V->src_sub_count[c] == 0) continue;
          m2m(M[c], p, &V->box_center[3 * c], V->box_radius[c], &V->box_center[3 * b], V->box_radius[b], M[b]);
        }
      }
    };

    if (phase & 1) {
      // Stage 2: form multipoles (leaves), then M2M in postorder (children have larger ids).
#pragma omp parallel for schedule(dynamic, 16)
      for (int b = 0; b < nb; ++b) {
        if (V->child_starts[b + 1] != V->child_starts[b] || !has(b, QBXG_SHARD_OWN)) continue;
        for (int i = 0; i < V->src_own_count[b]; ++i)
          p2m(S, src_of(V->src_own_start[b] + i), &V->box_center[3 * b], V->box_radius[b], p, M[b]);
      }
      for (int l = V->n_levels - 2; l >= 0; --l) m2m_level(l, false);
      if (Mbuf)
        for (int b = 0; b < nb; ++b)
          for (int i = 0; i < KP; ++i) {
            Mbuf[2 * (size_t(b) * KP + i)] = M[b][i].real();
            Mbuf[2 * (size_t(b) * KP + i) + 1] = M[b][i].imag();
          }
    }
    if (!(phase & 2)) return;
    if (!(phase & 1) && Mbuf)
      for (int b = 0; b < nb; ++b)
        for (int i = 0; i < KP; ++i) M[b][i] = cd(Mbuf[2 * (size_t(b) * KP + i)], Mbuf[2 * (size_t(b) * KP + i) + 1]);
    if (mask)
      for (int l = V->n_levels - 2; l >= 0; --l) m2m_level(l, true);
    t[1] = now();

    const int64_t nc = V->n_centers;
    std::vector<std::vector<cd>> Lc(nc, std::vector<cd>(KQ, cd(0)));  // indexed by sorted centre position
    const int64_t nconv = V->n_conv_targets;
    std::vector<double> phi_conv(nconv, 0.0);  // sorted conventional-target position

    // Stages 3, 5a, 6a: direct interactions from U, W_close, X_close (targets in the box only)
    const int near_lists[3] = {QBXG_LIST_U, QBXG_LIST_W_CLOSE, QBXG_LIST_X_CLOSE};
#pragma omp parallel for schedule(dynamic, 4)
    for (int b = 0; b < nb; ++b) {
      if (!(V->box_flags[b] & QBXG_BOX_TARGET) || !has(b, QBXG_SHARD_OWN)) continue;
      for (int li : near_lists) {
        for (int64_t e = V->list_starts[li][b]; e < V->list_starts[li][b + 1]; ++e) {
          const int d = V->list_boxes[li][e];
          for (int i = 0; i < V->src_own_count[d]; ++i) {
            const int64_t s = src_of(V->src_own_start[d] + i);
            for (int j = 0; j < V->ctr_own_count[b]; ++j) {
              const int64_t cs = V->ctr_own_start[b] + j;
              const int64_t c = V->ctr_perm[cs];
              p2l(S, s, &center_pos[3 * c], center_radius[c], q, Lc[cs]);
            }
            for (int j = 0; j < V->tgt_own_count[b]; ++j) {
              const int64_t ts = V->tgt_own_start[b] + j;
              phi_conv[ts] += p2p(S, s, &target_pos[3 * int64_t(V->tgt_perm[ts])]);
            }
          }
        }
      }
    }
    t[2] = now();

    // Stage 4: M2L over List 2
    std::vector<std::vector<cd>> Lb(nb, std::vector<cd>(KP, cd(0)));
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int64_t e = V->list_starts[QBXG_LIST_V][b]; has(b, QBXG_SHARD_DOWN) && e < V->list_starts[QBXG_LIST_V][b + 1];
           ++e) {
        const int d = V->list_boxes[QBXG_LIST_V][e];
        m2l(M[d], p, &V->box_center[3 * d], V->box_radius[d], &V->box_center[3 * b], V->box_radius[b], p, Lb[b]);
      }
    t[3] = now();

    // Stage 5b: List 3 far: M2P at conventional targets, M2QBXL at centres
#pragma omp parallel for schedule(dynamic, 4)
    for (int b = 0; b < nb; ++b) {
      if (!(V->box_flags[b] & QBXG_BOX_TARGET) || !has(b, QBXG_SHARD_OWN)) continue;
      for (int64_t e = V->list_starts[QBXG_LIST_W_FAR][b]; e < V->list_starts[QBXG_LIST_W_FAR][b + 1]; ++e) {
        const int d = V->list_boxes[QBXG_LIST_W_FAR][e];
        for (int j = 0; j < V->ctr_own_count[b]; ++j) {
          const int64_t cs = V->ctr_own_start[b] + j;
          const int64_t c = V->ctr_perm[cs];
          m2l(M[d], p, &V->box_center[3 * d], V->box_radius[d], &center_pos[3 * c], center_radius[c], q, Lc[cs]);
        }
        for (int j = 0; j < V->tgt_own_count[b]; ++j) {
          const int64_t ts = V->tgt_own_start[b] + j;
          phi_conv[ts] += eval_multipole(M[d], p, &V->box_center[3 * d], V->box_radius[d],
                                         &target_pos[3 * int64_t(V->tgt_perm[ts])]);
        }
      }
    }
    t[4] = now();

    // Stage 6b: List 4 far: P2L into the box local
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int64_t e = V->list_starts[QBXG_LIST_X_FAR][b];
           has(b, QBXG_SHARD_DOWN) && e < V->list_starts[QBXG_LIST_X_FAR][b + 1]; ++e) {
        const int d = V->list_boxes[QBXG_LIST_X_FAR][e];
        for (int i = 0; i < V->src_own_count[d]; ++i)
          p2l(S, src_of(V->src_own_start[d] + i), &V->box_center[3 * b], V->box_radius[b], p, Lb[b]);
      }
    t[5] = now();

    // Stage 7: L2L in preorder (parents have smaller level)
    for (int l = 1; l < V->n_levels; ++l) {
#pragma omp parallel for schedule(dynamic, 16)
      for (int i = V->level_starts[l]; i < V->level_starts[l + 1]; ++i) {
        const int b = V->level_boxes[i];
        if (!(V->box_flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR)) || !has(b, QBXG_SHARD_DOWN)) continue;
        const int a = V->box_parent[b];
        l2l(Lb[a], p, &V->box_center[3 * a], V->box_radius[a], &V->box_center[3 * b], V->box_radius[b], p, Lb[b]);
      }
    }
    t[6] = now();

    // Stage 8: L2QBXL at every centre from its owning box's local
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int j = 0; has(b, QBXG_SHARD_OWN) && j < V->ctr_own_count[b]; ++j) {
        const int64_t cs = V->ctr_own_start[b] + j;
        const int64_t c = V->ctr_perm[cs];
        l2l(Lb[b], p, &V->box_center[3 * b], V->box_radius[b], &center_pos[3 * c], center_radius[c], q, Lc[cs]);
      }
    t[7] = now();

    // Stage 9: evaluate
    std::vector<int64_t> ctr_sorted_pos(nc);
    for (int64_t cs = 0; cs < nc; ++cs) ctr_sorted_pos[V->ctr_perm[cs]] = cs;
    std::vector<uint8_t> ctr_owned(nc, 1);
    if (mask)
      for (int b = 0; b < nb; ++b)
        for (int j = 0; j < V->ctr_own_count[b]; ++j) ctr_owned[V->ctr_own_start[b] + j] = has(b, QBXG_SHARD_OWN);
    const int64_t nt = V->n_targets;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t a = association[i];
      if (a >= 0) {
        const int64_t cs = ctr_sorted_pos[a];
        out_pot[i] = ctr_owned[cs] ? kInv4Pi * eval_local(Lc[cs], q, &center_pos[3 * int64_t(a)], center_radius[a],
                                                          &target_pos[3 * i])
                                   : 0.0;
      }
    }
#pragma omp parallel for schedule(dynamic, 16)
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < V->tgt_own_count[b]; ++j) {
        if (!has(b, QBXG_SHARD_OWN)) {
          out_pot[V->tgt_perm[V->tgt_own_start[b] + j]] = 0.0;
          continue;
        }
        const int64_t ts = V->tgt_own_start[b] + j;
        const int64_t ti = V->tgt_perm[ts];
        const double lf = eval_local(Lb[b], p, &V->box_center[3 * b], V->box_radius[b], &target_pos[3 * ti]);
        out_pot[ti] = kInv4Pi * (phi_conv[ts] + lf);
      }
    if (out_center_coeffs) {
      const int kq = (q + 1) * (q + 2) / 2;
#pragma omp parallel for schedule(static)
      for (int64_t cs = 0; cs < nc; ++cs) {
        const int64_t c = V->ctr_perm[cs];
        const double r = center_radius[c];
        for (int n = 0; n <= q; ++n)
          for (int m = 0; m <= n; ++m) {
            const cd v = ctr_owned[cs] ? Lc[cs][idx(n, m)] / std::pow(r, n) * paper_factor(n, m) : cd(0);
            out_center_coeffs[2 * (c * kq + n * (n + 1) / 2 + m)] = v.real();
            out_center_coeffs[2 * (c * kq + n * (n + 1) / 2 + m) + 1] = v.imag();
          }
      }
    }
    t[8] = now();
    if (stage_seconds)
      for (int k = 0; k < 8; ++k) stage_seconds[k] = t[k + 1] - t[k];
  });
}

// ---- direct QBX: every centre's local from ALL sources ------
int qbxo_direct_qbx(int64_t ns, const double* src_pos, const double* weights, const double* dipoles, int64_t nc,
                    const double* center_pos, const double* center_radius, int64_t nt, const double* target_pos,
                    const int32_t* association, int q, double* out_pot) {
  return guard([&] {
    Src S{src_pos, weights, dipoles};
    const int KQ = nfull(q);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t a = association[i];
      const double* t = &target_pos[3 * i];
      if (a >= 0) {
        std::vector<cd> L(KQ, cd(0));
        for (int64_t s = 0; s < ns; ++s) p2l(S, s, &center_pos[3 * int64_t(a)], center_radius[a], q, L);
        out_pot[i] = kInv4Pi * eval_local(L, q, &center_pos[3 * int64_t(a)], center_radius[a], t);
      } else {
        double acc = 0;
        for (int64_t s = 0; s < ns; ++s) acc += p2p(S, s, t);
        out_pot[i] = kInv4Pi * acc;
      }
    }
  });
}

}  // extern "C"
