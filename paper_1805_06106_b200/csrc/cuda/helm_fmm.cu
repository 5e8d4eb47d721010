// Helmholtz single-layer FMM stages (BASELINE config 3) on the
// tree, lists and stage order of the Laplace path; complex densities and
// potentials, full tables (p+1)^2, formulation of oracle/helm_oracle.cpp:
//   multipole M = ik sum w j_n conj(Y), phi = sum M h_n Y;  local L = ik sum w h_n conj(Y), phi = sum L j_n Y
//   E_n^m(x+t) = sum_{n',m'} [4 pi sum_l i^{n'+l-n} G(n,m;n',m';l) F_l^{m-m'}(t)] E'_{n'}^{m'}(x)
// Operators are not scale invariant: M2M / L2L use one dense complex operator per
// (level, octant), M2L one per (level, offset), all built on the device from the
// Gaunt table; M2L applies them as operator-batched complex GEMMs (CUDA cores)
// into CSR-ordered staging rows reduced per target box.  The centre translations
// (M2QBXL, L2QBXL) contract the box expansion with the Gaunt table once per box
// and azimuthal index mu -- C_mu(n',m',l) = 4 pi sum_n i^{n'+l-n} G X_n^{m'+mu} --
// and each centre then only needs its wave-function column F_l^mu(c - c_box):
// (q+1)^2 (p+q+1) work per centre and mu instead of a per-centre operator.
// Every output has one owner and a fixed summation order (deterministic).
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "helm.cuh"
#include "helm_math.cuh"

namespace qbxg {
namespace dev {
namespace {

using namespace hm;

__device__ __forceinline__ void nm_of(int i, int& n, int& m) {
  n = int(sqrt(double(i)));
  while (n * n > i) --n;
  while ((n + 1) * (n + 1) <= i) ++n;
  m = i - n * n - n;
}

// Recurrence coefficients of the fully normalised solid harmonics
// S_n^m(v) = |v|^n Y_n^m(v/|v|) (m >= 0), a polynomial in (x, y, z):
//   S_m^m = a_m (x + i y) S_{m-1}^{m-1},  S_{m+1}^m = b_m z S_m^m,
//   S_n^m = c_nm (z S_{n-1}^m - d_nm |v|^2 S_{n-2}^m)
// (the normalised-Legendre recurrences times |v|^n; no trigonometry, no square roots
// per pair).  Filled by helm_upload_constants().
constexpr int kHSolid = 42;  // degrees covered: operator tables need 2p (p <= 20) + 1
__constant__ double c_sa[kHSolid + 1], c_sb[kHSolid + 1];
__constant__ double c_sc[(kHSolid + 1) * (kHSolid + 1)], c_sd[(kHSolid + 1) * (kHSolid + 1)];
// the same tables in global memory, for loops whose lanes index different orders m (the
// constant cache serialises divergent addresses; these go through L1 coalesced)
__device__ double g_sa[kHSolid + 1], g_sb[kHSolid + 1];
__device__ double g_sap[kHSolid + 1];  // Y_0^0 prod_{i <= m} sa_i: the diagonal S_m^m = g_sap[m] (x + i y)^m
__device__ double g_sc[(kHSolid + 1) * (kHSolid + 1)], g_sd[(kHSolid + 1) * (kHSolid + 1)];

// j_n(k r) / r^n and y_n(k r) / r^n for n <= Q without divisions in the loops:
//   Jt_n = j_n / r^n:  series for Jt_Q, Jt_{Q+1} (x < 1), then Jt_{n-1} = (2n+1)/k Jt_n - r^2 Jt_{n+1}
//   Yt_n = y_n / r^n:  Yt_{n+1} = ((2n+1)/k Yt_n - Yt_{n-1}) / r^2
constexpr int kHSer = 14;
__constant__ double c_jser[(kHSolid + 2) * kHSer];  // -1/(2 t (2n+2t+1))
__constant__ double c_odd[2 * kHSolid + 4];          // 2n+1 and 1/(2n+1) interleaved

template <int Q>
__device__ __forceinline__ void radial_over_rn(double k, double r, double ir, double2 (&g)[Q + 1]) {
  const double x = k * r, x2 = x * x, r2 = r * r, ik = 1.0 / k, ir2 = ir * ir;
  double jt[Q + 2];
  if (x < 1.0) {
    double kn = 1.0;  // k^n / (2n+1)!!
    for (int n = 1; n <= Q; ++n) kn *= k * c_odd[2 * n + 1];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = Q + e;
      if (e == 1) kn *= k * c_odd[2 * n + 1];
      double term = 1.0, sum = 1.0;
#pragma unroll
      for (int t = 1; t <= kHSer; ++t) {
        term *= x2 * c_jser[n * kHSer + t - 1];
        sum += term;
      }
      jt[n] = kn * sum;
    }
#pragma unroll
    for (int n = Q + 1; n >= 1; --n) {
      const double nxt = n + 1 <= Q + 1 ? jt[n + 1] : 0.0;
      if (n <= Q) jt[n - 1] = c_odd[2 * n] * ik * jt[n] - r2 * nxt;
      else jt[n - 1] = jt[n - 1];
    }
  } else {
    double jq[Q + 1];
    sph_j_upto<Q>(x, jq);
    double irn = 1.0;
#pragma unroll
    for (int n = 0; n <= Q; ++n) {
      jt[n] = jq[n] * irn;
      irn *= ir;
    }
  }
  double sn, cs;
  sincos(x, &sn, &cs);
  const double ix = ik * ir;
  double ym = -cs * ix, y0 = (-cs * ix * ix - sn * ix) * ir;
#pragma unroll
  for (int n = 0; n <= Q; ++n) {
    double yn;
    if (n == 0) {
      yn = ym;
    } else if (n == 1) {
      yn = y0;
    } else {
      yn = (c_odd[2 * (n - 1)] * ik * y0 - ym) * ir2;
      ym = y0;
      y0 = yn;
    }
    g[n] = make_double2(jt[n], yn);
  }
}

// runtime-degree radial table rad[n] = (j_n(k r) + i s y_n(k r)) / r^n, n <= P,
// division-free recurrences as above (series for x < 1, Miller's recurrence above);
// computed by one thread
__device__ void radial_table(double k, double r, int P, bool singular, double2* rad) {
  const double x = k * r, x2 = x * x, r2 = r * r, ik = 1.0 / k, ir = 1.0 / r, ir2 = ir * ir;
  if (x < 1.0) {
    double kn = 1.0;
    for (int n = 1; n <= P; ++n) kn *= k * c_odd[2 * n + 1];
    double jt[2];
    for (int e = 0; e < 2; ++e) {
      const int n = P + e;
      if (e == 1) kn *= k * c_odd[2 * n + 1];
      double term = 1.0, sum = 1.0;
      for (int t = 1; t <= kHSer; ++t) {
        term *= x2 * c_jser[n * kHSer + t - 1];
        sum += term;
      }
      jt[e] = kn * sum;
    }
    double jn = jt[0], jn1 = jt[1];
    rad[P].x = jn;
    for (int n = P; n >= 1; --n) {
      const double jm = c_odd[2 * n] * ik * jn - r2 * jn1;
      jn1 = jn;
      jn = jm;
      rad[n - 1].x = jm;
    }
  } else {
    sph_j_upto_rt(P, x, ir, rad);
  }
  if (singular) {
    double sn, cs;
    sincos(x, &sn, &cs);
    const double ix = ik * ir;
    double ym = -cs * ix, y0 = (-cs * ix * ix - sn * ix) * ir;
    rad[0].y = ym;
    if (P >= 1) rad[1].y = y0;
    for (int n = 2; n <= P; ++n) {
      const double yn = (c_odd[2 * (n - 1)] * ik * y0 - ym) * ir2;
      ym = y0;
      y0 = yn;
      rad[n].y = yn;
    }
  } else {
    for (int n = 0; n <= P; ++n) rad[n].y = 0.0;
  }
}

// column mu >= 0 of the solid harmonics S_n^mu(v), n = mu..P, into out[n] (one thread)
__device__ __forceinline__ void solid_column(int mu, int P, double vx, double vy, double vz, double r2, double2* out) {
  double2 d = make_double2(0.28209479177387814347, 0.0);  // S_0^0 = 1/sqrt(4 pi)
  for (int i = 1; i <= mu; ++i)
    d = make_double2(c_sa[i] * (d.x * vx - d.y * vy), c_sa[i] * (d.x * vy + d.y * vx));
  out[mu] = d;
  if (mu + 1 > P) return;
  double2 a = d, b = make_double2(c_sb[mu] * vz * d.x, c_sb[mu] * vz * d.y);
  out[mu + 1] = b;
  for (int n = mu + 2; n <= P; ++n) {
    const double cn = c_sc[n * (kHSolid + 1) + mu], dn = c_sd[n * (kHSolid + 1) + mu] * r2;
    const double2 c2 = make_double2(cn * (vz * b.x - dn * a.x), cn * (vz * b.y - dn * a.y));
    out[n] = c2;
    a = b;
    b = c2;
  }
}

// cooperative wave-function table F[fi(l, mu)] = rad_l Y_l^mu(t) = (rad_l / r^l) S_l^mu(t),
// l <= P: threads 0..P build one solid-harmonic column each (Cartesian recurrences),
// thread 0 the radial table; rad = j_l (regular) or h_l = j_l + i y_l (singular).
// `rad` must hold P + 1 entries; F (P+1)^2.  Ends with __syncthreads.
__device__ void wave_table_cta(double k, int P, double tx, double ty, double tz, bool singular, double2* F,
                               double2* rad) {
  const double r2 = tx * tx + ty * ty + tz * tz;
  const double r = sqrt(r2);
  if (threadIdx.x == 32 || (blockDim.x <= 32 && threadIdx.x == 0)) radial_table(k, r, P, singular, rad);
  for (int m = threadIdx.x; m <= P; m += blockDim.x) {
    // column m into F[fi(n, m)] (n = m..P), mirrored to -m
    double2 d = make_double2(0.28209479177387814347, 0.0);
    for (int i = 1; i <= m; ++i)
      d = make_double2(g_sa[i] * (d.x * tx - d.y * ty), g_sa[i] * (d.x * ty + d.y * tx));
    F[fi(m, m)] = d;
    if (m + 1 <= P) {
      double2 a = d, b = make_double2(g_sb[m] * tz * d.x, g_sb[m] * tz * d.y);
      F[fi(m + 1, m)] = b;
      for (int n = m + 2; n <= P; ++n) {
        const double cn = g_sc[n * (kHSolid + 1) + m], dn = g_sd[n * (kHSolid + 1) + m] * r2;
        const double2 c2 = make_double2(cn * (tz * b.x - dn * a.x), cn * (tz * b.y - dn * a.y));
        F[fi(n, m)] = c2;
        a = b;
        b = c2;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (P + 1) * (P + 1); i += blockDim.x) {
    int n, m;
    nm_of(i, n, m);
    double2 v = F[fi(n, m < 0 ? -m : m)];
    if (m < 0) v.y = -v.y;  // S_n^{-m} = conj(S_n^m)
    F[i] = make_double2(v.x, v.y);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (P + 1) * (P + 1); i += blockDim.x) {
    int n, m;
    nm_of(i, n, m);
    F[i] = cmul(F[i], rad[n]);
  }
  __syncthreads();
}

__global__ void k_h_gather(int64_t ns, const int* __restrict__ perm, const double* __restrict__ w,
                           const double* __restrict__ mu, double2* __restrict__ hw, double2* __restrict__ hmu) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const int64_t o = perm[i];
  hw[i] = make_double2(w[2 * o], w[2 * o + 1]);
  if (mu)
    for (int d = 0; d < 3; ++d) hmu[3 * i + d] = make_double2(mu[6 * o + 2 * d], mu[6 * o + 2 * d + 1]);
}

// Double layer on a CTA-shared wave table F (order PF >= n + 1, index n^2 + n + m):
// mu . grad_v F_n^m by the ladder identities (dipole_terms in helm_math.cuh)
__device__ double2 grad_dot_tab(double k, const double2* F, int PF, int n, int m, const double2 (&mu)[3]) {
  auto at = [&](int nn, int mm) -> double2 {
    if (nn < 0 || nn > PF || mm > nn || -mm > nn) return make_double2(0.0, 0.0);
    return F[fi(nn, mm)];
  };
  const double dn = n, dm = m;
  const double a0 = lad_sq((dn * dn - dm * dm) / ((2 * dn - 1) * (2 * dn + 1)));
  const double a1 = lad_sq(((dn + 1) * (dn + 1) - dm * dm) / ((2 * dn + 1) * (2 * dn + 3)));
  const double c = lad_sq((dn - dm - 1) * (dn - dm) / ((2 * dn - 1) * (2 * dn + 1)));
  const double e = lad_sq((dn + dm + 1) * (dn + dm + 2) / ((2 * dn + 1) * (2 * dn + 3)));
  const double f = lad_sq((dn + dm - 1) * (dn + dm) / ((2 * dn - 1) * (2 * dn + 1)));
  const double g = lad_sq((dn - dm + 1) * (dn - dm + 2) / ((2 * dn + 1) * (2 * dn + 3)));
  const double2 Fa = at(n - 1, m), Fb = at(n + 1, m);
  const double2 dz = make_double2(k * (a0 * Fa.x - a1 * Fb.x), k * (a0 * Fa.y - a1 * Fb.y));
  const double sp = m >= 0 ? -k : k, sm = m > 0 ? k : -k;
  const double2 Fc = at(n - 1, m + 1), Fe = at(n + 1, m + 1), Ff = at(n - 1, m - 1), Fg = at(n + 1, m - 1);
  const double2 dp = make_double2(sp * (c * Fc.x + e * Fe.x), sp * (c * Fc.y + e * Fe.y));
  const double2 dmi = make_double2(sm * (f * Ff.x + g * Fg.x), sm * (f * Ff.y + g * Fg.y));
  const double2 hp = make_double2(0.5 * (mu[0].x + mu[1].y), 0.5 * (mu[0].y - mu[1].x));
  const double2 hm = make_double2(0.5 * (mu[0].x - mu[1].y), 0.5 * (mu[0].y + mu[1].x));
  double2 t = cmul(mu[2], dz);
  t = cfma(hp, dp, t);
  return cfma(hm, dmi, t);
}

// Stage 2 P2M at leaves: M_b += ik w conj(R_n^m(s - c_b))
__global__ void __launch_bounds__(256) k_h_p2m(HelmData H, const int* __restrict__ boxes) {
  extern __shared__ double2 sm[];
  double2* R = sm;
  double2* rad = sm + H.KP;
  const int b = boxes[blockIdx.x];
  const double4 bc = H.box[b];
  const int s0 = H.src_own_start[b], ns = H.src_own_count[b];
  const int PF = H.hmu ? H.P + 1 : H.P;  // the double layer needs one more degree
  rad = sm + (PF + 1) * (PF + 1);
  double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
  for (int si = 0; si < ns; ++si) {
    const double4 x = H.src[s0 + si];
    const double2 w = H.hw[s0 + si];
    __syncthreads();
    wave_table_cta(H.k, PF, x.x - bc.x, x.y - bc.y, x.z - bc.z, false, R, rad);
    const double2 f = make_double2(-H.k * w.y, H.k * w.x);  // ik w
    int slot = 0;
    for (int i = threadIdx.x; i < H.KP; i += blockDim.x, ++slot)
      acc[slot] = cfma(f, make_double2(R[i].x, -R[i].y), acc[slot]);
    if (H.hmu) {  // + ik mu . grad_s conj(R_n^m)(s - c) = ik mu . grad R_n^{-m}
      const double2 mu[3] = {H.hmu[3 * size_t(s0 + si)], H.hmu[3 * size_t(s0 + si) + 1], H.hmu[3 * size_t(s0 + si) + 2]};
      slot = 0;
      for (int i = threadIdx.x; i < H.KP; i += blockDim.x, ++slot) {
        int n, m;
        nm_of(i, n, m);
        acc[slot] = cfma(make_double2(0.0, H.k), grad_dot_tab(H.k, R, PF, n, -m, mu), acc[slot]);
      }
    }
  }
  int slot = 0;
  for (int i = threadIdx.x; i < H.KP; i += blockDim.x, ++slot) H.M[size_t(b) * H.KP + i] = acc[slot];
}

template <int NB>
__global__ void __launch_bounds__(512) k_h_shift_b(HelmData H, int mode, const int2* __restrict__ pairs, int n,
                                                   const double2* __restrict__ T) {
  extern __shared__ double2 smb[];  // NB x KP
  const int KP = H.KP, i = threadIdx.x, p0 = blockIdx.x * NB;
  const int np = min(NB, n - p0);
  double2* Xs = mode == 0 ? H.M : H.L;
  for (int e = threadIdx.x; e < NB * KP; e += blockDim.x) {
    const int j = e / KP, q = e - j * KP;
    smb[e] = j < np ? Xs[size_t(pairs[p0 + j].x) * KP + q] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (i >= KP) return;
  double2 acc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j] = make_double2(0.0, 0.0);
  for (int k2 = 0; k2 < KP; ++k2) {
    const double2 a = __ldg(T + size_t(k2) * KP + i);
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = cfma(a, smb[j * KP + k2], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < NB; ++j)
    if (j < np) {
      double2* d = Xs + size_t(pairs[p0 + j].y) * KP + i;
      const double2 v = *d;
      *d = make_double2(v.x + acc[j].x, v.y + acc[j].y);
    }
}

// operator builder, one CTA per operator: T[k][i] = 4 pi sum_l i^{n'+l-n} G F_l^{m-m'}(t)
__global__ void __launch_bounds__(256) k_h_build_ops(HelmData H, const double4* __restrict__ shifts,
                                                     double2* __restrict__ ops) {
  extern __shared__ double2 sm[];
  const int P = H.P, KP = H.KP, L = 2 * P;
  double2* F = sm;
  double2* rad = sm + (L + 1) * (L + 1);
  const double4 t = shifts[blockIdx.x];  // (tx, ty, tz, singular)
  wave_table_cta(H.k, L, t.x, t.y, t.z, t.w != 0.0, F, rad);
  double2* T = ops + size_t(blockIdx.x) * KP * KP;
  for (int e = threadIdx.x; e < KP * KP; e += blockDim.x) {
    const int kin = e / KP, iout = e % KP;
    int n, m, n2, m2;
    nm_of(kin, n, m);
    nm_of(iout, n2, m2);
    const double* g = H.gaunt + (size_t(kin) * KP + iout) * H.GL;
    double2 acc = make_double2(0, 0);
    const int l0 = abs(n - n2);
    for (int li = 0; li < H.GL; ++li) {
      const int l = l0 + 2 * li;
      if (l > n + n2) break;
      const double gv = g[li];
      if (gv == 0.0 || abs(m - m2) > l) continue;
      const double2 f = cmul(ipow(n2 + l - n), F[fi(l, m - m2)]);
      acc.x += gv * f.x;
      acc.y += gv * f.y;
    }
    T[e] = make_double2(4.0 * kPi * acc.x, 4.0 * kPi * acc.y);
  }
}

// ---- Stage 4 M2L, split form -------------------------------------------------
// Rotating the frame about z by alpha = atan2(dy, dx) puts the offset in the
// xz-plane (t'); there Y_l^mu(t') is real and F_l^{-mu} = F_l^mu, and with the
// sign symmetry of the Gaunt coefficients T(-m', -m) = T(m', m).  In the even / odd
// coordinates a_m = x_m + x_{-m}, b_m = x_m - x_{-m} (m > 0), a_0 = x_0 the operator
// is block diagonal:
//   A_{m'} = sum_{m>0} [T(m',m) + T(m',-m)] a_m + c T(m',0) a_0  (c = 2 for m' > 0, 1 for m' = 0,
//            and the m > 0 terms are halved for m' = 0)
//   B_{m'} = sum_{m>0} [T(m',m) - T(m',-m)] b_m
// (sizes (p+1)(p+2)/2 and p(p+1)/2: half the complex MACs of the full operator).
// Columns enter as M' = M e^{i m alpha}; the reduce rebuilds y_{+-m'} = (A +- B)/2
// and rotates back, L = y e^{-i m alpha}.
__device__ __forceinline__ int ev_idx(int n, int m) { return n * (n + 1) / 2 + m; }      // m >= 0
__device__ __forceinline__ int od_idx(int n, int m) { return n * (n - 1) / 2 + m - 1; }  // m >= 1
__device__ __forceinline__ void ev_nm(int e, int& n, int& m) {
  n = int((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while ((n + 1) * (n + 2) / 2 <= e) ++n;
  while (n * (n + 1) / 2 > e) --n;
  m = e - n * (n + 1) / 2;
}
__device__ __forceinline__ void od_nm(int o, int& n, int& m) {
  n = int((1.0 + sqrt(8.0 * o + 1.0)) * 0.5);
  while (n * (n - 1) / 2 > o) --n;
  while ((n + 1) * n / 2 <= o) ++n;
  m = o - n * (n - 1) / 2 + 1;
}

// one operator entry T(n',m' <- n,m) of the rotated-frame operator from the F table
__device__ __forceinline__ double2 t_entry(const HelmData& H, const double2* F, int n2, int m2, int n, int m) {
  const double* g = H.gaunt + (size_t(fi(n, m)) * H.KP + fi(n2, m2)) * H.GL;
  double2 acc = make_double2(0, 0);
  const int l0 = abs(n - n2);
  for (int li = 0; li < H.GL; ++li) {
    const int l = l0 + 2 * li;
    if (l > n + n2) break;
    const double gv = g[li];
    if (gv == 0.0 || abs(m - m2) > l) continue;
    const double2 f = cmul(ipow(n2 + l - n), F[fi(l, m - m2)]);
    acc.x += gv * f.x;
    acc.y += gv * f.y;
  }
  return make_double2(4.0 * kPi * acc.x, 4.0 * kPi * acc.y);
}

// point-and-shoot tiles: up to kHColsS same-operator List-2 entries (k_h_m2l_pas)
constexpr int kHColsS = 16;
__global__ void __launch_bounds__(512) k_h_m2l_reduce_split(HelmData H, const int* __restrict__ boxes, int64_t base,
                                                            const double2* __restrict__ temp,
                                                            const int* __restrict__ ent_op,
                                                            const double2* __restrict__ cs) {
  const int b = boxes[blockIdx.x];
  const int P = H.P, KP = H.KP, NE = (P + 1) * (P + 2) / 2;
  const int i = threadIdx.x;
  if (i >= KP) return;
  int n, m;
  nm_of(i, n, m);
  const int am = abs(m);
  const int ie = ev_idx(n, am), io = am > 0 ? NE + od_idx(n, am) : -1;
  double2 s = make_double2(0, 0);
  for (int64_t pos = H.v_starts[b]; pos < H.v_starts[b + 1]; ++pos) {
    const double2* row = temp + size_t(pos - base) * KP;
    double2 y = row[ie];
    if (am > 0) {
      const double2 bv = row[io];
      y = m > 0 ? make_double2(0.5 * (y.x + bv.x), 0.5 * (y.y + bv.y))
                : make_double2(0.5 * (y.x - bv.x), 0.5 * (y.y - bv.y));
    }
    double2 r = cs[size_t(ent_op[pos]) * (P + 1) + am];  // e^{i |m| alpha}
    if (m >= 0) r.y = -r.y;                            // L = y e^{-i m alpha}
    const double2 v = cmul(y, r);
    s.x += v.x;
    s.y += v.y;
  }
  const double2 v = H.L[size_t(b) * KP + i];
  H.L[size_t(b) * KP + i] = make_double2(v.x + s.x, v.y + s.y);
}

// Stages 3, 5a, 6a: P2QBXL, thread per (centre, source slice):
//   Lc_n^m += ik w h_n(k r) conj(Y_n^m) = [ik w h_n(k r) / r^n] conj(S_n^m)   (S^{-m} = conj S^m)
template <int Q>
__global__ void __launch_bounds__(128) k_h_near(HelmData H, const int* __restrict__ boxes) {
  constexpr int KQ = (Q + 1) * (Q + 1);
  constexpr int KH = (Q + 1) * (Q + 2) / 2;
  extern __shared__ double2 red[];  // KQ x 128
  const int b = boxes[blockIdx.x];
  const int nctr = H.ctr_own_count[b], c0 = H.ctr_own_start[b];
  const int64_t sb = H.near_starts[b], se = H.near_starts[b + 1];
  const double k = H.k;
  for (int cc = 0; cc < nctr; cc += 128) {
    const int ncc = min(128, nctr - cc);
    const int S = 128 / ncc;
    const int ci = threadIdx.x / S, sl = threadIdx.x % S;
    const bool active = ci < ncc;
    double4 c = make_double4(0, 0, 0, 1);
    if (active) c = H.ctr[c0 + cc + ci];
    double2 acc[KQ];
#pragma unroll
    for (int i = 0; i < KQ; ++i) acc[i] = make_double2(0, 0);
    if (active) {
      int f = sl;
      for (int64_t sg = sb; sg < se; ++sg) {
        const int2 seg = H.near_seg[sg];
        for (; f < seg.y; f += S) {
          const int s = seg.x + f;
          const double4 x = H.src[s];
          const double2 w = H.hw[s];
          const double vx = x.x - c.x, vy = x.y - c.y, vz = x.z - c.z;
          const double r2 = vx * vx + vy * vy + vz * vz;
          const double ir = rsqrt(r2), r = r2 * ir;  // one rsqrt instead of sqrt + divide
          double2 Sh[KH];  // S_n^m, m >= 0, index n(n+1)/2 + m
#pragma unroll
          for (int m = 0; m <= Q; ++m) {
            const int dm = m * (m + 1) / 2 + m;
            if (m == 0) {
              Sh[0] = make_double2(0.28209479177387814347, 0.0);  // 1/sqrt(4 pi)
            } else {
              const double2 d = Sh[(m - 1) * m / 2 + m - 1];
              Sh[dm] = make_double2(c_sa[m] * (d.x * vx - d.y * vy), c_sa[m] * (d.x * vy + d.y * vx));
            }
            if (m + 1 <= Q) {
              const double f1 = c_sb[m] * vz;
              Sh[(m + 1) * (m + 2) / 2 + m] = make_double2(f1 * Sh[dm].x, f1 * Sh[dm].y);
            }
#pragma unroll
            for (int n = m + 2; n <= Q; ++n) {
              const double cn = c_sc[n * (kHSolid + 1) + m], dn = c_sd[n * (kHSolid + 1) + m] * r2;
              const double2 a1 = Sh[(n - 1) * n / 2 + m], a2 = Sh[(n - 2) * (n - 1) / 2 + m];
              Sh[n * (n + 1) / 2 + m] = make_double2(cn * (vz * a1.x - dn * a2.x), cn * (vz * a1.y - dn * a2.y));
            }
          }
          double2 g[Q + 1];
          radial_over_rn<Q>(k, r, ir, g);
          const double2 f0 = make_double2(-k * w.y, k * w.x);  // ik w
          // L_n^m += fh conj(S_n^m), L_n^-m += fh S_n^m with fh = c + i d, S = a + i b:
          // the two share the four real products, so accumulate (sum c a, sum d b) in slot
          // (n, m) and (sum d a, sum c b) in slot (n, -m) -- 4 FMAs instead of 8 -- and form
          // the coefficients after the slice reduction.  S_n^0 is real: L_n^0 += fh a.
#pragma unroll
          for (int n = 0; n <= Q; ++n) {
            const double2 fh = cmul(f0, g[n]);
#pragma unroll
            for (int m = 0; m <= n; ++m) {
              const double2 sv = Sh[n * (n + 1) / 2 + m];
              if (m == 0) {
                acc[fi(n, 0)].x = fma(fh.x, sv.x, acc[fi(n, 0)].x);
                acc[fi(n, 0)].y = fma(fh.y, sv.x, acc[fi(n, 0)].y);
              } else {
                acc[fi(n, m)].x = fma(fh.x, sv.x, acc[fi(n, m)].x);    // c a
                acc[fi(n, m)].y = fma(fh.y, sv.y, acc[fi(n, m)].y);    // d b
                acc[fi(n, -m)].x = fma(fh.y, sv.x, acc[fi(n, -m)].x);  // d a
                acc[fi(n, -m)].y = fma(fh.x, sv.y, acc[fi(n, -m)].y);  // c b
              }
            }
          }
        }
        f -= seg.y;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KQ; ++i) red[i * 128 + threadIdx.x] = acc[i];
    __syncthreads();
    if (active && sl == 0) {
      double2* out = H.Lc + size_t(c0 + cc + ci) * KQ;
      for (int n = 0; n <= Q; ++n)
        for (int m = 0; m <= n; ++m) {
          double2 sp = make_double2(0, 0), sm2 = make_double2(0, 0);
          for (int k2 = 0; k2 < S; ++k2) {
            const double2 vp = red[fi(n, m) * 128 + threadIdx.x + k2];
            sp.x += vp.x;
            sp.y += vp.y;
            if (m > 0) {
              const double2 vm = red[fi(n, -m) * 128 + threadIdx.x + k2];
              sm2.x += vm.x;
              sm2.y += vm.y;
            }
          }
          if (m == 0) {
            out[fi(n, 0)] = sp;
          } else {  // (ca + db, da - cb) and (ca - db, da + cb)
            out[fi(n, m)] = make_double2(sp.x + sp.y, sm2.x - sm2.y);
            out[fi(n, -m)] = make_double2(sp.x - sp.y, sm2.x + sm2.y);
          }
        }
    }
    __syncthreads();
  }
}

// Double-layer part of P2QBXL (a second pass after k_h_near, same slices and fixed
// slice-order reduction): Lc_n^m += ik mu . grad_s [h_n conj(Y_n^m)](s - c).
template <int Q>
__global__ void __launch_bounds__(128) k_h_near_dip(HelmData H, const int* __restrict__ boxes) {
  constexpr int KQ = (Q + 1) * (Q + 1);
  extern __shared__ double2 red[];  // KQ x 128
  const int b = boxes[blockIdx.x];
  const int nctr = H.ctr_own_count[b], c0 = H.ctr_own_start[b];
  const int64_t sb = H.near_starts[b], se = H.near_starts[b + 1];
  for (int cc = 0; cc < nctr; cc += 128) {
    const int ncc = min(128, nctr - cc);
    const int S = 128 / ncc;
    const int ci = threadIdx.x / S, sl = threadIdx.x % S;
    const bool active = ci < ncc;
    double4 c = make_double4(0, 0, 0, 1);
    if (active) c = H.ctr[c0 + cc + ci];
    double2 acc[KQ];
#pragma unroll
    for (int i = 0; i < KQ; ++i) acc[i] = make_double2(0, 0);
    if (active) {
      int f = sl;
      for (int64_t sg = sb; sg < se; ++sg) {
        const int2 seg = H.near_seg[sg];
        for (; f < seg.y; f += S) {
          const int s = seg.x + f;
          const double4 x = H.src[s];
          const double2 mu[3] = {H.hmu[3 * size_t(s)], H.hmu[3 * size_t(s) + 1], H.hmu[3 * size_t(s) + 2]};
          dipole_terms<Q, true>(H.k, x.x - c.x, x.y - c.y, x.z - c.z, mu, make_double2(0.0, H.k), acc);
        }
        f -= seg.y;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KQ; ++i) red[i * 128 + threadIdx.x] = acc[i];
    __syncthreads();
    if (active && sl == 0) {
      double2* out = H.Lc + size_t(c0 + cc + ci) * KQ;
      for (int i = 0; i < KQ; ++i) {
        double2 sp = out[i];
        for (int k2 = 0; k2 < S; ++k2) {
          sp.x += red[i * 128 + threadIdx.x + k2].x;
          sp.y += red[i * 128 + threadIdx.x + k2].y;
        }
        out[i] = sp;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) k_h_p2p(HelmData H, const int* __restrict__ boxes) {
  const int b = boxes[blockIdx.x];
  const int ntg = H.tgt_own_count[b], t0 = H.tgt_own_start[b];
  for (int ti = threadIdx.x; ti < ntg; ti += blockDim.x) {
    const double4 t = H.tgt[t0 + ti];
    double2 acc = make_double2(0, 0);
    for (int64_t sg = H.near_starts[b]; sg < H.near_starts[b + 1]; ++sg) {
      const int2 seg = H.near_seg[sg];
      for (int j = 0; j < seg.y; ++j) {
        const double4 x = H.src[seg.x + j];
        const double dx = t.x - x.x, dy = t.y - x.y, dz = t.z - x.z;
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        double s, co;
        sincos(H.k * r, &s, &co);
        acc = cfma(H.hw[seg.x + j], make_double2(co / (4.0 * kPi * r), s / (4.0 * kPi * r)), acc);
        if (H.hmu) {
          const double2 mu[3] = {H.hmu[3 * size_t(seg.x + j)], H.hmu[3 * size_t(seg.x + j) + 1],
                                 H.hmu[3 * size_t(seg.x + j) + 2]};
          const double2 v = dipole_kernel(H.k, dx, dy, dz, r, mu);
          acc.x += v.x;
          acc.y += v.y;
        }
      }
    }
    H.phi[t0 + ti] = acc;
  }
}

// Stage 6b P2L over List 4 far: L_b += ik w h_n conj(Y) = ik w (h_n Y)_n^{-m}
__global__ void __launch_bounds__(256) k_h_p2l(HelmData H, const int* __restrict__ boxes) {
  extern __shared__ double2 sm[];
  double2* T = sm;
  double2* rad = sm + H.KP;
  const int b = boxes[blockIdx.x];
  const double4 bc = H.box[b];
  const int PF = H.hmu ? H.P + 1 : H.P;  // the double layer needs one more degree
  rad = sm + (PF + 1) * (PF + 1);
  double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
  for (int64_t sg = H.xfar_starts[b]; sg < H.xfar_starts[b + 1]; ++sg) {
    const int2 seg = H.xfar_seg[sg];
    for (int j = 0; j < seg.y; ++j) {
      const double4 x = H.src[seg.x + j];
      const double2 w = H.hw[seg.x + j];
      __syncthreads();
      wave_table_cta(H.k, PF, x.x - bc.x, x.y - bc.y, x.z - bc.z, true, T, rad);
      const double2 f = make_double2(-H.k * w.y, H.k * w.x);
      int slot = 0;
      for (int i = threadIdx.x; i < H.KP; i += blockDim.x, ++slot) {
        int n, m;
        nm_of(i, n, m);
        acc[slot] = cfma(f, T[fi(n, -m)], acc[slot]);
        if (H.hmu) {
          const double2 mu[3] = {H.hmu[3 * size_t(seg.x + j)], H.hmu[3 * size_t(seg.x + j) + 1],
                                 H.hmu[3 * size_t(seg.x + j) + 2]};
          acc[slot] = cfma(make_double2(0.0, H.k), grad_dot_tab(H.k, T, PF, n, -m, mu), acc[slot]);
        }
      }
    }
  }
  int slot = 0;
  for (int i = threadIdx.x; i < H.KP; i += blockDim.x, ++slot) {
    const double2 v = H.L[size_t(b) * H.KP + i];
    H.L[size_t(b) * H.KP + i] = make_double2(v.x + acc[slot].x, v.y + acc[slot].y);
  }
}

// P2M (own sources of a leaf, regular j_n) and P2L (List 4 far, singular h_n), one
// source per warp: lane 0 forms the radial table, lanes 0..P the
// solid-harmonic columns m >= 0 (Cartesian recurrences), then every lane adds its
// ceil(KP/32) coefficients f h_n conj(Y_n^m) -- the negative orders read the m >= 0
// column (Y^{-m} = conj(Y^m)).  8 sources in flight per CTA instead of one CTA-wide
// table per source; the warps' partial sums are added in warp order (deterministic).
constexpr int kHP2LSlots = 14;  // ceil(441 / 32): P <= 20
constexpr int kHP2LBatch = 16;  // sources per warp whose radial tables are formed together, one per lane
template <bool P2M>
__global__ void __launch_bounds__(256, 2) k_h_p2w(HelmData H, const int* __restrict__ boxes) {
  extern __shared__ double2 smw[];
  const int P = H.P, KP = H.KP, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NW = blockDim.x >> 5;
  double2* T = smw + warp * (KP + kHP2LBatch * (P + 1));
  double2* rad = T + KP;  // kHP2LBatch radial tables
  const int b = boxes[blockIdx.x];
  const double4 bc = H.box[b];
  double2 acc[kHP2LSlots];
  int code[kHP2LSlots];  // fi(n, |m|) | n << 16 | (m < 0) << 30
#pragma unroll
  for (int sl = 0; sl < kHP2LSlots; ++sl) {
    acc[sl] = make_double2(0.0, 0.0);
    const int i = lane + 32 * sl;
    code[sl] = -1;
    if (i < KP) {
      int n, m;
      nm_of(i, n, m);
      code[sl] = fi(n, m < 0 ? -m : m) | n << 16 | (m < 0 ? 1 << 30 : 0);
    }
  }
  // sources: P2M the leaf's own (one segment), P2L its List-4-far segments; warp w takes
  // flat sources w, w + NW, ...
  int64_t sb, se;
  if (P2M) {
    sb = 0;
    se = H.src_own_count[b] > 0 ? 1 : 0;
  } else {
    sb = H.xfar_starts[b];
    se = H.xfar_starts[b + 1];
  }
  auto seg_at = [&](int64_t kk) {
    return P2M ? make_int2(H.src_own_start[b], H.src_own_count[b]) : H.xfar_seg[kk];
  };
  int64_t k = sb;
  int off = warp, st = 0, cnt = 0;
  if (k < se) {
    st = seg_at(k).x;
    cnt = seg_at(k).y;
  }
  while (k < se && off >= cnt) {
    off -= cnt;
    if (++k < se) {
      st = seg_at(k).x;
      cnt = seg_at(k).y;
    }
  }
  while (k < se) {
    // The radial tables of the warp's next kHP2LBatch sources, one source per lane (the
    // recurrences are serial in n: one lane per table used to idle the other 31).  Lane
    // j < kHP2LBatch walks the segment cursor j sources ahead.
    int64_t kj = k;
    int offj = off + lane * NW, stj = st, cntj = cnt;
    if (lane < kHP2LBatch) {
      while (kj < se && offj >= cntj) {
        offj -= cntj;
        if (++kj < se) {
          stj = seg_at(kj).x;
          cntj = seg_at(kj).y;
        }
      }
    }
    const bool valid = lane < kHP2LBatch && kj < se;
    const int srcj = valid ? stj + offj : -1;
    if (valid) {
      const double4 xj = H.src[srcj];
      const double ax = xj.x - bc.x, ay = xj.y - bc.y, az = xj.z - bc.z;
      radial_table(H.k, sqrt(ax * ax + ay * ay + az * az), P, !P2M, rad + lane * (P + 1));
    }
    const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));  // lanes 0 .. nvalid - 1
    __syncwarp();
    for (int j = 0; j < nvalid; ++j) {
      const int src = __shfl_sync(0xffffffffu, srcj, j);
      const double4 x = H.src[src];
      const double2 w = H.hw[src];
      const double tx = x.x - bc.x, ty = x.y - bc.y, tz = x.z - bc.z, r2 = tx * tx + ty * ty + tz * tz;
      const double2* rj = rad + j * (P + 1);
      if (lane <= P) {  // column m = lane of S_n^m(t), n = m..P
        const int m = lane;
        // diagonal S_m^m = g_sap[m] (tx + i ty)^m by repeated squaring (5 lock-step
        // rounds instead of up to P dependent products)
        double2 pw = make_double2(1.0, 0.0), qz = make_double2(tx, ty);
#pragma unroll
        for (int bit = 0; bit < 5; ++bit) {
          if ((m >> bit) & 1) pw = cmul(pw, qz);
          qz = cmul(qz, qz);
        }
        const double2 d = make_double2(g_sap[m] * pw.x, g_sap[m] * pw.y);
        T[fi(m, m)] = d;
        if (m + 1 <= P) {
          double2 a = d, bb = make_double2(g_sb[m] * tz * d.x, g_sb[m] * tz * d.y);
          T[fi(m + 1, m)] = bb;
          for (int n = m + 2; n <= P; ++n) {
            const double cn = g_sc[n * (kHSolid + 1) + m], dn = g_sd[n * (kHSolid + 1) + m] * r2;
            const double2 c2 = make_double2(cn * (tz * bb.x - dn * a.x), cn * (tz * bb.y - dn * a.y));
            T[fi(n, m)] = c2;
            a = bb;
            bb = c2;
          }
        }
      }
      __syncwarp();
      const double2 f = make_double2(-H.k * w.y, H.k * w.x);  // i k w
#pragma unroll
      for (int sl = 0; sl < kHP2LSlots; ++sl) {
        if (code[sl] < 0) continue;
        double2 v = T[code[sl] & 0xffff];
        if (!(code[sl] >> 30)) v.y = -v.y;  // m >= 0: conj(S_n^m)
        const double2 fr = cmul(f, rj[(code[sl] >> 16) & 0x3fff]);
        acc[sl] = cfma(fr, v, acc[sl]);
      }
      __syncwarp();
    }
    // the warp's cursor moves past the batch: the last valid lane's position, one step on
    k = __shfl_sync(0xffffffffu, kj, nvalid - 1);
    off = __shfl_sync(0xffffffffu, offj, nvalid - 1) + NW;
    st = __shfl_sync(0xffffffffu, stj, nvalid - 1);
    cnt = __shfl_sync(0xffffffffu, cntj, nvalid - 1);
    while (k < se && off >= cnt) {
      off -= cnt;
      if (++k < se) {
        st = seg_at(k).x;
        cnt = seg_at(k).y;
      }
    }
  }
  __syncthreads();
  double2* red = smw;  // NW x KP
#pragma unroll
  for (int sl = 0; sl < kHP2LSlots; ++sl)
    if (code[sl] >= 0) red[warp * KP + lane + 32 * sl] = acc[sl];
  __syncthreads();
  for (int i = threadIdx.x; i < KP; i += blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int ww = 0; ww < NW; ++ww) {
      sx += red[ww * KP + i].x;
      sy += red[ww * KP + i].y;
    }
    double2* out = (P2M ? H.M : H.L) + size_t(b) * KP + i;
    const double2 v = *out;
    *out = make_double2(v.x + sx, v.y + sy);
  }
}

// Stage 5b M2QBXL / Stage 8 L2QBXL: box expansion X (order p) -> up to kHCtrMax
// centres (order q).  For mu = -(p+q)..p+q: C_mu[i'][l] from X and the Gaunt
// table, F_l^mu(c_j - c_box) per centre, acc[j][i'] += sum_l F C.
constexpr int kHCtrAcc = 12;  // per-thread outputs: 2 rows i' x up to 6 centres (q <= 8, 256 threads)
// Gaunt coefficients of the centre translations, term-major (HelmData::gaunt_ctr):
// entry (|mu|, sign, l, k, i') = G(n, m' + mu; n', m'; l) with n = n_lo + 2k, the k-th
// term of C_mu[i'][l] (zero beyond the last term)
__global__ void k_h_gaunt_ctr(HelmData H, double* __restrict__ out, size_t total) {
  const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int P = H.P, Q = H.Q, KQ = H.KQ, NL = P + Q + 1, KT = Q + 1;
  const int iout = int(idx % KQ);
  size_t r = idx / KQ;
  const int k = int(r % KT);
  r /= KT;
  const int l = int(r % NL);
  r /= NL;
  const int sg = int(r & 1), amu = int(r >> 1);
  double v = 0.0;
  if (l >= amu && !(amu == 0 && sg)) {
    int n2, m2;
    nm_of(iout, n2, m2);
    const int m = m2 + (sg ? -amu : amu);
    int nlo = max(abs(m), abs(l - n2));
    nlo += (nlo + n2 + l) & 1;
    const int nhi = min(P, l + n2), n = nlo + 2 * k;
    if (n <= nhi) v = H.gaunt[(size_t(fi(n, m)) * H.KP + iout) * H.GL + ((l - abs(n - n2)) >> 1)];
  }
  out[idx] = v;
}

// acc[2a + h] += sum_{sign} sum_l F[a][l] C[h][l] for CPG centres and two C rows: 2 + CPG
// shared loads per 2 CPG complex multiply-adds.  Centres beyond nj repeat the last
// valid one (their sums are never stored), so the loop has no predicates.
template <int CPG>
__device__ __forceinline__ void ctr_dot(double2 (&acc)[12], const double2* __restrict__ F0,
                                        const double2* __restrict__ C0, int c1_off, int c_sign_stride, int NL, int nj,
                                        int ns, int amu, int L) {
  int fo[CPG];
#pragma unroll
  for (int a = 0; a < CPG; ++a) fo[a] = min(a, nj - 1) * NL;
  for (int sg = 0; sg < ns; ++sg) {
    const double2* F = F0 + sg * kHCtrMax * NL;
    const double2* C = C0 + sg * c_sign_stride;
    for (int l = amu; l <= L; ++l) {
      const double2 c0 = C[l], c1 = C[c1_off + l];
#pragma unroll
      for (int a = 0; a < CPG; ++a) {
        const double2 f = F[fo[a] + l];
        acc[2 * a] = cfma(f, c0, acc[2 * a]);
        acc[2 * a + 1] = cfma(f, c1, acc[2 * a + 1]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_h_ctr(HelmData H, int singular, const double2* __restrict__ X,
                                               const int4* __restrict__ ctas, const int* __restrict__ ctr_of,
                                               const int* __restrict__ out_row, double2* __restrict__ out,
                                               int accumulate) {
  extern __shared__ double2 sm[];
  const int P = H.P, Q = H.Q, KP = H.KP, KQ = H.KQ, L = P + Q, NL = L + 1;
  const int NLp = NL | 1;  // odd row stride of C: lanes reading consecutive rows hit different banks
  const int4 cta = ctas[blockIdx.x];  // (box, first item, count, -)
  const int nctr = cta.z;
  double2* Xs = sm;                      // KP
  double2* Cm = Xs + KP;                 // 2 x KQ x NLp: C_{+|mu|}, C_{-|mu|}
  double2* rad = Cm + 2 * KQ * NLp;      // kHCtrMax x NL
  double2* Fc = rad + kHCtrMax * NL;     // 2 x kHCtrMax x NL: F^{+|mu|}, F^{-|mu|}
  double* geo = reinterpret_cast<double*>(Fc + 2 * kHCtrMax * NL);  // kHCtrMax x 4: t, |t|^2
  const double4 bc = H.box[cta.x];
  for (int j = threadIdx.x; j < KP; j += blockDim.x) Xs[j] = X[size_t(cta.x) * KP + j];
  for (int j = threadIdx.x; j < nctr; j += blockDim.x) {  // per centre: t, and rad_l / r^l
    const double4 c = H.ctr[ctr_of[cta.y + j]];
    const double tx = c.x - bc.x, ty = c.y - bc.y, tz = c.z - bc.z;
    geo[4 * j] = tx;
    geo[4 * j + 1] = ty;
    geo[4 * j + 2] = tz;
    geo[4 * j + 3] = tx * tx + ty * ty + tz * tz;
    radial_table(H.k, sqrt(geo[4 * j + 3]), L, singular != 0, rad + j * NL);
  }
  double2 acc[kHCtrAcc];
#pragma unroll
  for (int a = 0; a < kHCtrAcc; ++a) acc[a] = make_double2(0, 0);
  // output tiling: KQ2 row pairs (i0, i0 + KQ2) x ngrp centre groups of cpg centres
  const int KQ2 = (KQ + 1) / 2, ngrp = min(int(blockDim.x) / KQ2, kHCtrMax);
  const int cpg = (nctr + ngrp - 1) / ngrp;  // centres per group of this CTA; <= kHCtrAcc / 2 for q <= 8
  const int grp = threadIdx.x / KQ2, i0 = threadIdx.x - grp * KQ2, j0 = grp * cpg;
  const bool has1 = i0 + KQ2 < KQ;
  // C_mu contraction: thread = (row i', residue class of l) among the first 7 warps
  const int c_ng = max(1, (int(blockDim.x) - 32) / KQ), c_iout = threadIdx.x % KQ, c_lg = threadIdx.x / KQ;
  const bool c_act = int(threadIdx.x) < c_ng * KQ && int(threadIdx.x) < int(blockDim.x) - 32;
  int c_n2, c_m2;
  nm_of(c_iout, c_n2, c_m2);
  const int nj = max(0, min(cpg, nctr - j0));
  __syncthreads();
  // mu and -mu together: one solid-harmonic column per |mu| serves both signs
  // (S^{-mu} = conj S^mu), and half as many barriers
  for (int amu = 0; amu <= L; ++amu) {
    const int ns = amu == 0 ? 1 : 2;  // sign index 0: mu = +|mu|, 1: mu = -|mu|
    // C_mu[i'][l] = 4 pi sum_n i^{n'+l-n} G(n, m'+mu; n', m'; l) X_n^{m'+mu} over the used
    // terms only: l >= |mu| and n + n' + l even
    // the last warp forms the centres' F columns (a recurrence in l per centre) while the
    // other warps contract C_mu, so the column recurrence is off the critical path
    // (thread = row i' x one of c_ng residue classes of l: no index divisions in the loop;
    // the terms of one sum differ by a factor -1 from one n to the next, n stepping by 2, so
    // the power of i is applied once to the signed sum -- exact, same rounding as term by term)
    if (c_act)
      for (int sg = 0; sg < ns; ++sg) {
        const int mu = sg ? -amu : amu, m = c_m2 + mu;
        // term range and table row of one l
        auto range = [&](int l, int& nlo, int& nhi, const double*& gt) {
          nlo = max(abs(m), abs(l - c_n2));
          nlo += (nlo + c_n2 + l) & 1;
          nhi = l <= L ? min(P, l + c_n2) : -1;
          gt = H.gaunt_ctr + (size_t((amu * 2 + sg) * NL + min(l, L)) * (Q + 1)) * KQ + c_iout;
        };
        auto first4 = [&](int nlo, int nhi, const double* gt, double (&g)[4]) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // term-major table: the warp's rows i' read one 8-byte run
            g[u] = 0.0;
            if (nlo + 2 * u <= nhi) g[u] = __ldg(gt + u * KQ);
          }
        };
        auto finish = [&](int l, int nlo, int nhi, const double* gt, const double (&g0)[4]) {
          double sx = 0.0, sy = 0.0;
          for (int n = nlo; n <= nhi; n += 8) {
            double g[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int nn = n + 2 * u;
              g[u] = g0[u];
              if (n > nlo) g[u] = nn <= nhi ? __ldg(gt + ((nn - nlo) >> 1) * KQ) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int nn = n + 2 * u;
              if (nn <= nhi) {
                const double2 x = Xs[fi(nn, m)];
                const double gu = (u & 1) ? -g[u] : g[u];
                sx = fma(gu, x.x, sx);
                sy = fma(gu, x.y, sy);
              }
            }
          }
          const double2 t = nlo <= nhi ? cmul(ipow(c_n2 + l - nlo), make_double2(sx, sy)) : make_double2(0.0, 0.0);
          Cm[(sg * KQ + c_iout) * NLp + l] = make_double2(4.0 * kPi * t.x, 4.0 * kPi * t.y);
        };
        // two l at a time: the Gaunt loads of both are in flight before either sum starts
        for (int l = amu + c_lg; l <= L; l += 2 * c_ng) {
          int nloA, nhiA, nloB, nhiB;
          const double *gtA, *gtB;
          range(l, nloA, nhiA, gtA);
          range(l + c_ng, nloB, nhiB, gtB);
          double gA[4], gB[4];
          first4(nloA, nhiA, gtA, gA);
          first4(nloB, nhiB, gtB, gB);
          finish(l, nloA, nhiA, gtA, gA);
          if (l + c_ng <= L) finish(l + c_ng, nloB, nhiB, gtB, gB);
        }
      }
    const int nth_c = blockDim.x - 32;
    // F columns per centre: (rad_l / r^l) S_l^{+-|mu|}(t), l = |mu|..L
    for (int j = int(threadIdx.x) - nth_c; j >= 0 && j < nctr; j += 32) {
      double2* colp = Fc + j * NL;
      double2* colm = Fc + (kHCtrMax + j) * NL;
      solid_column(amu, L, geo[4 * j], geo[4 * j + 1], geo[4 * j + 2], geo[4 * j + 3], colp);
      for (int l = amu; l <= L; ++l) {
        const double2 sv = colp[l], rl = rad[j * NL + l];
        colp[l] = cmul(rl, sv);
        colm[l] = cmul(rl, make_double2(sv.x, -sv.y));
      }
    }
    __syncthreads();
    // acc[j][i'] += sum_l F[j][l] C[i'][l], register-tiled: a thread owns rows i0 and
    // i0 + KQ2 of C and cpg centres, so one l step costs 2 + cpg shared loads for 2 cpg
    // complex multiply-adds (a centre's sum runs in the same order as before)
    if (nj > 0) {
      switch (cpg) {
        case 1: ctr_dot<1>(acc, Fc + j0 * NL, Cm + i0 * NLp, has1 ? KQ2 * NLp : 0, KQ * NLp, NL, nj, ns, amu, L); break;
        case 2: ctr_dot<2>(acc, Fc + j0 * NL, Cm + i0 * NLp, has1 ? KQ2 * NLp : 0, KQ * NLp, NL, nj, ns, amu, L); break;
        case 3: ctr_dot<3>(acc, Fc + j0 * NL, Cm + i0 * NLp, has1 ? KQ2 * NLp : 0, KQ * NLp, NL, nj, ns, amu, L); break;
        case 4: ctr_dot<4>(acc, Fc + j0 * NL, Cm + i0 * NLp, has1 ? KQ2 * NLp : 0, KQ * NLp, NL, nj, ns, amu, L); break;
        case 5: ctr_dot<5>(acc, Fc + j0 * NL, Cm + i0 * NLp, has1 ? KQ2 * NLp : 0, KQ * NLp, NL, nj, ns, amu, L); break;
        default: ctr_dot<6>(acc, Fc + j0 * NL, Cm + i0 * NLp, has1 ? KQ2 * NLp : 0, KQ * NLp, NL, nj, ns, amu, L); break;
      }
    }
    __syncthreads();
  }
  if (nj > 0) {
#pragma unroll
    for (int a = 0; a < kHCtrAcc / 2; ++a)
      if (a < nj) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !has1) continue;
          double2* o = out + size_t(out_row[cta.y + j0 + a]) * KQ + i0 + h * KQ2;
          if (accumulate) {
            const double2 v = *o;
            *o = make_double2(v.x + acc[2 * a + h].x, v.y + acc[2 * a + h].y);
          } else {
            *o = acc[2 * a + h];
          }
        }
      }
  }
}

__global__ void k_h_pair_reduce(HelmData H, const int* __restrict__ centres, const int* __restrict__ starts, int n,
                                const double2* __restrict__ rows) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= int64_t(n) * H.KQ) return;
  const int i = int(t / H.KQ), j = int(t % H.KQ);
  double2 a = H.Lc[size_t(centres[i]) * H.KQ + j];
  for (int p2 = starts[i]; p2 < starts[i + 1]; ++p2) {
    const double2 v = rows[size_t(p2) * H.KQ + j];
    a.x += v.x;
    a.y += v.y;
  }
  H.Lc[size_t(centres[i]) * H.KQ + j] = a;
}

// M2P at conventional targets of boxes with List 3 far entries
__global__ void __launch_bounds__(128) k_h_m2p(HelmData H, const int* __restrict__ boxes) {
  extern __shared__ double2 sm[];
  double2* S = sm;
  double2* rad = sm + H.KP;
  __shared__ double2 part[128];
  const int b = boxes[blockIdx.x];
  for (int j = 0; j < H.tgt_own_count[b]; ++j) {
    const int ts = H.tgt_own_start[b] + j;
    const double4 t = H.tgt[ts];
    double2 tot = make_double2(0, 0);
    for (int64_t e = H.wfar_starts[b]; e < H.wfar_starts[b + 1]; ++e) {
      const int d = H.wfar_box[e];
      const double4 dc = H.box[d];
      __syncthreads();
      wave_table_cta(H.k, H.P, t.x - dc.x, t.y - dc.y, t.z - dc.z, true, S, rad);
      double2 a = make_double2(0, 0);
      for (int i = threadIdx.x; i < H.KP; i += blockDim.x) a = cfma(H.M[size_t(d) * H.KP + i], S[i], a);
      part[threadIdx.x] = a;
      __syncthreads();
      if (threadIdx.x == 0)
        for (int i = 0; i < blockDim.x; ++i) {
          tot.x += part[i].x;
          tot.y += part[i].y;
        }
    }
    if (threadIdx.x == 0) {
      const double2 v = H.phi[ts];
      H.phi[ts] = make_double2(v.x + tot.x, v.y + tot.y);
    }
  }
}

// Stage 9
__global__ void k_h_eval_assoc(HelmData H, int n, const int* __restrict__ items, const double* __restrict__ tpos,
                               const int* __restrict__ assoc, const int* __restrict__ ctr_sorted,
                               double* __restrict__ pot) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int i = items[t];
  const int cs = ctr_sorted[assoc[i]];
  const double4 c = H.ctr[cs];
  const double vx = tpos[3 * i] - c.x, vy = tpos[3 * i + 1] - c.y, vz = tpos[3 * i + 2] - c.z;
  const double x = H.k * sqrt(vx * vx + vy * vy + vz * vz);
  double2 Y[(kHQmax + 1) * (kHQmax + 1)];
  ylm_all(H.Q, vx, vy, vz, Y);
  double2 a = make_double2(0, 0);
  for (int nn = 0; nn <= H.Q; ++nn) {
    const double jn = sph_j1(nn, x);
    for (int m = -nn; m <= nn; ++m) {
      const double2 v = cmul(H.Lc[size_t(cs) * H.KQ + fi(nn, m)], Y[fi(nn, m)]);
      a.x += jn * v.x;
      a.y += jn * v.y;
    }
  }
  pot[2 * size_t(i)] = a.x;
  pot[2 * size_t(i) + 1] = a.y;
  if (!isfinite(a.x) || !isfinite(a.y)) atomicOr(H.bad, 1u);
}

__global__ void __launch_bounds__(128) k_h_eval_conv(HelmData H, const int* __restrict__ boxes,
                                                     const int* __restrict__ tgt_perm, double* __restrict__ pot) {
  extern __shared__ double2 sm[];
  double2* R = sm;
  double2* rad = sm + H.KP;
  __shared__ double2 part[128];
  const int b = boxes[blockIdx.x];
  const double4 bc = H.box[b];
  for (int j = 0; j < H.tgt_own_count[b]; ++j) {
    const int ts = H.tgt_own_start[b] + j;
    const double4 t = H.tgt[ts];
    __syncthreads();
    wave_table_cta(H.k, H.P, t.x - bc.x, t.y - bc.y, t.z - bc.z, false, R, rad);
    double2 a = make_double2(0, 0);
    for (int i = threadIdx.x; i < H.KP; i += blockDim.x) a = cfma(H.L[size_t(b) * H.KP + i], R[i], a);
    part[threadIdx.x] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 s = H.phi[ts];
      for (int i = 0; i < blockDim.x; ++i) {
        s.x += part[i].x;
        s.y += part[i].y;
      }
      pot[2 * size_t(tgt_perm[ts])] = s.x;
      pot[2 * size_t(tgt_perm[ts]) + 1] = s.y;
      if (!isfinite(s.x) || !isfinite(s.y)) atomicOr(H.bad, 1u);
    }
  }
}

__global__ void k_h_centre_out(HelmData H, int nc, const int* __restrict__ ctr_perm, double* __restrict__ out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= int64_t(nc) * H.KQ) return;
  const int cs = int(t / H.KQ), i = int(t % H.KQ);
  const double2 v = H.Lc[t];
  const int64_t o = (int64_t(ctr_perm[cs]) * H.KQ + i) * 2;
  out[o] = v.x;
  out[o + 1] = v.y;
  if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(H.bad, 2u);
}

template <int Q>
void near_q(const HelmData& H, const int* boxes, int n, cudaStream_t s) {
  const size_t smem = size_t((Q + 1) * (Q + 1)) * 128 * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_h_near<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_h_near<Q><<<n, 128, smem, s>>>(H, boxes);
}


// ---------------------------------------------------------------- point-and-shoot M2L
// (the Helmholtz M2L for P <= 20)
// In the split M2L's azimuthal frame the operator of offset v' = (rho, 0, z) factors as
// V(theta) Z(|v'|) W(theta): W rotates the multipole so v' lies on +z, Z translates along
// z (diagonal in m, one complex (P+1-m)^2 block per m, the same for the even and odd
// parts), V rotates the local back (csrc/host/helm_rot.cpp).  All three keep the even /
// odd split (A = y_m + y_-m, B = y_m - y_-m), so one CTA takes one parity of a tile of
// kHColsS entries: (2 x 231 or 2 x 210 real rows) x 16 columns in shared memory, and each
// phase runs its blocks in place as m8n8k4 DMMAs (W, V real, applied to the Re and Im
// rows separately; Z as the real embedding [[Re, -Im], [Im, Re]]).  Output rows are the
// split M2L's staging rows, so k_h_m2l_reduce_split finishes the job.  Per List-2 entry at
// p = 20: 8 x (3,311 + 2,870) real multiply-adds instead of 4 x (231^2 + 210^2).
constexpr int kHpW = 8, kHpLD = kHColsS + 1;
constexpr int kHpGat = 8;  // gather elements per thread with their loads in flight together

__device__ __forceinline__ void hp_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// one block of runtime size S <= 8 MT in place: operator A-fragments (ks, mt) from L2
// (two k-steps ahead), rows rw[] x 16 columns from shared memory.  MT (row tiles of 8)
// is a template parameter so no predicated-off loads or DMMAs are issued for small blocks.
template <int MT>
__device__ __forceinline__ void hp_block_t(double* X, const int* rw, int S, const double* __restrict__ Ob, int lane) {
  const int KS = (S + 3) >> 2;
  double acc[MT][2][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) acc[mt][0][0] = acc[mt][0][1] = acc[mt][1][0] = acc[mt][1][1] = 0.0;
  // operator fragments two k-steps ahead (ring of two register sets)
  double A0[MT], A1[MT];
  auto load = [&](double (&A)[MT], int ks) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) A[mt] = __ldg(Ob + (ks * MT + mt) * 32 + lane);
  };
  auto step = [&](const double (&a)[MT], int ks) {
    const int k = ks * 4 + (lane & 3);
    const int row = k < S ? rw[k] : -1;
    const double b0 = row >= 0 ? X[row * kHpLD + (lane >> 2)] : 0.0;
    const double b1 = row >= 0 ? X[row * kHpLD + 8 + (lane >> 2)] : 0.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      hp_dmma(acc[mt][0][0], acc[mt][0][1], a[mt], b0);
      hp_dmma(acc[mt][1][0], acc[mt][1][1], a[mt], b1);
    }
  };
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) A0[mt] = A1[mt] = 0.0;
  load(A0, 0);
  if (KS > 1) load(A1, 1);
  for (int ks = 0; ks < KS; ks += 2) {
    {
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = A0[mt];
      if (ks + 2 < KS) load(A0, ks + 2);
      step(a, ks);
    }
    if (ks + 1 < KS) {
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = A1[mt];
      if (ks + 3 < KS) load(A1, ks + 3);
      step(a, ks + 1);
    }
  }
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = mt * 8 + (lane >> 2);
    if (r < S) {
      double* x = X + rw[r] * kHpLD + (lane & 3) * 2;
      x[0] = acc[mt][0][0];
      x[1] = acc[mt][0][1];
      x[8] = acc[mt][1][0];
      x[9] = acc[mt][1][1];
    }
  }
}

__device__ __forceinline__ void hp_block(double* X, const int* rw, int S, const double* __restrict__ Ob, int lane) {
  switch ((S + 7) >> 3) {
    case 1: hp_block_t<1>(X, rw, S, Ob, lane); break;
    case 2: hp_block_t<2>(X, rw, S, Ob, lane); break;
    case 3: hp_block_t<3>(X, rw, S, Ob, lane); break;
    case 4: hp_block_t<4>(X, rw, S, Ob, lane); break;
    case 5: hp_block_t<5>(X, rw, S, Ob, lane); break;
    default: hp_block_t<6>(X, rw, S, Ob, lane); break;
  }
}

// W / V: the Re rows and the Im rows of a degree take the same real operator, so one call
// serves both (rw[0..S) Re rows, rw[S..2S) Im rows): the operator fragments are read from L2
// once and feed four DMMAs (two column groups x Re / Im) instead of two.
template <int MT>
__device__ __forceinline__ void hp_block_dual_t(double* X, const int* rw, int S, const double* __restrict__ Ob,
                                                int lane) {
  const int KS = (S + 3) >> 2;
  double acc[MT][4][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[mt][g][0] = acc[mt][g][1] = 0.0;
  double A0[MT], A1[MT];
  auto load = [&](double (&A)[MT], int ks) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) A[mt] = __ldg(Ob + (ks * MT + mt) * 32 + lane);
  };
  auto step = [&](const double (&a)[MT], int ks) {
    const int k = ks * 4 + (lane & 3);
    const int rr = k < S ? rw[k] : -1, ri = k < S ? rw[S + k] : -1;
    const double b0 = rr >= 0 ? X[rr * kHpLD + (lane >> 2)] : 0.0;
    const double b1 = rr >= 0 ? X[rr * kHpLD + 8 + (lane >> 2)] : 0.0;
    const double b2 = ri >= 0 ? X[ri * kHpLD + (lane >> 2)] : 0.0;
    const double b3 = ri >= 0 ? X[ri * kHpLD + 8 + (lane >> 2)] : 0.0;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      hp_dmma(acc[mt][0][0], acc[mt][0][1], a[mt], b0);
      hp_dmma(acc[mt][1][0], acc[mt][1][1], a[mt], b1);
      hp_dmma(acc[mt][2][0], acc[mt][2][1], a[mt], b2);
      hp_dmma(acc[mt][3][0], acc[mt][3][1], a[mt], b3);
    }
  };
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) A0[mt] = A1[mt] = 0.0;
  load(A0, 0);
  if (KS > 1) load(A1, 1);
  for (int ks = 0; ks < KS; ks += 2) {
    {
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = A0[mt];
      if (ks + 2 < KS) load(A0, ks + 2);
      step(a, ks);
    }
    if (ks + 1 < KS) {
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = A1[mt];
      if (ks + 3 < KS) load(A1, ks + 3);
      step(a, ks + 1);
    }
  }
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = mt * 8 + (lane >> 2);
    if (r < S) {
      double* x = X + rw[r] * kHpLD + (lane & 3) * 2;
      x[0] = acc[mt][0][0];
      x[1] = acc[mt][0][1];
      x[8] = acc[mt][1][0];
      x[9] = acc[mt][1][1];
      double* y = X + rw[S + r] * kHpLD + (lane & 3) * 2;
      y[0] = acc[mt][2][0];
      y[1] = acc[mt][2][1];
      y[8] = acc[mt][3][0];
      y[9] = acc[mt][3][1];
    }
  }
}

__device__ __forceinline__ void hp_block_dual(double* X, const int* rw, int S, const double* __restrict__ Ob,
                                              int lane) {
  switch ((S + 7) >> 3) {
    case 1: hp_block_dual_t<1>(X, rw, S, Ob, lane); break;
    case 2: hp_block_dual_t<2>(X, rw, S, Ob, lane); break;
    default: hp_block_dual_t<3>(X, rw, S, Ob, lane); break;  // S <= P + 1 = 21
  }
}

struct HpHead {
  int base[2][3];  // table offset of (parity, phase)
};

__global__ void __launch_bounds__(kHpW * 32, 2)
    k_h_m2l_pas(HelmData H, const int* __restrict__ tab, int tab_n, HpHead hd, const int4* __restrict__ tiles,
                const int* __restrict__ col_src, const int* __restrict__ col_pos, const double* __restrict__ zops,
                int zstride, const double* __restrict__ wvops, int wvstride, const int* __restrict__ op_cls,
                const double2* __restrict__ cs, double2* __restrict__ temp) {
  extern __shared__ double smp[];
  const int P = H.P, KP = H.KP;
  const int NE = (P + 1) * (P + 2) / 2, NO = P * (P + 1) / 2;
  const int par = blockIdx.x & 1, NC = par ? NO : NE;
  double* X = smp;                                              // 2 NE rows x kHpLD
  int* s_tab = reinterpret_cast<int*>(X + 2 * NE * kHpLD);  // this parity's three tables
  const int t0 = hd.base[par][0], tn = (par == 0 ? hd.base[1][0] : tab_n) - t0;
  int* s_nm = s_tab + tn;                                      // NC: n | m << 8
  __shared__ int s_src[kHColsS], s_pos[kHColsS];
  __shared__ double2 s_cs[kHSolid + 1];
  const int4 tile = tiles[blockIdx.x >> 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // block tables by cp.async: in flight behind the gather, awaited before the first phase
  for (int i = tid; i < tn; i += blockDim.x)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(s_tab + i))),
                 "l"(tab + t0 + i));
  for (int r = tid; r < NC; r += blockDim.x) {
    int n, m;
    if (par)
      od_nm(r, n, m);
    else
      ev_nm(r, n, m);
    s_nm[r] = n | m << 8;
  }
  if (tid < kHColsS) {
    s_src[tid] = tid < tile.z ? col_src[tile.y + tid] : -1;
    s_pos[tid] = tid < tile.z ? col_pos[tile.y + tid] : -1;
  }
  if (tid <= P) s_cs[tid] = cs[size_t(tile.x) * (P + 1) + tid];
  __syncthreads();
  // gather: M' = M e^{i m alpha}, then A = M'_m + M'_-m (A_0 = M'_0) or B = M'_m - M'_-m.
  // A thread owns a row (n, m) -- its rotation factor is read once -- and walks the
  // columns kHpGat at a time with their multipole loads in flight together.
  for (int r = tid; r < NC; r += blockDim.x) {
    const int nm = s_nm[r], n = nm & 255, m = nm >> 8;
    const double2 ro = s_cs[m], rc = make_double2(ro.x, -ro.y);
    const int ip = fi(n, m), im = fi(n, -m);
#pragma unroll
    for (int c0 = 0; c0 < kHColsS; c0 += kHpGat) {
      double2 vp[kHpGat], vm[kHpGat];
#pragma unroll
      for (int u = 0; u < kHpGat; ++u) {
        const int src = s_src[c0 + u];
        vp[u] = vm[u] = make_double2(0.0, 0.0);
        if (src >= 0) {
          const double2* Mb = H.M + size_t(src) * KP;
          vp[u] = __ldg(Mb + ip);
          if (m) vm[u] = __ldg(Mb + im);
        }
      }
#pragma unroll
      for (int u = 0; u < kHpGat; ++u) {
        const double2 xp = cmul(vp[u], ro);
        double2 v = xp;
        if (m) {
          const double2 xm = cmul(vm[u], rc);
          v = par ? make_double2(xp.x - xm.x, xp.y - xm.y) : make_double2(xp.x + xm.x, xp.y + xm.y);
        }
        X[(2 * r) * kHpLD + c0 + u] = v.x;
        X[(2 * r + 1) * kHpLD + c0 + u] = v.y;
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const double* wv = wvops + size_t(op_cls[tile.x]) * wvstride;
  const double* z = zops + size_t(tile.x) * zstride;
#pragma unroll 1
  for (int ph = 0; ph < 3; ++ph) {
    const int* T = s_tab + (hd.base[par][ph] - t0);
    const int nblk = T[0];
    const int* rowoff = T + 1;
    const int* opoff = rowoff + nblk + 1;
    const int* bsz = opoff + nblk;
    const int* rows = bsz + nblk;
    const int* woff = rows + rowoff[nblk];
    const int* wblk = woff + kHpW + 1;
    const double* Op = ph == 1 ? z : wv;
#pragma unroll 1
    for (int i = woff[warp]; i < woff[warp + 1]; ++i) {
      const int b = wblk[i];
      if (ph == 1)
        hp_block(X, rows + rowoff[b], bsz[b], Op + opoff[b], lane);
      else
        hp_block_dual(X, rows + rowoff[b], bsz[b] >> 1, Op + opoff[b], lane);  // Re rows, then Im rows
    }
    __syncthreads();
  }
  // staging rows: [A (NE) ; B (NO)] complex per entry
  for (int r = tid; r < NC; r += blockDim.x)
    for (int c = 0; c < tile.z; ++c)
      temp[size_t(s_pos[c]) * KP + (par ? NE : 0) + r] =
          make_double2(X[(2 * r) * kHpLD + c], X[(2 * r + 1) * kHpLD + c]);
}

// Z blocks (fragment order, real embedding) and e^{i m alpha} per operator
struct HpZOff {
  int off[kHSolid + 1];
};
__global__ void __launch_bounds__(256) k_h_build_zpas(HelmData H, const double4* __restrict__ shifts, HpZOff zo,
                                                      int zstride, double* __restrict__ zops,
                                                      double2* __restrict__ cs) {
  extern __shared__ double2 smz[];
  const int P = H.P, L = 2 * P;
  double2* F = smz;
  double2* rad = F + (L + 1) * (L + 1);
  double2* Zc = rad + L + 1;  // per m: (P+1-m)^2, row-major [out n2][in n]
  const double4 t = shifts[blockIdx.x];
  const double rho = sqrt(t.x * t.x + t.y * t.y);
  const double alpha = rho > 0 ? atan2(t.y, t.x) : 0.0;
  if (threadIdx.x <= P) {
    double sn, cn;
    sincos(threadIdx.x * alpha, &sn, &cn);
    cs[size_t(blockIdx.x) * (P + 1) + threadIdx.x] = make_double2(cn, sn);
  }
  wave_table_cta(H.k, L, 0.0, 0.0, sqrt(rho * rho + t.z * t.z), true, F, rad);
  int tot = 0;
  for (int m = 0; m <= P; ++m) tot += (P + 1 - m) * (P + 1 - m);
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int m = 0, base = 0;
    while (e >= base + (P + 1 - m) * (P + 1 - m)) {
      base += (P + 1 - m) * (P + 1 - m);
      ++m;
    }
    const int tq = P + 1 - m, i = (e - base) / tq, j = (e - base) % tq;
    Zc[e] = t_entry(H, F, m + i, m, m + j, m);
  }
  __syncthreads();
  double* Zb = zops + size_t(blockIdx.x) * zstride;
  int base = 0;
  for (int m = 0; m <= P; ++m) {
    const int tq = P + 1 - m, s = 2 * tq, MT = (s + 7) / 8, KS = (s + 3) / 4;
    for (int e = threadIdx.x; e < MT * KS * 32; e += blockDim.x) {
      const int fr = e >> 5, l = e & 31, ks = fr / MT, mt = fr - ks * MT;
      const int i = mt * 8 + l / 4, j = ks * 4 + l % 4;
      double v = 0.0;
      if (i < s && j < s) {
        const double2 zz = Zc[base + (i % tq) * tq + (j % tq)];
        const int pi = i / tq, pj = j / tq;
        v = (pi == pj) ? zz.x : (pi == 0 ? -zz.y : zz.y);
      }
      Zb[zo.off[m] + e] = v;
    }
    base += tq * tq;
  }
}

}  // namespace

void helm_upload_constants() {
  double sa[kHSolid + 1] = {0}, sb[kHSolid + 1] = {0};
  double sc[(kHSolid + 1) * (kHSolid + 1)] = {0}, sd[(kHSolid + 1) * (kHSolid + 1)] = {0};
  for (int m = 1; m <= kHSolid; ++m) sa[m] = std::sqrt((2.0 * m + 1.0) / (2.0 * m));
  for (int m = 0; m <= kHSolid; ++m) sb[m] = std::sqrt(2.0 * m + 3.0);
  for (int n = 2; n <= kHSolid; ++n)
    for (int m = 0; m + 2 <= n; ++m) {
      sc[n * (kHSolid + 1) + m] = std::sqrt((4.0 * n * n - 1.0) / (double(n) * n - double(m) * m));
      sd[n * (kHSolid + 1) + m] = std::sqrt(((n - 1.0) * (n - 1.0) - double(m) * m) / (4.0 * (n - 1.0) * (n - 1.0) - 1.0));
    }
  double jser[(kHSolid + 2) * kHSer], odd[2 * kHSolid + 4];
  for (int n = 0; n < kHSolid + 2; ++n)
    for (int t = 1; t <= kHSer; ++t) jser[n * kHSer + t - 1] = -1.0 / (2.0 * t * (2.0 * n + 2.0 * t + 1.0));
  for (int n = 0; n < kHSolid + 2; ++n) {
    odd[2 * n] = 2.0 * n + 1.0;
    odd[2 * n + 1] = 1.0 / (2.0 * n + 1.0);
  }
  cudaMemcpyToSymbol(c_jser, jser, sizeof(jser));
  cudaMemcpyToSymbol(c_odd, odd, sizeof(odd));
  cudaMemcpyToSymbol(c_sa, sa, sizeof(sa));
  cudaMemcpyToSymbol(c_sb, sb, sizeof(sb));
  cudaMemcpyToSymbol(c_sc, sc, sizeof(sc));
  cudaMemcpyToSymbol(c_sd, sd, sizeof(sd));
  double sap[kHSolid + 1];
  sap[0] = 0.28209479177387814347;
  for (int m = 1; m <= kHSolid; ++m) sap[m] = sap[m - 1] * sa[m];
  cudaMemcpyToSymbol(g_sap, sap, sizeof(sap));
  cudaMemcpyToSymbol(g_sa, sa, sizeof(sa));
  cudaMemcpyToSymbol(g_sb, sb, sizeof(sb));
  cudaMemcpyToSymbol(g_sc, sc, sizeof(sc));
  cudaMemcpyToSymbol(g_sd, sd, sizeof(sd));
}

int helm_gather(const HelmData& H, int64_t ns, const int* perm, const double* w, const double* mu, cudaStream_t s) {
  if (ns == 0) return 0;
  k_h_gather<<<unsigned((ns + 255) / 256), 256, 0, s>>>(ns, perm, w, H.hmu ? mu : nullptr, H.hw, H.hmu);
  return 1;
}

int helm_p2m(const HelmData& H, const int* leaves, int n, cudaStream_t s) {
  if (n == 0) return 0;
  if (!H.hmu && H.KP <= 32 * kHP2LSlots) {  // single layer: one source per warp
    const size_t smem = size_t(8) * (H.KP + kHP2LBatch * (H.P + 1)) * sizeof(double2);
    cudaFuncSetAttribute(k_h_p2w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_h_p2w<true><<<n, 256, smem, s>>>(H, leaves);
    return 1;
  }
  const int PF = H.hmu ? H.P + 1 : H.P;
  k_h_p2m<<<n, 256, ((PF + 1) * (PF + 1) + PF + 1) * sizeof(double2), s>>>(H, leaves);
  return 1;
}

int helm_shift_pairs(const HelmData& H, int mode, const int2* pairs, int n, const double2* ops, cudaStream_t s) {
  if (n == 0) return 0;
  constexpr int NB = 8;  // 16 measured slower (fewer CTAs per SM)
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_h_shift_b<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int th = H.KP <= 128 ? 128 : H.KP <= 256 ? 256 : 512;
  k_h_shift_b<NB><<<(n + NB - 1) / NB, th, size_t(NB) * H.KP * sizeof(double2), s>>>(H, mode, pairs, n, ops);
  return 1;
}

int helm_build_ops(const HelmData& H, int n_ops, const double4* shifts, double2* ops, cudaStream_t s) {
  if (n_ops == 0) return 0;
  const int L = 2 * H.P;
  const size_t smem = size_t((L + 1) * (L + 1) + L + 1) * sizeof(double2);
  cudaFuncSetAttribute(k_h_build_ops, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_h_build_ops<<<n_ops, 256, smem, s>>>(H, shifts, ops);
  return 1;
}

int helm_m2l_split_cols() { return kHColsS; }


bool helm_pas_supported(int P) { return P >= 1 && P <= 20; }

int helm_build_zpas(const HelmData& H, int n_ops, const double4* shifts, const int* z_off, int zstride, double* zops,
                    double2* cs, cudaStream_t s) {
  if (n_ops == 0) return 0;
  const int L = 2 * H.P;
  int tot = 0;
  for (int m = 0; m <= H.P; ++m) tot += (H.P + 1 - m) * (H.P + 1 - m);
  const size_t smem = size_t((L + 1) * (L + 1) + L + 1 + tot) * sizeof(double2);
  HpZOff zo{};
  for (int m = 0; m <= H.P; ++m) zo.off[m] = z_off[m];
  cudaFuncSetAttribute(k_h_build_zpas, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_h_build_zpas<<<n_ops, 256, smem, s>>>(H, shifts, zo, zstride, zops, cs);
  return 1;
}

// block tables of the pas kernel: per (parity, phase) [nblk][rowoff (nblk+1)][opoff][size]
// [rows][warp offsets (kHpW+1)][block ids], whole blocks per warp by longest-first
void helm_pas_tables(int P, const size_t* wv_off_w0, const size_t* wv_off_w1, const size_t* wv_off_v0,
                     const size_t* wv_off_v1, const size_t* z_off, std::vector<int>& tab, int (&base)[2][3]) {
  auto ev = [](int n, int m) { return n * (n + 1) / 2 + m; };
  auto od = [](int n, int m) { return n * (n - 1) / 2 + m - 1; };
  tab.clear();
  for (int par = 0; par < 2; ++par)
    for (int ph = 0; ph < 3; ++ph) {
      std::vector<std::vector<int>> blocks;
      std::vector<int> opo;
      auto cr = [&](int n, int m) { return par ? od(n, m) : ev(n, m); };
      if (ph != 1) {
        const size_t* off = ph == 0 ? (par ? wv_off_w1 : wv_off_w0) : (par ? wv_off_v1 : wv_off_v0);
        for (int n = par; n <= P; ++n) {  // one block per degree: Re rows, then Im rows, same operator
          std::vector<int> b;
          for (int part = 0; part < 2; ++part)
            for (int m = par; m <= n; ++m) b.push_back(2 * cr(n, m) + part);
          blocks.push_back(b);
          opo.push_back(int(off[n - par]));
        }
      } else {
        for (int m = par; m <= P; ++m) {
          std::vector<int> b;
          for (int part = 0; part < 2; ++part)
            for (int n = m; n <= P; ++n) b.push_back(2 * cr(n, m) + part);
          blocks.push_back(b);
          opo.push_back(int(z_off[m]));
        }
      }
      const int nb = int(blocks.size());
      base[par][ph] = int(tab.size());
      tab.push_back(nb);
      std::vector<int> rows, rowoff{0};
      for (auto& b : blocks) {
        rows.insert(rows.end(), b.begin(), b.end());
        rowoff.push_back(int(rows.size()));
      }
      tab.insert(tab.end(), rowoff.begin(), rowoff.end());
      tab.insert(tab.end(), opo.begin(), opo.end());
      for (auto& b : blocks) tab.push_back(int(b.size()));
      tab.insert(tab.end(), rows.begin(), rows.end());
      std::vector<int> order(nb);
      for (int i = 0; i < nb; ++i) order[i] = i;
      auto cost = [&](int i) {  // DMMA fragments; a W / V block holds two row sets of half its size
        const int sz = ph == 1 ? int(blocks[i].size()) : int(blocks[i].size()) / 2;
        return long((sz + 7) / 8) * ((sz + 3) / 4) * (ph == 1 ? 1 : 2);
      };
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
      std::vector<std::vector<int>> wl(kHpW);
      std::vector<long> load(kHpW, 0);
      for (int bi : order) {
        const int w = int(std::min_element(load.begin(), load.end()) - load.begin());
        load[w] += cost(bi);
        wl[w].push_back(bi);
      }
      std::vector<int> woff{0}, wblk;
      for (auto& v : wl) {
        wblk.insert(wblk.end(), v.begin(), v.end());
        woff.push_back(int(wblk.size()));
      }
      tab.insert(tab.end(), woff.begin(), woff.end());
      tab.insert(tab.end(), wblk.begin(), wblk.end());
    }
}

int helm_m2l_pas(const HelmData& H, int n_tiles, const int4* tiles, const int* col_src, const int* col_pos,
                 const int* tab, int tab_n, const int (&base)[2][3], const double* zops, int zstride,
                 const double* wvops, int wvstride, const int* op_cls, const double2* cs, double2* temp, int n_boxes,
                 const int* boxes, int64_t vbase, const int* ent_op, cudaStream_t s) {
  if (n_tiles == 0) return 0;
  const int P = H.P, NE = (P + 1) * (P + 2) / 2;
  const size_t smem = size_t(2 * NE * kHpLD) * sizeof(double) + size_t(std::max(base[1][0], tab_n - base[1][0]) + NE) * sizeof(int);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_h_m2l_pas, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
      return -1;
    attr = smem;
  }
  HpHead hd;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) hd.base[a][b] = base[a][b];
  k_h_m2l_pas<<<2 * n_tiles, kHpW * 32, smem, s>>>(H, tab, tab_n, hd, tiles, col_src, col_pos, zops, zstride, wvops,
                                                    wvstride, op_cls, cs, temp);
  const int th = H.KP <= 128 ? 128 : H.KP <= 256 ? 256 : 512;
  k_h_m2l_reduce_split<<<n_boxes, th, 0, s>>>(H, boxes, vbase, temp, ent_op, cs);
  return 2;
}

template <int Q>
void near_dip_q(const HelmData& H, const int* boxes, int n, cudaStream_t s) {
  const size_t smem = size_t((Q + 1) * (Q + 1)) * 128 * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_h_near_dip<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_h_near_dip<Q><<<n, 128, smem, s>>>(H, boxes);
}

int helm_near(const HelmData& H, const int* boxes, int n, cudaStream_t s) {
  if (n == 0) return 0;
  switch (H.Q) {
#define QBXG_HNEAR(Q)                             \
  case Q:                                         \
    near_q<Q>(H, boxes, n, s);                    \
    if (H.hmu) near_dip_q<Q>(H, boxes, n, s);     \
    break;
    QBXG_HNEAR(0) QBXG_HNEAR(1) QBXG_HNEAR(2) QBXG_HNEAR(3) QBXG_HNEAR(4) QBXG_HNEAR(5) QBXG_HNEAR(6)
#undef QBXG_HNEAR
    default: return -1;
  }
  return H.hmu ? 2 : 1;
}

int helm_p2p(const HelmData& H, const int* boxes, int n, cudaStream_t s) {
  if (n == 0) return 0;
  k_h_p2p<<<n, 128, 0, s>>>(H, boxes);
  return 1;
}

int helm_p2l(const HelmData& H, const int* boxes, int n, cudaStream_t s) {
  if (n == 0) return 0;
  // warp per source (single layer, P <= 20); the double layer takes the CTA-wide table
  // (one more degree for the ladder identities)
  if (!H.hmu && H.KP <= 32 * kHP2LSlots) {
    const size_t smem = size_t(8) * (H.KP + kHP2LBatch * (H.P + 1)) * sizeof(double2);
    cudaFuncSetAttribute(k_h_p2w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_h_p2w<false><<<n, 256, smem, s>>>(H, boxes);
    return 1;
  }
  const int PF = H.hmu ? H.P + 1 : H.P;
  k_h_p2l<<<n, 256, ((PF + 1) * (PF + 1) + PF + 1) * sizeof(double2), s>>>(H, boxes);
  return 1;
}

size_t helm_gaunt_ctr_size(int P, int Q) {
  const size_t NL = P + Q + 1;
  return NL * 2 * NL * (Q + 1) * size_t((Q + 1) * (Q + 1));
}

int helm_build_gaunt_ctr(const HelmData& H, double* out, cudaStream_t s) {
  const size_t n = helm_gaunt_ctr_size(H.P, H.Q);
  k_h_gaunt_ctr<<<unsigned((n + 255) / 256), 256, 0, s>>>(H, out, n);
  return 1;
}

int helm_ctr(const HelmData& H, int singular, const double2* X, int n_ctas, const int4* ctas, const int* ctr_of,
             const int* out_row, double2* out, int accumulate, cudaStream_t s) {
  if (n_ctas == 0) return 0;
  const int NL = H.P + H.Q + 1;
  const size_t smem =
      size_t(H.KP + 2 * H.KQ * (NL | 1) + 3 * kHCtrMax * NL) * sizeof(double2) + size_t(4 * kHCtrMax) * sizeof(double);
  cudaFuncSetAttribute(k_h_ctr, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_h_ctr<<<n_ctas, 256, smem, s>>>(H, singular, X, ctas, ctr_of, out_row, out, accumulate);
  return 1;
}

int helm_pair_reduce(const HelmData& H, const int* centres, const int* starts, int n, const double2* rows,
                     cudaStream_t s) {
  if (n == 0) return 0;
  const int64_t nt = int64_t(n) * H.KQ;
  k_h_pair_reduce<<<unsigned((nt + 255) / 256), 256, 0, s>>>(H, centres, starts, n, rows);
  return 1;
}

int helm_m2p(const HelmData& H, const int* boxes, int n, cudaStream_t s) {
  if (n == 0) return 0;
  k_h_m2p<<<n, 128, (H.KP + H.P + 1) * sizeof(double2), s>>>(H, boxes);
  return 1;
}

int helm_eval(const HelmData& H, int n_assoc, const int* assoc_items, const double* tpos, const int* assoc,
              const int* ctr_sorted, int n_tboxes, const int* tboxes, const int* tgt_perm, double* pot,
              cudaStream_t s) {
  int k = 0;
  if (n_assoc) {
    k_h_eval_assoc<<<(n_assoc + 127) / 128, 128, 0, s>>>(H, n_assoc, assoc_items, tpos, assoc, ctr_sorted, pot);
    ++k;
  }
  if (n_tboxes) {
    k_h_eval_conv<<<n_tboxes, 128, (H.KP + H.P + 1) * sizeof(double2), s>>>(H, tboxes, tgt_perm, pot);
    ++k;
  }
  return k;
}

int helm_centre_out(const HelmData& H, int nc, const int* ctr_perm, double* out, cudaStream_t s) {
  if (nc == 0) return 0;
  const int64_t nt = int64_t(nc) * H.KQ;
  k_h_centre_out<<<unsigned((nt + 255) / 256), 256, 0, s>>>(H, nc, ctr_perm, out);
  return 1;
}

}  // namespace dev
}  // namespace qbxg
