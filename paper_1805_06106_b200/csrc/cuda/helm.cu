// Helmholtz single (+ double) layer G_k = e^{ik|x-y|}/(4 pi |x-y|) (BASELINE config 3,
// SURVEY.md §8 a18): the unaccelerated paths on the GPU -- the direct sum and
// direct QBX (every centre's order-q local from all sources) --
// in complex128, with the formulation of oracle/helm_oracle.cpp:
//   L_n^m = ik sum_s w_s h_n(k|s-c|) conj(Y_n^m(s-c)) [+ ik mu_s . grad_s of the same],
//   phi(t) = sum L_n^m j_n(k|t-c|) Y_n^m(t-c),
// orthonormal Y_n^m without the Condon-Shortley phase, full tables (q+1)^2, index
// n^2 + n + m.  The FMM stages are in helm_fmm.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "helm_math.cuh"
#include "kernels.cuh"

namespace qbxg {
namespace dev {
namespace {

using namespace hm;

constexpr int kHChunk = 256;

// direct sum, thread per target, sources staged per CTA
__global__ void __launch_bounds__(256) k_helm_direct_sum(double k, int ns, const double4* __restrict__ src,
                                                         const double2* __restrict__ w,
                                                         const double2* __restrict__ mu, int nt,
                                                         const double4* __restrict__ tgt, double2* __restrict__ pot,
                                                         unsigned long long* __restrict__ bad) {
  __shared__ double4 s_src[kHChunk];
  __shared__ double2 s_w[kHChunk];
  __shared__ double2 s_mu[kHChunk][3];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const double4 x = t < nt ? tgt[t] : make_double4(0, 0, 0, 0);
  double2 acc = make_double2(0, 0);
  for (int ch = 0; ch < ns; ch += kHChunk) {
    const int nch = min(kHChunk, ns - ch);
    __syncthreads();
    for (int f = threadIdx.x; f < nch; f += blockDim.x) {
      s_src[f] = src[ch + f];
      s_w[f] = w[ch + f];
      if (mu)
        for (int d = 0; d < 3; ++d) s_mu[f][d] = mu[3 * size_t(ch + f) + d];
    }
    __syncthreads();
    if (t < nt)
      for (int j = 0; j < nch; ++j) {
        const double dx = x.x - s_src[j].x, dy = x.y - s_src[j].y, dz = x.z - s_src[j].z;
        const double r = sqrt(dx * dx + dy * dy + dz * dz);
        if (r == 0.0) {
          atomicMin(bad, (static_cast<unsigned long long>(t) << 32) | static_cast<unsigned>(ch + j));
          continue;
        }
        double s, c;
        sincos(k * r, &s, &c);
        const double f = 1.0 / (4.0 * kPi * r);
        acc = cfma(s_w[j], make_double2(c * f, s * f), acc);
        if (mu) {
          const double2 m3[3] = {s_mu[j][0], s_mu[j][1], s_mu[j][2]};
          const double2 v = dipole_kernel(k, dx, dy, dz, r, m3);
          acc.x += v.x;
          acc.y += v.y;
        }
      }
  }
  if (t < nt) pot[t] = acc;
}

// direct QBX: 32 centres x 4 source slices per CTA; Lc = ik sum w h_n conj(Y)
template <int Q, bool DIP>
__global__ void __launch_bounds__(128) k_helm_direct_qbx(double k, int ns, const double4* __restrict__ src,
                                                         const double2* __restrict__ w,
                                                         const double2* __restrict__ mu, int nc,
                                                         const double4* __restrict__ ctr, double2* __restrict__ Lc) {
  constexpr int KQ = (Q + 1) * (Q + 1);
  __shared__ double4 s_src[kHChunk];
  __shared__ double2 s_w[kHChunk];
  __shared__ double2 s_mu[DIP ? kHChunk : 1][3];
  const int ci = threadIdx.x >> 2, sl = threadIdx.x & 3;
  const int cid = blockIdx.x * 32 + ci;
  const bool active = cid < nc;
  const double4 c = active ? ctr[cid] : make_double4(0, 0, 0, 1);
  double2 acc[KQ];
#pragma unroll
  for (int i = 0; i < KQ; ++i) acc[i] = make_double2(0, 0);
  for (int ch = 0; ch < ns; ch += kHChunk) {
    const int nch = min(kHChunk, ns - ch);
    __syncthreads();
    for (int f = threadIdx.x; f < nch; f += blockDim.x) {
      s_src[f] = src[ch + f];
      s_w[f] = w[ch + f];
      if (DIP)
        for (int d = 0; d < 3; ++d) s_mu[f][d] = mu[3 * size_t(ch + f) + d];
    }
    __syncthreads();
    if (!active) continue;
    for (int j = sl; j < nch; j += 4) {
      const double vx = s_src[j].x - c.x, vy = s_src[j].y - c.y, vz = s_src[j].z - c.z;
      const double x = k * sqrt(vx * vx + vy * vy + vz * vz);
      double2 Y[KQ];
      ylm_all(Q, vx, vy, vz, Y);
      // y_n upward (stable), j_n accurate for the Im part
      double ym = -cos(x) / x, y0 = -cos(x) / (x * x) - sin(x) / x;
      const double2 f0 = make_double2(-k * s_w[j].y, k * s_w[j].x);  // ik w
#pragma unroll
      for (int n = 0; n <= Q; ++n) {
        double yn;
        if (n == 0) {
          yn = ym;
        } else if (n == 1) {
          yn = y0;
        } else {
          yn = (2.0 * n - 1.0) / x * y0 - ym;
          ym = y0;
          y0 = yn;
        }
        const double2 fh = cmul(f0, make_double2(sph_j1(n, x), yn));
#pragma unroll
        for (int m = -n; m <= n; ++m) {
          const double2 yc = make_double2(Y[fi(n, m)].x, -Y[fi(n, m)].y);
          acc[fi(n, m)] = cfma(fh, yc, acc[fi(n, m)]);
        }
      }
      if (DIP) {
        const double2 m3[3] = {s_mu[j][0], s_mu[j][1], s_mu[j][2]};
        dipole_terms<Q, true>(k, vx, vy, vz, m3, make_double2(0.0, k), acc);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < KQ; ++i) {
    acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, 1, 4);
    acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, 1, 4);
    acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, 2, 4);
    acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, 2, 4);
  }
  if (active && sl == 0)
#pragma unroll
    for (int i = 0; i < KQ; ++i) Lc[size_t(cid) * KQ + i] = acc[i];
}

// QBXL2P for the associated targets (caller's order)
__global__ void k_helm_direct_qbx_eval(double k, int q, int n, const double* __restrict__ tpos,
                                       const int* __restrict__ assoc, const double4* __restrict__ ctr,
                                       const double2* __restrict__ Lc, double2* __restrict__ pot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = assoc[i];
  if (a < 0) return;
  const double4 c = ctr[a];
  const double vx = tpos[3 * i] - c.x, vy = tpos[3 * i + 1] - c.y, vz = tpos[3 * i + 2] - c.z;
  const double x = k * sqrt(vx * vx + vy * vy + vz * vz);
  double2 Y[(kHQmax + 1) * (kHQmax + 1)];
  ylm_all(q, vx, vy, vz, Y);
  const int KQ = (q + 1) * (q + 1);
  double2 acc = make_double2(0, 0);
  for (int nn = 0; nn <= q; ++nn) {
    const double jn = sph_j1(nn, x);
    for (int m = -nn; m <= nn; ++m) {
      const double2 v = cmul(Lc[size_t(a) * KQ + fi(nn, m)], Y[fi(nn, m)]);
      acc.x += jn * v.x;
      acc.y += jn * v.y;
    }
  }
  pot[i] = acc;
}

template <int Q>
void helm_qbx_q(double k, int ns, const double4* src, const double2* w, const double2* mu, int nc,
                const double4* ctr, double2* Lc, cudaStream_t s) {
  if (mu)
    k_helm_direct_qbx<Q, true><<<(nc + 31) / 32, 128, 0, s>>>(k, ns, src, w, mu, nc, ctr, Lc);
  else
    k_helm_direct_qbx<Q, false><<<(nc + 31) / 32, 128, 0, s>>>(k, ns, src, w, mu, nc, ctr, Lc);
}

}  // namespace

int launch_helm_direct_sum(double k, int ns, const double4* src, const double2* w, const double2* mu, int nt,
                           const double4* tgt, double2* pot, unsigned long long* bad, cudaStream_t s) {
  if (nt == 0) return 0;
  k_helm_direct_sum<<<(nt + 255) / 256, 256, 0, s>>>(k, ns, src, w, mu, nt, tgt, pot, bad);
  return 1;
}

int launch_helm_direct_qbx(double k, int q, int ns, const double4* src, const double2* w, const double2* mu, int nc,
                           const double4* ctr, double2* Lc, int nt, const double* tpos, const int* assoc,
                           double2* pot, cudaStream_t s) {
  if (nc > 0) {
    switch (q) {
      case 0: helm_qbx_q<0>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 1: helm_qbx_q<1>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 2: helm_qbx_q<2>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 3: helm_qbx_q<3>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 4: helm_qbx_q<4>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 5: helm_qbx_q<5>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 6: helm_qbx_q<6>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 7: helm_qbx_q<7>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      case 8: helm_qbx_q<8>(k, ns, src, w, mu, nc, ctr, Lc, s); break;
      default: return -1;
    }
  }
  if (nt > 0) k_helm_direct_qbx_eval<<<(nt + 127) / 128, 128, 0, s>>>(k, q, nt, tpos, assoc, ctr, Lc, pot);
  return 2;
}

}  // namespace dev
}  // namespace qbxg
