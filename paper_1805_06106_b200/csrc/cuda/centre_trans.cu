// Box expansion -> QBX-centre local translations and M2P:
//   Stage 5b M2QBXL (List 3 far):
//     L~_c(n,m) += (r/h)^n (1/h) (-1)^{n+m} sum_{j<=p,k} M~_d(j,k) I_{j+n}^{k-m}((c - c_d)/h)
//   Stage 8 L2QBXL:
//     L~_c(n,m) += (r/h)^n sum_{j>=n,k} L~_b(j,k) R_{j-n}^{k-m}((c - c_b)/h)
//   Stage 5b M2P at conventional targets:
//     phi_t += (1/h) sum_{n,m} M~_d(n,m) I_n^m((t - c_d)/h)
// M2QBXL runs box-major over (centre, List-3-far box) pairs (k_m2qbxl3 + the centre-major
// pair reduce), L2QBXL over CTAs of <= 128 centres from <= 8 boxes (k_l2qbxl3); both
// stage the box expansions in shared memory and stream each centre's harmonics one
// azimuthal column at a time in registers.
#include <cuda_runtime.h>

#include "harmonics.cuh"
#include "kernels.cuh"

namespace qbxg {
namespace dev {

namespace {

// M2P: conventional targets of boxes with List 3 far entries; thread per target.
__global__ void __launch_bounds__(128) k_m2p(DevData D, const int* __restrict__ boxes) {
  extern __shared__ double2 sm[];
  const int b = boxes[blockIdx.x];
  const int ntg = D.tgt_own_count[b], t0 = D.tgt_own_start[b];
  const int64_t eb = D.wfar_starts[b], ee = D.wfar_starts[b + 1];
  for (int tc = 0; tc < ntg; tc += blockDim.x) {
    const int ti = tc + threadIdx.x;
    double4 t = make_double4(0, 0, 0, 0);
    if (ti < ntg) t = D.tgt[t0 + ti];
    double acc = 0.0;
    for (int64_t e = eb; e < ee; ++e) {
      const int d = D.wfar_box[e];
      const double4 bd = D.box[d];
      const double ih = 1.0 / bd.w;
      __syncthreads();
      for (int i = threadIdx.x; i < D.kp; i += blockDim.x) sm[i] = D.M[size_t(d) * D.kp + i];
      __syncthreads();
      if (ti < ntg) {
        // Re sum_{n,|m|<=n} M I = sum_n [M_n^0 I_n^0 + 2 sum_{m>0} Re(M_n^m I_n^m)]
        const double x = (t.x - bd.x) * ih, y = (t.y - bd.y) * ih, z = (t.z - bd.z) * ih;
        const double ir2 = 1.0 / (x * x + y * y + z * z);
        double2 dg = make_double2(sqrt(ir2), 0.0);
        double s = 0.0;
        for (int m = 0; m <= D.p; ++m) {
          const double fm = m ? 2.0 : 1.0;
          if (m > 0) {
            const double sc = (2 * m - 1) * ir2;
            dg = make_double2((dg.x * x - dg.y * y) * sc, (dg.x * y + dg.y * x) * sc);
          }
          double2 a = dg, mm = sm[hidx(m, m)];
          s += fm * (mm.x * a.x - mm.y * a.y);
          if (m + 1 > D.p) break;
          const double s1 = (2 * m + 1) * z * ir2;
          double2 bb = make_double2(s1 * dg.x, s1 * dg.y);
          mm = sm[hidx(m + 1, m)];
          s += fm * (mm.x * bb.x - mm.y * bb.y);
          for (int n = m + 2; n <= D.p; ++n) {
            const double c1 = (2 * n - 1) * z, c2 = double((n - 1 + m) * (n - 1 - m));
            const double2 cc = make_double2((c1 * bb.x - c2 * a.x) * ir2, (c1 * bb.y - c2 * a.y) * ir2);
            mm = sm[hidx(n, m)];
            s += fm * (mm.x * cc.x - mm.y * cc.y);
            a = bb;
            bb = cc;
          }
        }
        acc += ih * s;
      }
    }
    if (ti < ntg) D.phi[t0 + ti] += acc;
  }
}

__global__ void k_pair_reduce(const int* __restrict__ centres, const int* __restrict__ starts, int n, int kq,
                              int pair_base, const double2* __restrict__ temp, double2* __restrict__ Lc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * kq) return;
  const int i = t / kq, c = t % kq;
  double2 acc = Lc[size_t(centres[i]) * kq + c];
  for (int p = starts[i]; p < starts[i + 1]; ++p) {
    const double2 v = temp[size_t(p - pair_base) * kq + c];
    acc.x += v.x;
    acc.y += v.y;
  }
  Lc[size_t(centres[i]) * kq + c] = acc;
}


// L2QBXL, box-table variant: a CTA takes up to kL3Threads consecutive centres
// spanning at most kL3Boxes boxes (host-built descriptors).  Each box's local
// is staged once as a zero-padded full table of degree p+q in shared memory, so
// the contraction
//   L~_c(n,m) = (r/h)^n sum_{N,K} [T(N+n, m+K) R_N^K + T(N+n, m-K) R_N^{-K}]
// needs no range predicates, no conjugate-symmetry branches and no global loads:
// per (N, K) every thread issues 2 x hsize(q) complex FMAs against warp-broadcast
// shared reads, with R_N^K streamed from a register recurrence.
template <int Q>
// (166 registers, 3 CTAs per SM: 4.03 ms at config 1.  Measured and not kept: a minimum of
// 4 resident CTAs -> 128 registers with spills, 4.50 ms; a minimum of 1 -> ptxas takes more
// registers still, 4.88 ms.)
__global__ void __launch_bounds__(kL3Threads) k_l2qbxl3(DevData D, const int* __restrict__ items,
                                                        const int2* __restrict__ ctas,
                                                        const int* __restrict__ ctr_box) {
  constexpr int KQ = hsize(Q);
  extern __shared__ double2 s_tab[];  // kL3Boxes x TS
  __shared__ int s_box[kL3Boxes];
  __shared__ int s_wcount[kL3Threads / 32];
  const int P = D.p, NT = P + Q + 1, TS = NT * NT;
  const int2 cta = ctas[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const bool active = t < cta.y;
  int cs = -1, b = -1, prevb = -2;
  if (active) {
    cs = items[cta.x + t];
    b = ctr_box[cs];
    if (t > 0) prevb = ctr_box[items[cta.x + t - 1]];
  }
  const bool head = active && b != prevb;
  const unsigned bal = __ballot_sync(0xffffffffu, head);
  if (lane == 0) s_wcount[w] = __popc(bal);
  __syncthreads();
  int base = 0, nbox = 0;
#pragma unroll
  for (int i = 0; i < kL3Threads / 32; ++i) {
    base += i < w ? s_wcount[i] : 0;
    nbox += s_wcount[i];
  }
  const int slot = base + __popc(bal & ((2u << lane) - 1u)) - 1;
  if (head) s_box[slot] = b;
  __syncthreads();
  {  // zero-padded full tables of the CTA's boxes.  A thread's table positions r = t + 128 u
     // are the same for every box: their (degree, order) codes are formed once, and a box's
     // loads are all in flight together.
    constexpr int NU = 8;  // covers (P + Q + 1)^2 <= 1024
    int code[NU];          // -2: beyond the table, -1: degree > p (zero), else hidx | conj << 16 | odd << 17
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int r = t + u * kL3Threads;
      code[u] = -2;
      if (r < TS) {
        int j = int(sqrt(double(r)));
        while (j * j > r) --j;
        while ((j + 1) * (j + 1) <= r) ++j;
        const int k = r - j * j - j;
        code[u] = j <= P ? (hidx(j, k < 0 ? -k : k) | (k < 0 ? 1 << 16 : 0) | ((k & 1) << 17)) : -1;
      }
    }
    for (int sb = 0; sb < nbox; ++sb) {
      const double2* __restrict__ Lb = D.L + size_t(s_box[sb]) * D.kp;
      double2 h[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        h[u] = make_double2(0.0, 0.0);
        if (code[u] >= 0) h[u] = Lb[code[u] & 0xffff];
      }
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (code[u] >= -1) {
          double2 v = h[u];
          if (code[u] >= 0 && (code[u] >> 16 & 1)) v = (code[u] >> 17 & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
          s_tab[sb * TS + t + u * kL3Threads] = v;
        }
    }
  }
  __syncthreads();
  if (!active) return;
  const double2* __restrict__ tb = s_tab + slot * TS;
  const double4 bc = D.box[b];
  const double ih = 1.0 / bc.w;
  const double4 c = D.ctr[cs];
  const double x = (c.x - bc.x) * ih, y = (c.y - bc.y) * ih, z = (c.z - bc.z) * ih;
  const double r2 = x * x + y * y + z * z;
  double ax[KQ], ay[KQ];
#pragma unroll
  for (int i = 0; i < KQ; ++i) ax[i] = ay[i] = 0.0;
  double2 diag = make_double2(1.0, 0.0);
  for (int K = 0; K <= P; ++K) {
    if (K > 0) {
      const double s = 1.0 / (2.0 * K);
      diag = make_double2((diag.x * x - diag.y * y) * s, (diag.x * y + diag.y * x) * s);
    }
    const double sg = (K & 1) ? -1.0 : 1.0;
    double2 ra = make_double2(0.0, 0.0), rb = diag;
    for (int N = K; N <= P; ++N) {
      double2 cur;
      if (N == K) {
        cur = diag;
      } else if (N == K + 1) {
        cur = make_double2(z * diag.x, z * diag.y);
      } else {
        const double c1 = (2 * N - 1) * z;
        const double f = c_inv_nm[hidx(N, K)];  // 1 / ((N - K)(N + K)), uniform across the CTA
        cur = make_double2((c1 * rb.x - r2 * ra.x) * f, (c1 * rb.y - r2 * ra.y) * f);
      }
      if (N > K) {
        ra = rb;
        rb = cur;
      }
      const double2 cm = make_double2(sg * cur.x, -sg * cur.y);  // R_N^{-K}
#pragma unroll
      for (int n = 0; n <= Q; ++n) {
        if (N + n > P) break;  // the box local has no degree above p (uniform branch: ~1/3 of the terms)
        const int j = N + n;
        const double2* __restrict__ row = tb + j * j + j;
#pragma unroll
        for (int m = 0; m <= n; ++m) {
          const int id = hidx(n, m);
          const double2 a1 = row[m + K];
          ax[id] = fma(a1.x, cur.x, fma(-a1.y, cur.y, ax[id]));
          ay[id] = fma(a1.x, cur.y, fma(a1.y, cur.x, ay[id]));
          if (K > 0) {
            const double2 a2 = row[m - K];
            ax[id] = fma(a2.x, cm.x, fma(-a2.y, cm.y, ax[id]));
            ay[id] = fma(a2.x, cm.y, fma(a2.y, cm.x, ay[id]));
          }
        }
      }
    }
  }
  double f = 1.0;
  const double rh = c.w * ih;
  double2* out = D.Lc + size_t(cs) * KQ;
#pragma unroll
  for (int n = 0; n <= Q; ++n) {
#pragma unroll
    for (int m = 0; m <= n; ++m) {
      double2 v = out[hidx(n, m)];
      v.x += ax[hidx(n, m)] * f;
      v.y += ay[hidx(n, m)] * f;
      out[hidx(n, m)] = v;
    }
    f *= rh;
  }
}

template <int Q>
void l2qbxl3_q(const DevData& D, const int* items, const int2* ctas, int n_ctas, const int* ctr_box,
               cudaStream_t s) {
  const size_t smem = size_t(kL3Boxes) * (D.p + Q + 1) * (D.p + Q + 1) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_l2qbxl3<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  upload_inv_nm();  // this translation unit's copy of the reciprocal table
  k_l2qbxl3<Q><<<n_ctas, kL3Threads, smem, s>>>(D, items, ctas, ctr_box);
}

// M2QBXL over (centre, List-3-far box) pairs in box-major order: a CTA takes up
// to kW3Threads pairs drawn from at most kW3Boxes source boxes; each box's
// multipole is staged once as a zero-padded table T(j, k), j in [-q, p+q],
// |k| <= j + 2q, so that with I_N^K streamed from a register recurrence
//   L~_c(n,m) = (r/h)^n (1/h) (-1)^{n+m} sum_{N,K} [T(N-n, K+m) I_N^K + T(N-n, m-K) I_N^{-K}]
// runs without range predicates or global loads.  Each thread writes its pair's
// staging row; k_pair_reduce sums a centre's rows in list order as before.
template <int Q>
__device__ __forceinline__ int w3_idx(int j, int k, int P) {
  const int r = j + Q;
  return r * r + 2 * Q * r + r + Q + k;
}

template <int Q>
__global__ void __launch_bounds__(kW3Threads) k_m2qbxl3(DevData D, const int2* __restrict__ pairs,
                                                        const int* __restrict__ perm,
                                                        const int2* __restrict__ ctas,
                                                        double2* __restrict__ temp) {
  constexpr int KQ = hsize(Q);
  extern __shared__ double2 s_tab[];
  __shared__ int s_box[kW3Boxes];
  __shared__ int s_wcount[kW3Threads / 32];
  const int P = D.p, NR = P + 2 * Q + 1, TS = NR * (NR + 2 * Q);
  const int2 cta = ctas[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const bool active = t < cta.y;
  int pi = -1, d = -1, prevd = -2, cs = 0;
  if (active) {
    pi = perm[cta.x + t];
    const int2 pr = pairs[pi];
    cs = pr.x;
    d = pr.y;
    if (t > 0) prevd = pairs[perm[cta.x + t - 1]].y;
  }
  const bool head = active && d != prevd;
  const unsigned bal = __ballot_sync(0xffffffffu, head);
  if (lane == 0) s_wcount[w] = __popc(bal);
  __syncthreads();
  int base = 0, nbox = 0;
#pragma unroll
  for (int i = 0; i < kW3Threads / 32; ++i) {
    base += i < w ? s_wcount[i] : 0;
    nbox += s_wcount[i];
  }
  const int slot = base + __popc(bal & ((2u << lane) - 1u)) - 1;
  if (head) s_box[slot] = d;
  __syncthreads();
  for (int e = t; e < nbox * TS; e += kW3Threads) {
    const int sb = e / TS, o = e - sb * TS;
    // o = r^2 + 2 Q r + (r + Q) + k, k in [-(r + Q), r + Q]
    int r = int(sqrt(double(o + Q * Q))) - Q;
    while (r > 0 && r * r + 2 * Q * r > o) --r;
    while ((r + 1) * (r + 1) + 2 * Q * (r + 1) <= o) ++r;
    const int j = r - Q, k = o - (r * r + 2 * Q * r) - (r + Q);
    double2 v = make_double2(0.0, 0.0);
    if (j >= 0 && j <= P && k >= -j && k <= j) {
      const double2 h = D.M[size_t(s_box[sb]) * D.kp + hidx(j, k < 0 ? -k : k)];
      v = k >= 0 ? h : ((k & 1) ? make_double2(-h.x, h.y) : make_double2(h.x, -h.y));
    }
    s_tab[e] = v;
  }
  __syncthreads();
  if (!active) return;
  const double2* __restrict__ tb = s_tab + slot * TS;
  const double4 bd = D.box[d];
  const double ih = 1.0 / bd.w;
  const double4 c = D.ctr[cs];
  const double x = (c.x - bd.x) * ih, y = (c.y - bd.y) * ih, z = (c.z - bd.z) * ih;
  const double r2 = x * x + y * y + z * z;
  const double rs = rsqrt(r2);
  const double ir2 = rs * rs;
  double ax[KQ], ay[KQ];
#pragma unroll
  for (int i = 0; i < KQ; ++i) ax[i] = ay[i] = 0.0;
  const int NN = P + Q;
  double2 diag = make_double2(rs, 0.0);
  for (int K = 0; K <= NN; ++K) {
    if (K > 0) {
      const double f = (2 * K - 1) * ir2;
      diag = make_double2((diag.x * x - diag.y * y) * f, (diag.x * y + diag.y * x) * f);
    }
    const double sg = (K & 1) ? -1.0 : 1.0;
    double2 ra = make_double2(0.0, 0.0), rb = diag;
    for (int N = K; N <= NN; ++N) {
      double2 cur;
      if (N == K) {
        cur = diag;
      } else if (N == K + 1) {
        const double f = (2 * K + 1) * z * ir2;
        cur = make_double2(f * diag.x, f * diag.y);
      } else {
        const double c1 = (2 * N - 1) * z;
        const double c2 = double((N - 1 + K) * (N - 1 - K));
        cur = make_double2((c1 * rb.x - c2 * ra.x) * ir2, (c1 * rb.y - c2 * ra.y) * ir2);
      }
      if (N > K) {
        ra = rb;
        rb = cur;
      }
      const double2 cm = make_double2(sg * cur.x, -sg * cur.y);  // I_N^{-K}
#pragma unroll
      for (int n = 0; n <= Q; ++n) {
        const double2* __restrict__ row = tb + w3_idx<Q>(N - n, 0, P);
#pragma unroll
        for (int m = 0; m <= n; ++m) {
          const int id = hidx(n, m);
          const double2 a1 = row[K + m];
          ax[id] = fma(a1.x, cur.x, fma(-a1.y, cur.y, ax[id]));
          ay[id] = fma(a1.x, cur.y, fma(a1.y, cur.x, ay[id]));
          if (K > 0) {
            const double2 a2 = row[m - K];
            ax[id] = fma(a2.x, cm.x, fma(-a2.y, cm.y, ax[id]));
            ay[id] = fma(a2.x, cm.y, fma(a2.y, cm.x, ay[id]));
          }
        }
      }
    }
  }
  double f = ih;
  const double rh = c.w * ih;
  double2* out = temp + size_t(pi) * KQ;
#pragma unroll
  for (int n = 0; n <= Q; ++n) {
#pragma unroll
    for (int m = 0; m <= n; ++m) {
      const double sgn = ((n + m) & 1) ? -f : f;
      out[hidx(n, m)] = make_double2(sgn * ax[hidx(n, m)], sgn * ay[hidx(n, m)]);
    }
    f *= rh;
  }
}

template <int Q>
void w3_q(const DevData& D, const PairChunk& C, double2* temp, cudaStream_t s) {
  const int NR = D.p + 2 * Q + 1;
  const size_t smem = size_t(kW3Boxes) * NR * (NR + 2 * Q) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2qbxl3<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_m2qbxl3<Q><<<C.n_ctas, kW3Threads, smem, s>>>(D, C.pairs, C.perm, C.ctas, temp);
}

}  // namespace

int launch_m2p(const DevData& D, const int* tgt_boxes, int n_tgt, cudaStream_t s) {
  if (n_tgt == 0) return 0;
  k_m2p<<<n_tgt, 128, D.kp * sizeof(double2), s>>>(D, tgt_boxes);
  return 1;
}

int launch_m2qbxl_pairs(const DevData& D, const PairPlan& P, cudaStream_t s) {
  int k = 0;
  for (const PairChunk& C : P.chunks) {
    if (C.n_pairs == 0) continue;
    switch (D.q) {
      case 0: w3_q<0>(D, C, P.temp, s); break;
      case 1: w3_q<1>(D, C, P.temp, s); break;
      case 2: w3_q<2>(D, C, P.temp, s); break;
      case 3: w3_q<3>(D, C, P.temp, s); break;
      case 4: w3_q<4>(D, C, P.temp, s); break;
      case 5: w3_q<5>(D, C, P.temp, s); break;
      case 6: w3_q<6>(D, C, P.temp, s); break;
      case 7: w3_q<7>(D, C, P.temp, s); break;
      case 8: w3_q<8>(D, C, P.temp, s); break;
      default: return -1;
    }
    const int nthreads = C.n_centres * D.kq;
    k_pair_reduce<<<(nthreads + 255) / 256, 256, 0, s>>>(C.centres, C.starts, C.n_centres, D.kq, C.pair_base, P.temp,
                                                         D.Lc);
    k += 2;
  }
  return k;
}

int launch_l2qbxl3(const DevData& D, const int* items, const int2* ctas, int n_ctas, const int* ctr_box,
                   cudaStream_t s) {
  if (n_ctas == 0) return 0;
  switch (D.q) {
    case 0: l2qbxl3_q<0>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 1: l2qbxl3_q<1>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 2: l2qbxl3_q<2>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 3: l2qbxl3_q<3>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 4: l2qbxl3_q<4>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 5: l2qbxl3_q<5>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 6: l2qbxl3_q<6>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 7: l2qbxl3_q<7>(D, items, ctas, n_ctas, ctr_box, s); break;
    case 8: l2qbxl3_q<8>(D, items, ctas, n_ctas, ctr_box, s); break;
    default: return -1;
  }
  return 1;
}

}  // namespace dev
}  // namespace qbxg
