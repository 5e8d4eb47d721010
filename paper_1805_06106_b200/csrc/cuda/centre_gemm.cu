// Box expansion -> QBX-centre locals as small GEMMs on the fp64 tensor pipe.
//
// Both Stage 5b M2QBXL (List 3 far) and Stage 8 L2QBXL
// have the form
//   L_c(n,m) = sum_{N,|K|<=N} X_N^K(u_c) S_e(N,K; n,m)
// with X the centre's harmonics relative to the expansion centre (irregular
// I(u) for M2QBXL, u = (c - c_d)/|d|; regular R(u) for L2QBXL, u = (c - c_b)/|b|)
// and S_e a shifted copy of the expansion's coefficients:
//   L2QBXL: S = L~_b(N+n, K+m);   M2QBXL: S = (-1)^{n+m} M~_d(N-n, K+m).
// Folding X_N^{-K} = (-1)^K conj(X_N^K) turns it into a real product
//   C[centres x (q+1)^2] = A[centres x (NN+1)^2] * G_e[(NN+1)^2 x (q+1)^2]
// over real degrees of freedom.  G_e is built once per expansion in shared
// memory (with |e|^-n, or |e|^-(n+1), folded into its columns), A is one
// harmonic row per centre built column-wise by Cartesian recurrences, and the
// product runs as mma.sync m8n8k4 f64.  The epilogue applies r_c^n.
// One CTA = one (box, chunk of 16 centres) work item; M2QBXL accumulates over
// the box's List-3-far entries in the MMA accumulators (fixed order).
#include <cuda_runtime.h>

#include "harmonics.cuh"
#include "kernels.cuh"

namespace qbxg {
namespace dev {

namespace {

constexpr int kRows = 16;     // centres per work item (two m8 tiles)
constexpr int kThreads = 128;
constexpr int kMaxNT = 11;    // n8 tiles: (q+1)^2 <= 88

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int rdof(int n, int m, int part) { return n * n + (m == 0 ? 0 : 2 * m - 1 + part); }

// X_j^k of a half table with X_j^{-k} = (-1)^k conj(X_j^k); zero outside |k| <= j <= P.
__device__ __forceinline__ double2 coef(const double2* __restrict__ T, int P, int j, int k) {
  if (j < 0 || j > P || k > j || k < -j) return make_double2(0.0, 0.0);
  if (k >= 0) return T[hidx(j, k)];
  const double2 v = T[hidx(j, -k)];
  return (k & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
}

struct Geo {
  int P, Q, NN, KR, KRk, SA, NC, SG;  // see setup()
};

__device__ __forceinline__ Geo setup(int P, int Q, bool irreg) {
  Geo g;
  g.P = P;
  g.Q = Q;
  g.NN = irreg ? P + Q : P;
  g.KR = (g.NN + 1) * (g.NN + 1);
  g.KRk = (g.KR + 3) & ~3;
  g.SA = g.KRk;
  while ((g.SA & 7) != 4) g.SA += 4;
  g.NC = ((Q + 1) * (Q + 1) + 7) & ~7;
  g.SG = g.NC + 4;
  while ((g.SG & 7) != 4) g.SG += 4;
  return g;
}

// Build G_e in shared memory.  scale_n = base^(n + off) folds |e|^-n (and 1/|e|).
__device__ void build_G(const Geo& g, bool irreg, const double2* __restrict__ E, double inv_h, double* Gs) {
  const int ncol = (g.Q + 1) * (g.Q + 1);
  for (int idx = threadIdx.x; idx < g.KRk * g.NC; idx += blockDim.x) {
    const int row = idx / g.NC, col = idx % g.NC;
    double v = 0.0;
    if (row < g.KR && col < ncol) {
      int N = int(sqrt(double(row)));
      while (N * N > row) --N;
      while ((N + 1) * (N + 1) <= row) ++N;
      const int rr = row - N * N;
      const int K = rr == 0 ? 0 : (rr + 1) >> 1;
      const int pi = rr == 0 ? 0 : ((rr - 1) & 1);
      int n = int(sqrt(double(col)));
      while (n * n > col) --n;
      while ((n + 1) * (n + 1) <= col) ++n;
      const int cc = col - n * n;
      const int m = cc == 0 ? 0 : (cc + 1) >> 1;
      const int po = cc == 0 ? 0 : ((cc - 1) & 1);
      const int j = irreg ? N - n : N + n;
      double2 sp = coef(E, g.P, j, K + m);
      double2 sm = (K > 0) ? coef(E, g.P, j, m - K) : make_double2(0.0, 0.0);
      double sc = 1.0;
      for (int i = 0; i < n + (irreg ? 1 : 0); ++i) sc *= inv_h;
      if (irreg && ((n + m) & 1)) sc = -sc;
      double Ur, Ui, Wr, Wi;
      if (K == 0) {
        Ur = sp.x;
        Ui = sp.y;
        Wr = Wi = 0.0;
      } else {
        const double s = (K & 1) ? -1.0 : 1.0;
        Ur = sp.x + s * sm.x;
        Ui = sp.y + s * sm.y;
        Wr = sp.x - s * sm.x;
        Wi = sp.y - s * sm.y;
      }
      // L_re = a U_re - b W_im ;  L_im = a U_im + b W_re
      if (po == 0)
        v = (pi == 0) ? Ur : -Wi;
      else
        v = (pi == 0) ? Ui : Wr;
      v *= sc;
    }
    Gs[row * g.SG + col] = v;
  }
}

// Harmonic rows of up to kRows centres: task (centre, column K).
__device__ void build_A(const Geo& g, bool irreg, const double4* __restrict__ ctr, int nrow, double4 e, double inv_h,
                        double* As) {
  for (int t = threadIdx.x; t < kRows * (g.NN + 1); t += blockDim.x) {
    const int r = t / (g.NN + 1), K = t % (g.NN + 1);
    double* row = As + r * g.SA;
    if (r >= nrow) {
      for (int N = K; N <= g.NN; ++N) {
        row[rdof(N, K, 0)] = 0.0;
        if (K > 0) row[rdof(N, K, 1)] = 0.0;
      }
      continue;
    }
    const double4 c = ctr[r];
    const double x = (c.x - e.x) * inv_h, y = (c.y - e.y) * inv_h, z = (c.z - e.z) * inv_h;
    const double r2 = x * x + y * y + z * z;
    const double ir2 = 1.0 / r2;
    double2 d = irreg ? make_double2(sqrt(ir2), 0.0) : make_double2(1.0, 0.0);
    for (int k = 1; k <= K; ++k) {
      const double s = irreg ? (2 * k - 1) * ir2 : 1.0 / (2.0 * k);
      d = make_double2((d.x * x - d.y * y) * s, (d.x * y + d.y * x) * s);
    }
    double2 a = d;
    row[rdof(K, K, 0)] = a.x;
    if (K > 0) row[rdof(K, K, 1)] = a.y;
    if (K + 1 > g.NN) continue;
    const double s1 = irreg ? (2 * K + 1) * z * ir2 : z;
    double2 b = make_double2(s1 * a.x, s1 * a.y);
    row[rdof(K + 1, K, 0)] = b.x;
    if (K > 0) row[rdof(K + 1, K, 1)] = b.y;
    for (int N = K + 2; N <= g.NN; ++N) {
      const double c1 = (2 * N - 1) * z;
      double2 nv;
      if (irreg) {
        const double c2 = double((N - 1 + K) * (N - 1 - K));
        nv = make_double2((c1 * b.x - c2 * a.x) * ir2, (c1 * b.y - c2 * a.y) * ir2);
      } else {
        const double f = 1.0 / double((N - K) * (N + K));
        nv = make_double2((c1 * b.x - r2 * a.x) * f, (c1 * b.y - r2 * a.y) * f);
      }
      row[rdof(N, K, 0)] = nv.x;
      if (K > 0) row[rdof(N, K, 1)] = nv.y;
      a = b;
      b = nv;
    }
  }
  // zero the K padding rows
  for (int t = threadIdx.x; t < kRows * (g.KRk - g.KR); t += blockDim.x) {
    const int r = t / (g.KRk - g.KR), k = g.KR + t % (g.KRk - g.KR);
    As[r * g.SA + k] = 0.0;
  }
}

// C[16 x NC] += A[16 x KRk] * G[KRk x NC]; warps 0,1 take m-tiles, warps 2,3 split n-tiles.
__device__ __forceinline__ void mma_tile(const Geo& g, const double* As, const double* Gs, double (&acc)[kMaxNT][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = warp & 1;
  const int ntiles = g.NC / 8;
  const int half = (ntiles + 1) / 2;
  const int t0 = (warp >> 1) ? half : 0, t1 = (warp >> 1) ? ntiles : half;
  const double* a_row = As + (mt * 8 + (lane >> 2)) * g.SA + (lane & 3);
  for (int k = 0; k < g.KRk; k += 4) {
    const double a = a_row[k];
    const double* brow = Gs + (k + (lane & 3)) * g.SG + (lane >> 2);
#pragma unroll
    for (int t = 0; t < kMaxNT; ++t)
      if (t >= t0 && t < t1) dmma(acc[t][0], acc[t][1], a, brow[t * 8]);
  }
}

__device__ __forceinline__ void epilogue(const Geo& g, const double4* __restrict__ ctr, int nrow,
                                         double2* __restrict__ Lc, int kq, double (&acc)[kMaxNT][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = warp & 1;
  const int ntiles = g.NC / 8;
  const int half = (ntiles + 1) / 2;
  const int t0 = (warp >> 1) ? half : 0, t1 = (warp >> 1) ? ntiles : half;
  const int r = mt * 8 + (lane >> 2);
  if (r >= nrow) return;
  const double rc = ctr[r].w;
  double2* out = Lc + size_t(r) * kq;
  const int ncol = (g.Q + 1) * (g.Q + 1);
#pragma unroll
  for (int t = 0; t < kMaxNT; ++t) {
    if (t < t0 || t >= t1) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = t * 8 + (lane & 3) * 2 + h;
      if (col >= ncol) continue;
      int n = int(sqrt(double(col)));
      while (n * n > col) --n;
      while ((n + 1) * (n + 1) <= col) ++n;
      const int cc = col - n * n;
      const int m = cc == 0 ? 0 : (cc + 1) >> 1;
      const int po = cc == 0 ? 0 : ((cc - 1) & 1);
      double f = 1.0;
      for (int i = 0; i < n; ++i) f *= rc;
      double* dst = reinterpret_cast<double*>(out + hidx(n, m)) + po;
      *dst += f * acc[t][h];
    }
  }
}

// items: (box, first centre offset within the box); M2QBXL iterates the box's W_far entries.
template <bool IRREG>
__global__ void __launch_bounds__(kThreads) k_ctr_gemm(DevData D, const int2* __restrict__ items) {
  extern __shared__ double smem[];
  const Geo g = setup(D.p, D.q, IRREG);
  double* Gs = smem;                       // KRk x SG
  double* As = smem + g.KRk * g.SG;        // kRows x SA
  const int2 it = items[blockIdx.x];
  const int b = it.x;
  const int c0 = D.ctr_own_start[b] + it.y;
  const int nrow = min(kRows, D.ctr_own_count[b] - it.y);
  const double4* ctr = D.ctr + c0;
  double acc[kMaxNT][2];
#pragma unroll
  for (int t = 0; t < kMaxNT; ++t) acc[t][0] = acc[t][1] = 0.0;
  if (IRREG) {
    for (int64_t e = D.wfar_starts[b]; e < D.wfar_starts[b + 1]; ++e) {
      const int d = D.wfar_box[e];
      const double4 bd = D.box[d];
      const double ih = 1.0 / bd.w;
      __syncthreads();
      build_G(g, true, D.M + size_t(d) * D.kp, ih, Gs);
      build_A(g, true, ctr, nrow, bd, ih, As);
      __syncthreads();
      mma_tile(g, As, Gs, acc);
    }
  } else {
    const double4 bb = D.box[b];
    const double ih = 1.0 / bb.w;
    build_G(g, false, D.L + size_t(b) * D.kp, ih, Gs);
    build_A(g, false, ctr, nrow, bb, ih, As);
    __syncthreads();
    mma_tile(g, As, Gs, acc);
  }
  epilogue(g, ctr, nrow, D.Lc + size_t(c0) * D.kq, D.kq, acc);
}

size_t smem_bytes(int p, int q, bool irreg) {
  const int NN = irreg ? p + q : p;
  const int KR = (NN + 1) * (NN + 1);
  const int KRk = (KR + 3) & ~3;
  int SA = KRk;
  while ((SA & 7) != 4) SA += 4;
  const int NC = ((q + 1) * (q + 1) + 7) & ~7;
  int SG = NC + 4;
  while ((SG & 7) != 4) SG += 4;
  return size_t(KRk * SG + kRows * SA) * sizeof(double);
}

}  // namespace

bool ctr_gemm_fits(int p, int q, bool irreg) {
  return smem_bytes(p, q, irreg) <= 220 * 1024 && (q + 1) * (q + 1) <= 8 * kMaxNT;
}

int launch_ctr_gemm(const DevData& D, const int2* items, int n_items, bool irreg, cudaStream_t s) {
  if (n_items == 0) return 0;
  const size_t smem = smem_bytes(D.p, D.q, irreg);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ctr_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_ctr_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  if (irreg)
    k_ctr_gemm<true><<<n_items, kThreads, smem, s>>>(D, items);
  else
    k_ctr_gemm<false><<<n_items, kThreads, smem, s>>>(D, items);
  return 1;
}

}  // namespace dev
}  // namespace qbxg
