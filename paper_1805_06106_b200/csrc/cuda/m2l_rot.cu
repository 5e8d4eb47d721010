// Stage 4 M2L (List 2) by rotation, z-translation and back-rotation
// ("point and shoot"), batched by
// relative box offset exactly like the dense path (m2l_gemm.cu): every column
// of a CTA tile shares one offset, so the three factors are shared too and
// each phase is a small block GEMM on the fp64 tensor pipe (mma.sync m8n8k4):
//   1. X' = Rf X     block diagonal over degree j, (2j+1)^2 blocks   (host: rotation.cpp)
//   2. Y  = Z(rho) X' block diagonal over order m, rows n, cols j in [m,p]:
//                    Z_{nj} = (-1)^{n+m} (j+n)! / rho^{j+n+1}   (computed in the CTA)
//   3. L  = Rb Y     block diagonal over degree n
// Per column ~3.6x fewer tensor-pipe instructions than the dense 256x256
// operator at p = 15.  Output rows go to the same staging buffer and CSR-order
// reduction as the dense path (bitwise deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "harmonics.cuh"
#include "kernels.cuh"

namespace qbxg {
namespace dev {

namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__host__ __device__ __forceinline__ int rboff(int j) { return j * (4 * j * j - 1) / 3; }
inline size_t rot_blocks_size_dev(int p) { return size_t(p + 1) * (2 * p + 1) * (2 * p + 3) / 3; }

constexpr int kMaxKS = 12;  // k-steps per degree block: (2p+1)/4 rounded up, p <= 22

// Ys(rows of degree j) = Rj * Xs(rows of degree j), all degrees, warps round-robin over (j, m-tile).
template <int NT, int SB>
__device__ __forceinline__ void blockdiag(const double* __restrict__ R, int p, const double* Xs, double* Ys) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int item = 0;
  for (int j = 0; j <= p; ++j) {
    const int d = 2 * j + 1, nmt = (d + 7) >> 3, nks = (d + 3) >> 2;
    const double* Rj = R + rboff(j);
    const double* Xj = Xs + j * j * SB;
    double* Yj = Ys + j * j * SB;
    for (int mt = 0; mt < nmt; ++mt, ++item) {
      if ((item & 7) != warp) continue;
      const int row = mt * 8 + (lane >> 2);
      double a[kMaxKS];
#pragma unroll
      for (int ks = 0; ks < kMaxKS; ++ks) {
        const int k = ks * 4 + (lane & 3);
        a[ks] = (ks < nks && row < d && k < d) ? Rj[row * d + k] : 0.0;  // smem (rot2) or global (rot)
      }
      double acc[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < kMaxKS; ++ks) {
        if (ks >= nks) break;
        const int kb = ks * 4 + (lane & 3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b = kb < d ? Xj[kb * SB + nt * 8 + (lane >> 2)] : 0.0;
          dmma(acc[nt][0], acc[nt][1], a[ks], b);
        }
      }
      const int r = mt * 8 + (lane >> 2);
      if (r < d) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          Yj[r * SB + nt * 8 + (lane & 3) * 2] = acc[nt][0];
          Yj[r * SB + nt * 8 + (lane & 3) * 2 + 1] = acc[nt][1];
        }
      }
    }
  }
}

__device__ __forceinline__ int rdof_row(int n, int m, int part) { return n * n + (m == 0 ? 0 : 2 * m - 1 + part); }

// Xs(n, m, part) = sum_{j>=m} (-1)^{n+m} t[n+j] Ys(j, m, part) for every order m (z-axis M2L).
template <int NT, int SB>
__device__ __forceinline__ void ztranslate(const double* __restrict__ t, int p, const double* Ys, double* Xs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int item = 0;
  for (int m = 0; m <= p; ++m) {
    const int d = p + 1 - m, nmt = (d + 7) >> 3, nks = (d + 3) >> 2;
    for (int part = 0; part < (m == 0 ? 1 : 2); ++part)
      for (int mt = 0; mt < nmt; ++mt, ++item) {
        if ((item & 7) != warp) continue;
        const int i = mt * 8 + (lane >> 2);  // output row n = m + i
        double acc[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        for (int ks = 0; ks < nks; ++ks) {
          const int kk = ks * 4 + (lane & 3);  // A column j = m + kk
          double a = 0.0;
          if (i < d && kk < d) a = (i & 1) ? -t[2 * m + i + kk] : t[2 * m + i + kk];
          const int kb = ks * 4 + (lane & 3);
          const double* yrow = Ys + rdof_row(m + kb, m, part) * SB;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double b = kb < d ? yrow[nt * 8 + (lane >> 2)] : 0.0;
            dmma(acc[nt][0], acc[nt][1], a, b);
          }
        }
        if (i < d) {
          double* xrow = Xs + rdof_row(m + i, m, part) * SB;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            xrow[nt * 8 + (lane & 3) * 2] = acc[nt][0];
            xrow[nt * 8 + (lane & 3) * 2 + 1] = acc[nt][1];
          }
        }
      }
  }
}

template <int BN>
__global__ void __launch_bounds__(256) k_m2l_rot(int p, int KR, int KRp, const int4* __restrict__ tiles,
                                                 const int* __restrict__ col_src, const int* __restrict__ col_pos,
                                                 const double* __restrict__ col_scale, const int* __restrict__ rmap,
                                                 const double* __restrict__ M, int kp2,
                                                 const double* __restrict__ rotF, const double* __restrict__ rotB,
                                                 const double* __restrict__ rho_op, size_t rot_stride,
                                                 double* __restrict__ temp) {
  constexpr int NT = BN / 8, SB = BN + 4;
  extern __shared__ double sm[];
  double* Xs = sm;             // KR x SB
  double* Ys = sm + KR * SB;   // KR x SB
  __shared__ double s_t[2 * 24 + 2];
  __shared__ int s_src[BN];
  const int4 tile = tiles[blockIdx.x];
  const int op = tile.x, c0 = tile.y, ncol = tile.z;
  const int tid = threadIdx.x;
  if (tid < BN) s_src[tid] = tid < ncol ? col_src[c0 + tid] : -1;
  if (tid <= 2 * p) {  // t[N] = N! / rho^(N+1)
    const double irho = 1.0 / rho_op[op];
    double v = irho;
    for (int k = 1; k <= tid; ++k) v *= k * irho;
    s_t[tid] = v;
  }
  __syncthreads();
  for (int idx = tid; idx < KR * BN; idx += 256) {
    const int r = idx / BN, c = idx % BN;
    const int src = s_src[c];
    Xs[r * SB + c] = src >= 0 ? __ldg(M + size_t(src) * kp2 + rmap[r]) : 0.0;
  }
  __syncthreads();
  blockdiag<NT, SB>(rotF + size_t(op) * rot_stride, p, Xs, Ys);
  __syncthreads();
  ztranslate<NT, SB>(s_t, p, Ys, Xs);
  __syncthreads();
  blockdiag<NT, SB>(rotB + size_t(op) * rot_stride, p, Xs, Ys);
  __syncthreads();
  for (int idx = tid; idx < ncol * KR; idx += 256) {
    const int c = idx / KR, r = idx % KR;
    temp[size_t(col_pos[c0 + c]) * KRp + r] = Ys[r * SB + c];  // 1/|b| applied by the reduce
  }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Same three phases, with the op's rotation blocks staged in shared memory
// once per CTA and reused over up to kSuper columns (tile.z) of that offset,
// processed BN at a time with the next columns' gather in flight (cp.async).
template <int BN>
__global__ void __launch_bounds__(256) k_m2l_rot2(int p, int KR, int KRp, const int4* __restrict__ tiles,
                                                  const int* __restrict__ col_src, const int* __restrict__ col_pos,
                                                  const double* __restrict__ col_scale, const int* __restrict__ rmap,
                                                  const double* __restrict__ M, int kp2,
                                                  const double* __restrict__ rotF, const double* __restrict__ rotB,
                                                  const double* __restrict__ rho_op, size_t rot_stride,
                                                  double* __restrict__ temp) {
  constexpr int NT = BN / 8, SB = BN + 4;
  extern __shared__ double sm[];
  const int S = int(rot_stride);
  double* Rf = sm;                       // S
  double* Rb = sm + S;                   // S
  double* Xb[2] = {sm + 2 * S, sm + 2 * S + KR * SB};
  double* Ys = sm + 2 * S + 2 * KR * SB;
  __shared__ double s_t[2 * 24 + 2];
  const int4 tile = tiles[blockIdx.x];
  const int op = tile.x, c0 = tile.y, ncol = tile.z;
  const int tid = threadIdx.x;
  // stage the op's blocks (16-byte copies; rot_stride is odd-sized, tail by 8-byte copies)
  {
    const double* gf = rotF + size_t(op) * rot_stride;
    const double* gb = rotB + size_t(op) * rot_stride;
    const bool al = ((reinterpret_cast<uintptr_t>(gf) | reinterpret_cast<uintptr_t>(gb)) & 15) == 0 && (S & 1) == 0;
    const int n16 = al ? S / 2 : 0;
    for (int i = tid; i < n16; i += 256) {
      cp_async16(Rf + 2 * i, gf + 2 * i);
      cp_async16(Rb + 2 * i, gb + 2 * i);
    }
    for (int i = 2 * n16 + tid; i < S; i += 256) {
      cp_async8(Rf + i, gf + i);
      cp_async8(Rb + i, gb + i);
    }
  }
  if (tid <= 2 * p) {
    const double irho = 1.0 / rho_op[op];
    double v = irho;
    for (int k = 1; k <= tid; ++k) v *= k * irho;
    s_t[tid] = v;
  }
  auto gather = [&](double* X, int first) {
    for (int idx = tid; idx < KR * BN; idx += 256) {
      const int r = idx / BN, c = idx % BN;
      if (first + c < ncol)
        cp_async8(X + r * SB + c, M + size_t(col_src[c0 + first + c]) * kp2 + rmap[r]);
      else
        X[r * SB + c] = 0.0;
    }
  };
  gather(Xb[0], 0);
  cp_commit();
  int buf = 0;
  for (int first = 0; first < ncol; first += BN) {
    if (first + BN < ncol) {
      gather(Xb[buf ^ 1], first + BN);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    double* Xs = Xb[buf];
    blockdiag<NT, SB>(Rf, p, Xs, Ys);
    __syncthreads();
    ztranslate<NT, SB>(s_t, p, Ys, Xs);
    __syncthreads();
    blockdiag<NT, SB>(Rb, p, Xs, Ys);
    __syncthreads();
    const int nc = min(BN, ncol - first);
    for (int idx = tid; idx < nc * KR; idx += 256) {
      const int c = idx / KR, r = idx % KR;
      temp[size_t(col_pos[c0 + first + c]) * KRp + r] = Ys[r * SB + c];  // 1/|b| applied by the reduce
    }
    __syncthreads();
    buf ^= 1;
  }
}

// ---- v3: transposed block GEMMs, C[cols x out] = X^T[cols x in] R^T[in x out].
// A warp owns whole degree blocks (phases 1, 3) or order blocks (phase 2),
// LPT-balanced on the host; the block's operator is the MMA B operand held in
// registers, 32 columns stream through as 4 A m-tiles, so up to 16 independent
// accumulator chains per block and no barrier inside a phase.  p <= 15.
constexpr int kV3Cols = 32;
constexpr int kV3SB = kV3Cols + 4;
__constant__ int c_s1[8][24];  // phase 1/3: degrees per warp, -1 terminated
__constant__ int c_s2[8][24];  // phase 2: orders per warp

__device__ __forceinline__ void v3_rotate(const double* __restrict__ R, int j, const double* Xs, double* Ys) {
  const int lane = threadIdx.x & 31;
  const int d = 2 * j + 1, nnt = (d + 7) >> 3, nks = (d + 3) >> 2, base = j * j;
  const double* Rj = R + rboff(j);
  double bf[4][8];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int n = nt * 8 + (lane >> 2), k = ks * 4 + (lane & 3);
      bf[nt][ks] = (nt < nnt && ks < nks && n < d && k < d) ? __ldg(Rj + n * d + k) : 0.0;
    }
  double acc[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    if (ks >= nks) break;
    const int k = ks * 4 + (lane & 3);
    double a[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) a[mt] = k < d ? Xs[(base + k) * kV3SB + mt * 8 + (lane >> 2)] : 0.0;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      if (nt >= nnt) break;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[nt][ks]);
    }
  }
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    if (nt >= nnt) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = nt * 8 + (lane & 3) * 2 + h;
      if (n >= d) continue;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) Ys[(base + n) * kV3SB + mt * 8 + (lane >> 2)] = acc[mt][nt][h];
    }
  }
}

__device__ __forceinline__ void v3_ztrans(const double* __restrict__ t, int p, int m, const double* Ys, double* Xs) {
  const int lane = threadIdx.x & 31;
  const int d = p + 1 - m, nnt = (d + 7) >> 3, nks = (d + 3) >> 2;
  double bf[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int i = nt * 8 + (lane >> 2), kk = ks * 4 + (lane & 3);
      double v = 0.0;
      if (nt < nnt && ks < nks && i < d && kk < d) v = (i & 1) ? -t[2 * m + i + kk] : t[2 * m + i + kk];
      bf[nt][ks] = v;
    }
  for (int part = 0; part < (m == 0 ? 1 : 2); ++part) {
    double acc[4][2][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      if (ks >= nks) break;
      const int kk = ks * 4 + (lane & 3);
      const double* yrow = Ys + rdof_row(m + kk, m, part) * kV3SB;
      double a[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = kk < d ? yrow[mt * 8 + (lane >> 2)] : 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        if (nt >= nnt) break;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[nt][ks]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      if (nt >= nnt) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = nt * 8 + (lane & 3) * 2 + h;
        if (i >= d) continue;
        double* xrow = Xs + rdof_row(m + i, m, part) * kV3SB;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) xrow[mt * 8 + (lane >> 2)] = acc[mt][nt][h];
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_m2l_rot3(int p, int KR, int KRp, const int4* __restrict__ tiles,
                                                  const int* __restrict__ col_src, const int* __restrict__ col_pos,
                                                  const double* __restrict__ col_scale, const int* __restrict__ rmap,
                                                  const double* __restrict__ M, int kp2,
                                                  const double* __restrict__ rotF, const double* __restrict__ rotB,
                                                  const double* __restrict__ rho_op, size_t rot_stride,
                                                  double* __restrict__ temp) {
  extern __shared__ double sm[];
  double* Xb[2] = {sm, sm + KR * kV3SB};
  double* Ys = sm + 2 * KR * kV3SB;
  __shared__ double s_t[2 * 16 + 2];
  const int4 tile = tiles[blockIdx.x];
  const int op = tile.x, c0 = tile.y, ncol = tile.z;
  const int tid = threadIdx.x, warp = tid >> 5;
  const double* Rf = rotF + size_t(op) * rot_stride;
  const double* Rb = rotB + size_t(op) * rot_stride;
  if (tid <= 2 * p) {
    const double irho = 1.0 / rho_op[op];
    double v = irho;
    for (int k = 1; k <= tid; ++k) v *= k * irho;
    s_t[tid] = v;
  }
  auto gather = [&](double* X, int first) {
    for (int idx = tid; idx < KR * kV3Cols; idx += 256) {
      const int r = idx / kV3Cols, c = idx % kV3Cols;
      if (first + c < ncol)
        cp_async8(X + r * kV3SB + c, M + size_t(col_src[c0 + first + c]) * kp2 + rmap[r]);
      else
        X[r * kV3SB + c] = 0.0;
    }
  };
  gather(Xb[0], 0);
  cp_commit();
  int buf = 0;
  for (int first = 0; first < ncol; first += kV3Cols) {
    if (first + kV3Cols < ncol) {
      gather(Xb[buf ^ 1], first + kV3Cols);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    double* Xs = Xb[buf];
    for (int i = 0; i < 24 && c_s1[warp][i] >= 0; ++i) v3_rotate(Rf, c_s1[warp][i], Xs, Ys);
    __syncthreads();
    for (int i = 0; i < 24 && c_s2[warp][i] >= 0; ++i) v3_ztrans(s_t, p, c_s2[warp][i], Ys, Xs);
    __syncthreads();
    for (int i = 0; i < 24 && c_s1[warp][i] >= 0; ++i) v3_rotate(Rb, c_s1[warp][i], Xs, Ys);
    __syncthreads();
    const int nc = min(kV3Cols, ncol - first);
    for (int idx = tid; idx < nc * KR; idx += 256) {
      const int c = idx / KR, r = idx % KR;
      temp[size_t(col_pos[c0 + first + c]) * KRp + r] = Ys[r * kV3SB + c];  // 1/|b| applied by the reduce
    }
    __syncthreads();
    buf ^= 1;
  }
}

// ---- v4 = v3 with 16-column batches and the rotation blocks staged in shared memory.
// ---- (v3 text follows), C[cols x out] = X^T[cols x in] R^T[in x out].
// A warp owns whole degree blocks (phases 1, 3) or order blocks (phase 2),
// LPT-balanced on the host; the block's operator is the MMA B operand held in
// registers, 32 columns stream through as 4 A m-tiles, so up to 16 independent
// accumulator chains per block and no barrier inside a phase.  p <= 15.
constexpr int kV4Cols = 16;
constexpr int kV4SB = kV4Cols + 4;

__device__ __forceinline__ void v4_rotate(const double* __restrict__ R, int j, const double* Xs, double* Ys) {
  const int lane = threadIdx.x & 31;
  const int d = 2 * j + 1, nnt = (d + 7) >> 3, nks = (d + 3) >> 2, base = j * j;
  const double* Rj = R + rboff(j);
  double bf[4][8];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int n = nt * 8 + (lane >> 2), k = ks * 4 + (lane & 3);
      bf[nt][ks] = (nt < nnt && ks < nks && n < d && k < d) ? Rj[n * d + k] : 0.0;
    }
  double acc[2][4][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    if (ks >= nks) break;
    const int k = ks * 4 + (lane & 3);
    double a[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) a[mt] = k < d ? Xs[(base + k) * kV4SB + mt * 8 + (lane >> 2)] : 0.0;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      if (nt >= nnt) break;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[nt][ks]);
    }
  }
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    if (nt >= nnt) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = nt * 8 + (lane & 3) * 2 + h;
      if (n >= d) continue;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) Ys[(base + n) * kV4SB + mt * 8 + (lane >> 2)] = acc[mt][nt][h];
    }
  }
}

__device__ __forceinline__ void v4_ztrans(const double* __restrict__ t, int p, int m, const double* Ys, double* Xs) {
  const int lane = threadIdx.x & 31;
  const int d = p + 1 - m, nnt = (d + 7) >> 3, nks = (d + 3) >> 2;
  double bf[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int i = nt * 8 + (lane >> 2), kk = ks * 4 + (lane & 3);
      double v = 0.0;
      if (nt < nnt && ks < nks && i < d && kk < d) v = (i & 1) ? -t[2 * m + i + kk] : t[2 * m + i + kk];
      bf[nt][ks] = v;
    }
  for (int part = 0; part < (m == 0 ? 1 : 2); ++part) {
    double acc[2][2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      if (ks >= nks) break;
      const int kk = ks * 4 + (lane & 3);
      const double* yrow = Ys + rdof_row(m + kk, m, part) * kV4SB;
      double a[2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) a[mt] = kk < d ? yrow[mt * 8 + (lane >> 2)] : 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        if (nt >= nnt) break;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[nt][ks]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      if (nt >= nnt) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = nt * 8 + (lane & 3) * 2 + h;
        if (i >= d) continue;
        double* xrow = Xs + rdof_row(m + i, m, part) * kV4SB;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) xrow[mt * 8 + (lane >> 2)] = acc[mt][nt][h];
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_m2l_rot4(int p, int KR, int KRp, const int4* __restrict__ tiles,
                                                  const int* __restrict__ col_src, const int* __restrict__ col_pos,
                                                  const double* __restrict__ col_scale, const int* __restrict__ rmap,
                                                  const double* __restrict__ M, int kp2,
                                                  const double* __restrict__ rotF, const double* __restrict__ rotB,
                                                  const double* __restrict__ rho_op, size_t rot_stride,
                                                  double* __restrict__ temp) {
  extern __shared__ double sm[];
  const int S = int(rot_stride);
  double* Xb[2] = {sm, sm + KR * kV4SB};
  double* Ys = sm + 2 * KR * kV4SB;
  double* Rfs = sm + 3 * KR * kV4SB;
  double* Rbs = Rfs + S;
  __shared__ double s_t[2 * 16 + 2];
  const int4 tile = tiles[blockIdx.x];
  const int op = tile.x, c0 = tile.y, ncol = tile.z;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < S; i += 256) {
    cp_async8(Rfs + i, rotF + size_t(op) * rot_stride + i);
    cp_async8(Rbs + i, rotB + size_t(op) * rot_stride + i);
  }
  const double* Rf = Rfs;
  const double* Rb = Rbs;
  if (tid <= 2 * p) {
    const double irho = 1.0 / rho_op[op];
    double v = irho;
    for (int k = 1; k <= tid; ++k) v *= k * irho;
    s_t[tid] = v;
  }
  auto gather = [&](double* X, int first) {
    for (int idx = tid; idx < KR * kV4Cols; idx += 256) {
      const int r = idx / kV4Cols, c = idx % kV4Cols;
      if (first + c < ncol)
        cp_async8(X + r * kV4SB + c, M + size_t(col_src[c0 + first + c]) * kp2 + rmap[r]);
      else
        X[r * kV4SB + c] = 0.0;
    }
  };
  gather(Xb[0], 0);
  cp_commit();
  int buf = 0;
  for (int first = 0; first < ncol; first += kV4Cols) {
    if (first + kV4Cols < ncol) {
      gather(Xb[buf ^ 1], first + kV4Cols);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    double* Xs = Xb[buf];
    for (int i = 0; i < 24 && c_s1[warp][i] >= 0; ++i) v4_rotate(Rf, c_s1[warp][i], Xs, Ys);
    __syncthreads();
    for (int i = 0; i < 24 && c_s2[warp][i] >= 0; ++i) v4_ztrans(s_t, p, c_s2[warp][i], Ys, Xs);
    __syncthreads();
    for (int i = 0; i < 24 && c_s1[warp][i] >= 0; ++i) v4_rotate(Rb, c_s1[warp][i], Xs, Ys);
    __syncthreads();
    const int nc = min(kV4Cols, ncol - first);
    for (int idx = tid; idx < nc * KR; idx += 256) {
      const int c = idx / KR, r = idx % KR;
      temp[size_t(col_pos[c0 + first + c]) * KRp + r] = Ys[r * kV4SB + c];  // 1/|b| applied by the reduce
    }
    __syncthreads();
    buf ^= 1;
  }
}

// Longest-processing-time assignment of blocks to the 8 warps.
void lpt(int n_items, const std::vector<int>& cost, int (*out)[24]) {
  std::vector<int> order(n_items);
  for (int i = 0; i < n_items; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  int load[8] = {0}, cnt[8] = {0};
  for (int i = 0; i < 8; ++i)
    for (int k = 0; k < 24; ++k) out[i][k] = -1;
  for (int it : order) {
    int w = 0;
    for (int i = 1; i < 8; ++i)
      if (load[i] < load[w]) w = i;
    out[w][cnt[w]++] = it;
    load[w] += cost[it];
  }
}

}  // namespace

bool m2l_rot3_ok(int p) { return p <= 15 && size_t(3) * (p + 1) * (p + 1) * kV3SB * sizeof(double) <= 222 * 1024; }

int launch_m2l_rot3_chunk(const M2LPlan& P, const M2LChunk& C, const DevData& D, cudaStream_t s) {
  if (C.n_tiles == 0) return 0;
  static int sched_p = -1;
  if (sched_p != D.p) {
    const int p = D.p;
    std::vector<int> c1(p + 1), c2(p + 1);
    for (int j = 0; j <= p; ++j) c1[j] = ((2 * j + 8) / 8) * ((2 * j + 4) / 4);
    for (int m = 0; m <= p; ++m) c2[m] = ((p + 8 - m) / 8) * ((p + 4 - m) / 4) * (m == 0 ? 1 : 2);
    int s1[8][24], s2[8][24];
    lpt(p + 1, c1, s1);
    lpt(p + 1, c2, s2);
    cudaMemcpyToSymbol(c_s1, s1, sizeof(s1));
    cudaMemcpyToSymbol(c_s2, s2, sizeof(s2));
    cudaFuncSetAttribute(k_m2l_rot3, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    sched_p = p;
  }
  const size_t smem = size_t(3) * P.KR * kV3SB * sizeof(double);
  k_m2l_rot3<<<C.n_tiles, 256, smem, s>>>(D.p, P.KR, P.KRp, C.tiles, C.col_src, C.col_pos, C.col_scale, P.rmap,
                                           reinterpret_cast<const double*>(D.M), 2 * D.kp, P.rotF, P.rotB, P.rho_op,
                                           P.rot_stride, P.temp);
  return 1;
}

bool m2l_rot4_ok(int p) {
  const size_t KR = size_t(p + 1) * (p + 1);
  return p <= 15 && (3 * KR * kV4SB + 2 * rot_blocks_size_dev(p)) * sizeof(double) <= 222 * 1024;
}

int launch_m2l_rot4_chunk(const M2LPlan& P, const M2LChunk& C, const DevData& D, cudaStream_t s) {
  if (C.n_tiles == 0) return 0;
  static int sched_p = -1;
  if (sched_p != D.p) {
    const int p = D.p;
    std::vector<int> c1(p + 1), c2(p + 1);
    for (int j = 0; j <= p; ++j) c1[j] = ((2 * j + 8) / 8) * ((2 * j + 4) / 4);
    for (int m = 0; m <= p; ++m) c2[m] = ((p + 8 - m) / 8) * ((p + 4 - m) / 4) * (m == 0 ? 1 : 2);
    int s1[8][24], s2[8][24];
    lpt(p + 1, c1, s1);
    lpt(p + 1, c2, s2);
    cudaMemcpyToSymbol(c_s1, s1, sizeof(s1));
    cudaMemcpyToSymbol(c_s2, s2, sizeof(s2));
    cudaFuncSetAttribute(k_m2l_rot4, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    sched_p = p;
  }
  const size_t smem = (size_t(3) * P.KR * kV4SB + 2 * P.rot_stride) * sizeof(double);
  k_m2l_rot4<<<C.n_tiles, 256, smem, s>>>(D.p, P.KR, P.KRp, C.tiles, C.col_src, C.col_pos, C.col_scale, P.rmap,
                                           reinterpret_cast<const double*>(D.M), 2 * D.kp, P.rotF, P.rotB, P.rho_op,
                                           P.rot_stride, P.temp);
  return 1;
}

size_t m2l_rot_smem(int p, int bn) {
  const size_t KR = size_t(p + 1) * (p + 1);
  return (2 * (size_t(p + 1) * (2 * p + 1) * (2 * p + 3) / 3) + 3 * KR * (bn + 4)) * sizeof(double);
}

int launch_m2l_rot2_chunk(const M2LPlan& P, const M2LChunk& C, const DevData& D, cudaStream_t s) {
  if (C.n_tiles == 0) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_rot2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    cudaFuncSetAttribute(k_m2l_rot2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    attr = true;
  }
  const size_t smem = m2l_rot_smem(D.p, P.bn);
  if (P.bn == 8)
    k_m2l_rot2<8><<<C.n_tiles, 256, smem, s>>>(D.p, P.KR, P.KRp, C.tiles, C.col_src, C.col_pos, C.col_scale, P.rmap,
                                              reinterpret_cast<const double*>(D.M), 2 * D.kp, P.rotF, P.rotB,
                                              P.rho_op, P.rot_stride, P.temp);
  else
    k_m2l_rot2<16><<<C.n_tiles, 256, smem, s>>>(D.p, P.KR, P.KRp, C.tiles, C.col_src, C.col_pos, C.col_scale,
                                               P.rmap, reinterpret_cast<const double*>(D.M), 2 * D.kp, P.rotF,
                                               P.rotB, P.rho_op, P.rot_stride, P.temp);
  return 1;
}

size_t m2l_rot_smem_v1(int p, int bn) { return size_t(2) * (p + 1) * (p + 1) * (bn + 4) * sizeof(double); }

int launch_m2l_rot_chunk(const M2LPlan& P, const M2LChunk& C, const DevData& D, cudaStream_t s) {
  int k = 0;
  const int kp2 = 2 * D.kp;
  const int p = D.p;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_rot<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_m2l_rot<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const size_t smem = m2l_rot_smem_v1(p, P.bn);
  {
    if (C.n_tiles == 0) return 0;
    if (P.bn == 16)
      k_m2l_rot<16><<<C.n_tiles, 256, smem, s>>>(p, P.KR, P.KRp, C.tiles, C.col_src, C.col_pos, C.col_scale, P.rmap,
                                                  reinterpret_cast<const double*>(D.M), kp2, P.rotF, P.rotB, P.rho_op,
                                                  P.rot_stride, P.temp);
    else
      k_m2l_rot<32><<<C.n_tiles, 256, smem, s>>>(p, P.KR, P.KRp, C.tiles, C.col_src, C.col_pos, C.col_scale, P.rmap,
                                                  reinterpret_cast<const double*>(D.M), kp2, P.rotF, P.rotB, P.rho_op,
                                                  P.rot_stride, P.temp);
    k += 1;
  }
  return k;
}

}  // namespace dev
}  // namespace qbxg
