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
    temp[size_t(col_pos[c0 + c]) * KRp + r] = col_scale[c0 + c] * Ys[r * SB + c];
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
      temp[size_t(col_pos[c0 + first + c]) * KRp + r] = col_scale[c0 + first + c] * Ys[r * SB + c];
    }
    __syncthreads();
    buf ^= 1;
  }
}

}  // namespace

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
