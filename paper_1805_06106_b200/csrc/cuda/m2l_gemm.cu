// Tree shifts (Stage 2 M2M, Stage 7 L2L) as dense
// contractions on the fp64 tensor pipe (DMMA, mma.sync m8n8k4 f64).  (The Stage 4
// M2L lives in m2l_pas.cu.)
//
// For real densities M_j^{-k} = (-1)^k conj(M_j^k) and M_j^0, L_n^0 are real, so a
// shift acts on (p+1)^2 real degrees of freedom ("real DOF": per degree n, Re X_n^0,
// then Re/Im X_n^m for m = 1..n) as a real (p+1)^2 x (p+1)^2 matrix.  With
// box-scaled coefficients there are only 8 such matrices per direction (one per
// octant); one tree level is a GEMM per octant
//   C[KR x n_pairs] = T_octant[KR x KR] * B[KR x n_pairs]
// whose columns gather the shifted boxes' expansions; the results go to staging
// rows and a second kernel sums each receiving box's rows in a fixed order, so the
// result is bitwise reproducible and needs no atomics.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "qbxg.h"
#include "harmonics.cuh"
#include "kernels.cuh"

namespace qbxg {
namespace dev {

namespace {

constexpr int kKC = 16;          // K chunk per pipeline stage
constexpr int kAPad = kKC + 4;   // A smem row stride (doubles): conflict-free fragment reads
// columns (pairs) per CTA tile: BN = 64 (1 CTA/SM) or 32 (2 CTAs/SM); B smem row stride BN + 4

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__global__ void __launch_bounds__(256) k_shift_ops(int mode, int p, int KR, int KRp, const int4* __restrict__ rdof,
                                                   double* __restrict__ ops) {
  extern __shared__ double2 sR[];  // hsize(p)
  const int o = blockIdx.x;        // octant
  const double a = mode == 1 ? 1.0 : 0.5;
  const double ux = (o & 1) ? a : -a, uy = (o & 2) ? a : -a, uz = (o & 4) ? a : -a;
  if (threadIdx.x <= p) {
    double2 col[kMaxOrder + 1];
    regular_column(ux, uy, uz, threadIdx.x, p, col);
    for (int n = threadIdx.x; n <= p; ++n) sR[hidx(n, threadIdx.x)] = col[n - threadIdx.x];
  }
  __syncthreads();
  double* T = ops + size_t(o) * KRp * KRp;
  for (int idx = threadIdx.x; idx < KRp * KRp; idx += blockDim.x) {
    const int ro = idx / KRp, ri = idx % KRp;
    double v = 0.0;
    if (ro < KR && ri < KR) {
      const int4 ao = rdof[ro], bi = rdof[ri];
      const int n = ao.x, m = ao.y, po = ao.z, j = bi.x, k = bi.y, pi = bi.z;
      const double s = ldexp(1.0, -n);
      double2 A = make_double2(0, 0), B = make_double2(0, 0);
      auto R = [&](int nn, int mm) {
        if (nn < 0 || nn > p || mm > nn || mm < -nn) return make_double2(0.0, 0.0);
        return hget(sR, nn, mm);
      };
      if (mode == 1) {
        A = R(n - j, m - k);
        A.y = -A.y;
        if (k > 0) {
          B = R(n - j, m + k);
          B.y = -B.y;
          if (k & 1) B = make_double2(-B.x, -B.y);
        }
      } else {
        A = R(j - n, k - m);
        if (k > 0) {
          B = R(j - n, -k - m);
          if (k & 1) B = make_double2(-B.x, -B.y);
        }
      }
      if (po == 0)
        v = (pi == 0) ? (A.x + B.x) : -(A.y - B.y);
      else
        v = (pi == 0) ? (A.y + B.y) : (A.x - B.x);
      v *= s;
    }
    T[idx] = v;
  }
}

// out[b] (+)= sum of staged rows seg[i] = [first, last) for box boxes[i].
__global__ void __launch_bounds__(256) k_seg_reduce(const int* __restrict__ boxes, const int2* __restrict__ seg,
                                                    int KR, int KRp, const int* __restrict__ rmap,
                                                    const double* __restrict__ temp, double* __restrict__ out,
                                                    int kp2, int accumulate) {
  const int b = boxes[blockIdx.x];
  const int2 sg = seg[blockIdx.x];
  for (int r = threadIdx.x; r < KR; r += blockDim.x) {
    double s = 0.0;
    for (int pos = sg.x; pos < sg.y; ++pos) s += temp[size_t(pos) * KRp + r];
    double* dst = out + size_t(b) * kp2 + rmap[r];
    *dst = accumulate ? *dst + s : s;
  }
}

// One CTA: one offset, up to BN pairs; 8 warps x (8*MT rows); full K.
template <int MT, int BN>
__global__ void __launch_bounds__(256, BN == 32 ? 2 : 1) k_m2l_gemm(const double* __restrict__ ops, const int4* __restrict__ tiles,
                                                  const int* __restrict__ col_src, const int* __restrict__ col_pos,
                                                  const double* __restrict__ col_scale,
                                                  const int* __restrict__ rmap, const double* __restrict__ M,
                                                  int kp2, double* __restrict__ temp) {
  constexpr int KRp = 64 * MT;
  constexpr int kBN = BN, kBPad = BN + 4, NT = BN / 8;
  extern __shared__ double smem[];
  double* As = smem;                              // 2 x KRp x kAPad
  double* Bs = smem + 2 * KRp * kAPad;            // 2 x kKC x kBPad
  __shared__ int s_src[kBN];
  __shared__ int s_map[KRp];
  const int4 tile = tiles[blockIdx.x];  // (op index, first column, count, -)
  const double* T = ops + size_t(tile.x) * KRp * KRp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kBN) s_src[tid] = tid < tile.z ? col_src[tile.y + tid] : -1;
  for (int i = tid; i < KRp; i += 256) s_map[i] = rmap[i];
  __syncthreads();

  auto load_stage = [&](int buf, int k0) {
    double* A = As + buf * KRp * kAPad;
    // A: KRp rows x kKC doubles = KRp x 8 16-byte copies
    for (int i = tid; i < KRp * (kKC / 2); i += 256) {
      const int r = i / (kKC / 2), c = (i % (kKC / 2)) * 2;
      cp_async16(A + r * kAPad + c, T + size_t(r) * KRp + k0 + c);
    }
    double* B = Bs + buf * kKC * kBPad;
    for (int i = tid; i < kKC * kBN; i += 256) {
      const int kk = i / kBN, c = i % kBN;
      const int src = s_src[c];
      const int mo = s_map[k0 + kk];
      if (src >= 0 && mo >= 0)
        cp_async8(B + kk * kBPad + c, M + size_t(src) * kp2 + mo);
      else
        B[kk * kBPad + c] = 0.0;
    }
    cp_async_commit();
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = KRp / kKC;
  load_stage(0, 0);
  const int row_w = warp * 8 * MT;
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      load_stage((kc + 1) & 1, (kc + 1) * kKC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* A = As + (kc & 1) * KRp * kAPad;
    const double* B = Bs + (kc & 1) * kKC * kBPad;
#pragma unroll
    for (int kk = 0; kk < kKC; kk += 4) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = A[(row_w + i * 8 + (lane >> 2)) * kAPad + kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = B[(kk + (lane & 3)) * kBPad + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  // epilogue: temp[pos][row] = scale * acc
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = j * 8 + (lane & 3) * 2 + h;
      if (c >= tile.z) continue;
      const int pos = col_pos[tile.y + c];
      // no fp64 arithmetic here: it would queue behind the co-resident CTA's DMMAs
      // (shared pipe); the 1/|b| scale is applied once per target box in the reduce
      double* out = temp + size_t(pos) * KRp;
#pragma unroll
      for (int i = 0; i < MT; ++i) out[row_w + i * 8 + (lane >> 2)] = acc[i][j][h];
    }
  }
}

// DMMA throughput microbenchmark: 16 independent m8n8k4 accumulators per warp.
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
  double acc[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int MT>
void gemm_mt(const double* ops, int n_tiles, const int4* tiles, const int* col_src, const int* col_pos,
             const double* col_scale, const int* rmap, const double* X, int kp2, double* temp, cudaStream_t s,
             int bn) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_gemm<MT, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_m2l_gemm<MT, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const size_t smem = (2 * 64 * MT * kAPad + 2 * kKC * (bn + 4)) * sizeof(double);
  if (bn == 32)
    k_m2l_gemm<MT, 32><<<n_tiles, 256, smem, s>>>(ops, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp);
  else
    k_m2l_gemm<MT, 64><<<n_tiles, 256, smem, s>>>(ops, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp);
}

int gemm_any(int KRp, const double* ops, int n_tiles, const int4* tiles, const int* col_src, const int* col_pos,
             const double* col_scale, const int* rmap, const double* X, int kp2, double* temp, cudaStream_t s,
             int bn = 64) {
  switch (KRp / 64) {
    case 1: gemm_mt<1>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 2: gemm_mt<2>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 3: gemm_mt<3>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 4: gemm_mt<4>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 5: gemm_mt<5>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 6: gemm_mt<6>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 7: gemm_mt<7>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    case 8: gemm_mt<8>(ops, n_tiles, tiles, col_src, col_pos, col_scale, rmap, X, kp2, temp, s, bn); break;
    default: return -1;
  }
  return 1;
}

}  // namespace

int launch_shift_ops(int mode, int p, int KR, int KRp, const int4* rdof, double* ops, cudaStream_t s) {
  upload_inv_nm();  // k_shift_ops uses regular_column (this TU's constant table)
  cudaFuncSetAttribute(k_shift_ops, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_shift_ops<<<8, 256, hsize(p) * sizeof(double2), s>>>(mode, p, KR, KRp, rdof, ops);
  return 1;
}

// One tree level of M2M (src = M, out = M, overwrite) or L2L (src = L, out = L, accumulate).
int launch_shift_level(const M2LPlan& P, const ShiftLevel& S, const double* ops, double2* X, int kp, bool accumulate,
                       cudaStream_t s) {
  if (S.n_tiles == 0) return 0;
  double* Xd = reinterpret_cast<double*>(X);
  if (gemm_any(P.KRp, ops, S.n_tiles, S.tiles, S.col_src, S.col_pos, S.col_scale, P.rmap, Xd, 2 * kp, P.temp, s) < 0)
    return -1;
  k_seg_reduce<<<S.n_out, 256, 0, s>>>(S.out_boxes, S.out_seg, P.KR, P.KRp, P.rmap, P.temp, Xd, 2 * kp,
                                        accumulate ? 1 : 0);
  return 2;
}

}  // namespace dev
}  // namespace qbxg

extern "C" int qbxg_measure_dmma_peak(int32_t device, double* out_tflops) {
  cudaSetDevice(device);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return QBXG_ERR_CUDA;
  const int iters = 2048, blocks = nsm * 4, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    qbxg::dev::k_dmma_peak<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double flops = 2.0 * 256 * 16 * double(iters) * (blocks * threads / 32);
  *out_tflops = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? QBXG_OK : QBXG_ERR_CUDA;
}
