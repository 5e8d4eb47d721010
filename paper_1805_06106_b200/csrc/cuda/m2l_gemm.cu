// Stage 4 (M2L over List 2) as one dense contraction per
// relative box offset, on the fp64 tensor pipe (DMMA, mma.sync m8n8k4 f64).
//
// With box-scaled coefficients the M2L operator depends only on the offset
// delta = (c_b - c_d) / (2|b|) in [-5,5]^3 (11^3 - 5^3 = 1,206 used offsets,
// PAPER.md:3622-3626), up to a 1/|b| factor:
//   L~_b(n,m) += (1/|b|) (-1)^{n+m} sum_{j,k} M~_d(j,k) I_{j+n}^{k-m}(2 delta).
// For real densities M_j^{-k} = (-1)^k conj(M_j^k) and M_j^0, L_n^0 are real,
// so the map acts on (p+1)^2 real degrees of freedom ("real DOF": per degree n,
// Re L_n^0, then Re/Im L_n^m for m = 1..n) as a real (p+1)^2 x (p+1)^2 matrix
// T_delta (256 x 256 at p = 15).  Per offset that is a GEMM
//   C[KR x n_pairs] = T_delta[KR x KR] * B[KR x n_pairs]
// whose columns gather the source boxes' multipoles.  Columns of one offset
// hit distinct target boxes; results go to a per-entry staging buffer in List-2
// CSR order and a second kernel sums each target box's row in that order, so
// the result is bitwise reproducible and needs no atomics.
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

// Build T_delta for each used offset: rows/cols in real-DOF order, KRp x KRp
// row-major, zero padded.  rdof[r] = (n, m, part).
__global__ void __launch_bounds__(256) k_m2l_ops(int p, int KR, int KRp, const int* __restrict__ used_slot,
                                                 const int4* __restrict__ rdof, double* __restrict__ ops) {
  extern __shared__ double2 sI[];  // hsize(2p)
  const int o = blockIdx.x;
  const int slot = used_slot[o];
  const int dx = slot / 121 - 5, dy = (slot / 11) % 11 - 5, dz = slot % 11 - 5;
  const int P2 = 2 * p;
  if (threadIdx.x <= P2) {
    double2 col[kMaxOrder + 1];
    irregular_column(2.0 * dx, 2.0 * dy, 2.0 * dz, threadIdx.x, P2, col);
    for (int n = threadIdx.x; n <= P2; ++n) sI[hidx(n, threadIdx.x)] = col[n - threadIdx.x];
  }
  __syncthreads();
  double* T = ops + size_t(o) * KRp * KRp;
  for (int idx = threadIdx.x; idx < KRp * KRp; idx += blockDim.x) {
    const int ro = idx / KRp, ri = idx % KRp;
    double v = 0.0;
    if (ro < KR && ri < KR) {
      const int4 a = rdof[ro], b = rdof[ri];
      const int n = a.x, m = a.y, po = a.z, j = b.x, k = b.y, pi = b.z;
      const double s = ((n + m) & 1) ? -1.0 : 1.0;
      const double2 A = hget(sI, j + n, k - m);
      double2 B = make_double2(0, 0);
      if (k > 0) {
        B = hget(sI, j + n, -k - m);
        if (k & 1) B = make_double2(-B.x, -B.y);
      }
      // L = A M + B conj(M), M = x + i y:  Re: Re(A+B) x - Im(A-B) y;  Im: Im(A+B) x + Re(A-B) y
      if (po == 0)
        v = (pi == 0) ? (A.x + B.x) : -(A.y - B.y);
      else
        v = (pi == 0) ? (A.y + B.y) : (A.x - B.x);
      v *= s;
    }
    T[idx] = v;
  }
}

// Octant operators for the tree shifts in the same real-DOF form:
//   mode 1, M2M (child -> parent), u = (c_child - c_parent)/|child| in {+-1}^3:
//     M~_par(n,m) = 2^-n sum_{j<=n,k} M~_ch(j,k) conj(R_{n-j}^{m-k}(u))
//   mode 2, L2L (parent -> child), u = (c_child - c_parent)/|parent| in {+-1/2}^3:
//     L~_ch(n,m) = 2^-n sum_{j>=n,k} L~_par(j,k) R_{j-n}^{k-m}(u)
// Written as L = A X + B conj(X) per (output, input) pair, like k_m2l_ops.
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

// ---- azimuthally split M2L ------------------------------------------------
// Rotating the frame about z by alpha = atan2(dy, dx) puts the offset in the
// xz-plane, where I_N^K(v') is real.  With M' = M e^{i k alpha} and
// L = L' e^{-i m alpha} (both diagonal per coefficient) the M2L operator is then
// block diagonal in (Re, Im):
//   Re L'(n,m) = sum_{j,k>=0} s [I_{j+n}^{k-m} + (k>0)(-1)^k I_{j+n}^{-k-m}] Re M'(j,k)
//   Im L'(n,m) = sum_{j,k>=1} s [I_{j+n}^{k-m} -       (-1)^k I_{j+n}^{-k-m}] Im M'(j,k)
// with s = (-1)^{n+m}: two hsize(p) x hsize(p) real blocks (2 x 144^2 padded at
// p = 15) instead of one (p+1)^2 x (p+1)^2 block (256^2) -- 0.63x the DMMA work.
// Re block: rows and columns in half-table order q = hidx(n, m), padded to NH
// (multiple of 48).  Im block: rows in compacted order t = n(n-1)/2 + m - 1 over
// m >= 1 only (its m = 0 rows vanish), padded to NHI; columns in q order like
// the Re block, so one gathered multipole column feeds both blocks.
__device__ __forceinline__ void q_nm(int q, int& n, int& m) {
  n = int((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
  while (hidx(n + 1, 0) <= q) ++n;
  while (hidx(n, 0) > q) --n;
  m = q - hidx(n, 0);
}

__device__ __forceinline__ void t_nm(int t, int& n, int& m) {
  n = int((1.0f + sqrtf(1.0f + 8.0f * t)) * 0.5f);
  while (n * (n - 1) / 2 > t) --n;
  while ((n + 1) * n / 2 <= t) ++n;
  m = t - n * (n - 1) / 2 + 1;
}

__global__ void __launch_bounds__(256) k_m2l_ops_split(int p, int NH, int NHI, const int* __restrict__ used_slot,
                                                       double* __restrict__ ops, double2* __restrict__ cs) {
  extern __shared__ double2 sI[];  // hsize(2p)
  const int o = blockIdx.x;
  const int slot = used_slot[o];
  const int dx = slot / 121 - 5, dy = (slot / 11) % 11 - 5, dz = slot % 11 - 5;
  const int P2 = 2 * p, NR = hsize(p);
  const double rho = sqrt(double(dx * dx + dy * dy));
  const double alpha = (dx == 0 && dy == 0) ? 0.0 : atan2(double(dy), double(dx));
  if (threadIdx.x <= P2) {
    double2 col[kMaxOrder + 1];
    irregular_column(2.0 * rho, 0.0, 2.0 * dz, threadIdx.x, P2, col);
    for (int n = threadIdx.x; n <= P2; ++n) sI[hidx(n, threadIdx.x)] = col[n - threadIdx.x];
  }
  if (threadIdx.x <= p) {
    double sn, cn;
    sincos(threadIdx.x * alpha, &sn, &cn);
    cs[size_t(o) * (p + 1) + threadIdx.x] = make_double2(cn, sn);
  }
  __syncthreads();
  if (ops == nullptr) return;  // point-and-shoot needs only the (cos, sin) table
  double* T = ops + size_t(o) * (NH + NHI) * NH;
  for (int idx = threadIdx.x; idx < (NH + NHI) * NH; idx += blockDim.x) {
    const int ro = idx / NH, qi = idx % NH;
    const bool im = ro >= NH;
    const int qo = im ? ro - NH : ro;
    double v = 0.0;
    if (qo < (im ? NR - (p + 1) : NR) && qi < NR) {
      int n, m, j, k;
      if (im)
        t_nm(qo, n, m);
      else
        q_nm(qo, n, m);
      q_nm(qi, j, k);
      const double sg = ((n + m) & 1) ? -1.0 : 1.0;
      const double a = hget(sI, j + n, k - m).x;
      const double b = k > 0 ? ((k & 1) ? -1.0 : 1.0) * hget(sI, j + n, -k - m).x : 0.0;
      if (!im)
        v = sg * (a + b);
      else if (m > 0 && k > 0)
        v = sg * (a - b);
    }
    T[idx] = v;
  }
}

// One CTA: one offset, up to BN pairs; NW warps: the first half on the Re
// block, the second half on the Im block, NH/(NW/2) rows each; K chunks of 16
// double-buffered (operator rows by cp.async, rotated multipole columns
// through registers one chunk ahead).  NW = 6, BN = 32 at p = 15 gives 110 KB of
// shared memory and 2 CTAs per SM.
template <int NH, int NW, int BN, int KC>
__global__ void __launch_bounds__(2 * NW * 32, NH <= 144 ? 2 : 1) k_m2l_split(int NHI,
    const double* __restrict__ ops, const double2* __restrict__ cs_all, int p, const int4* __restrict__ tiles,
    const int* __restrict__ col_src, const int* __restrict__ col_pos, const double* __restrict__ col_scale,
    const double* __restrict__ M, int kp2, int KRp, double* __restrict__ temp) {
  // NW = warps on the Re block (NH rows); NHI / (8 MT) more warps on the Im block
  constexpr int MT = NH / (NW * 8);
  static_assert(MT * 8 * NW == NH, "Re rows must split evenly over the warps");
  constexpr int kBPad = BN + 4, NT = BN / 8;
  constexpr int kAP = KC + 4;                   // A row stride: conflict-free fragment reads
  constexpr int kLd = (KC * BN + 255) / 256;    // B elements per thread per chunk (>= 256 threads)
  const int NTH = blockDim.x, RA = NH + NHI;    // threads, operator rows
  extern __shared__ double smem[];
  double* As = smem;                          // 2 x RA x kAP
  double* Bs = smem + 2 * RA * kAP;           // 2 buffers x 2 halves x KC x kBPad
  __shared__ int s_src[BN];
  __shared__ double2 s_cs[kMaxOrder + 1];
  __shared__ unsigned char s_n[NH], s_m[NH];
  const int4 tile = tiles[blockIdx.x];  // (op index, first column, count, -)
  const double* T = ops + size_t(tile.x) * RA * NH;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NR = hsize(p), NI = NR - (p + 1);
  if (tid < BN) s_src[tid] = tid < tile.z ? col_src[tile.y + tid] : -1;
  if (tid <= p) s_cs[tid] = cs_all[size_t(tile.x) * (p + 1) + tid];
  for (int q = tid; q < NH; q += NTH) {
    int n = 0, m = 0;
    if (q < NR) q_nm(q, n, m);
    s_n[q] = (unsigned char)n;
    s_m[q] = (unsigned char)m;
  }
  __syncthreads();

  auto load_a = [&](int buf, int k0) {
    double* A = As + buf * RA * kAP;
    for (int i = tid; i < RA * (KC / 2); i += NTH) {
      const int r = i / (KC / 2), c = (i % (KC / 2)) * 2;
      cp_async16(A + r * kAP + c, T + size_t(r) * NH + k0 + c);
    }
    cp_async_commit();
  };
  double bx[kLd], by[kLd];
  auto fetch_b = [&](int k0) {
#pragma unroll
    for (int it = 0; it < kLd; ++it) {
      const int e = tid + it * NTH;
      bx[it] = by[it] = 0.0;
      if (e < KC * BN) {
        const int kk = e / BN, c = e % BN, q = k0 + kk, src = s_src[c];
        if (src >= 0 && q < NR) {
          const double2 v = *reinterpret_cast<const double2*>(M + size_t(src) * kp2 + 2 * q);
          bx[it] = v.x;
          by[it] = v.y;
        }
      }
    }
  };
  auto store_b = [&](int buf, int k0) {
    double* Br = Bs + buf * 2 * KC * kBPad;
    double* Bi = Br + KC * kBPad;
#pragma unroll
    for (int it = 0; it < kLd; ++it) {
      const int e = tid + it * NTH;
      if (e < KC * BN) {
        const int kk = e / BN, c = e % BN;
        const double2 r = s_cs[s_m[k0 + kk]];
        Br[kk * kBPad + c] = bx[it] * r.x - by[it] * r.y;  // M' = M e^{i k alpha}
        Bi[kk * kBPad + c] = bx[it] * r.y + by[it] * r.x;
      }
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = NH / KC;
  const bool imw = warp >= NW;
  const int row_w = warp * 8 * MT;  // Re rows [0, NH), Im rows [NH, NH + NHI)
  load_a(0, 0);
  fetch_b(0);
  store_b(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int cur = kc & 1;
    if (kc + 1 < nk) {
      load_a(cur ^ 1, (kc + 1) * KC);
      fetch_b((kc + 1) * KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* A = As + cur * RA * kAP;
    const double* B = Bs + cur * 2 * KC * kBPad + (imw ? KC * kBPad : 0);
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = A[(row_w + i * 8 + (lane >> 2)) * kAP + kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = B[(kk + (lane & 3)) * kBPad + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (kc + 1 < nk) store_b(cur ^ 1, (kc + 1) * KC);
    __syncthreads();
  }
  // epilogue: raw L' rows (rotated frame, unscaled) straight from registers into
  // the staging row (Re rows q at [q], Im rows t at [NR + t]: (p+1)^2 doubles),
  // 8 consecutive doubles per lane group.  No fp64 arithmetic here: it would queue
  // behind the co-resident CTA's DMMAs on the shared fp64 pipe.  The back
  // rotation and the 1/|b| scale are applied per entry in k_m2l_reduce_split.
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = j * 8 + (lane & 3) * 2 + h;
      if (c >= tile.z) continue;
      double* out = temp + size_t(col_pos[tile.y + c]) * KRp;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = row_w + i * 8 + (lane >> 2);
        if (!imw) {
          if (r < NR) out[r] = acc[i][j][h];
        } else if (r - NH < NI) {
          out[NR + r - NH] = acc[i][j][h];
        }
      }
    }
  }
}

constexpr int kSplitBN = 32;  // columns per split-M2L tile (40 measured slower: 72 vs 58 ms)

// Barrier-free variant: the whole rotated multipole tile (Re and Im halves,
// NH rows x BN columns) is gathered, rotated and stored in shared memory once per
// tile -- the only fp64 CUDA-core work, done while the co-resident CTA keeps the
// tensor pipe busy -- and every warp then streams its own operator rows from L2
// straight into registers (each operator element has exactly one consumer warp,
// so shared memory buys nothing), two k-steps ahead, with no barrier in the K loop.
template <int NH, int NW, int BN>
__global__ void __launch_bounds__(2 * NW * 32, NH <= 144 ? 2 : 1) k_m2l_split2(int NHI,
    const double* __restrict__ ops, const double2* __restrict__ cs_all, int p, const int4* __restrict__ tiles,
    const int* __restrict__ col_src, const int* __restrict__ col_pos, const double* __restrict__ M, int kp2,
    int KRp, double* __restrict__ temp) {
  constexpr int MT = NH / (NW * 8);
  static_assert(MT * 8 * NW == NH, "Re rows must split evenly over the warps");
  constexpr int kBPad = BN + 4, NT = BN / 8;
  constexpr int kSt = 8;  // staging gathers per thread per round (16 measured slower: register cap)
  const int NTH = blockDim.x, RA = NH + NHI;
  extern __shared__ double smem[];
  double* Br = smem;              // NH x kBPad: Re M'
  double* Bi = smem + NH * kBPad;  // NH x kBPad: Im M'
  __shared__ int s_src[BN];
  __shared__ double2 s_cs[kMaxOrder + 1];
  __shared__ unsigned char s_m[NH];
  const int4 tile = tiles[blockIdx.x];
  const double* T = ops + size_t(tile.x) * RA * NH;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NR = hsize(p), NI = NR - (p + 1);
  if (tid < BN) s_src[tid] = tid < tile.z ? col_src[tile.y + tid] : -1;
  if (tid <= p) s_cs[tid] = cs_all[size_t(tile.x) * (p + 1) + tid];
  for (int q = tid; q < NH; q += NTH) {
    int n = int((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
    while (hidx(n + 1, 0) <= q) ++n;
    while (hidx(n, 0) > q) --n;
    s_m[q] = (unsigned char)(q < NR ? q - hidx(n, 0) : 0);
  }
  __syncthreads();
  const bool imw = warp >= NW;
  const int row_w = warp * 8 * MT;
  const double* B = imw ? Bi : Br;
  const double* Arow = T + size_t(row_w + (lane >> 2)) * NH + (lane & 3);
  const int nks = (NR + 3) / 4;  // k-steps over nonzero K rows
  // first two operator k-steps in flight while the tile is staged
  double a0[MT], a1[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    a0[i] = __ldg(Arow + size_t(i * 8) * NH);
    a1[i] = nks > 1 ? __ldg(Arow + size_t(i * 8) * NH + 4) : 0.0;
  }
  // stage M' = M e^{i k alpha}: consecutive threads walk one column's contiguous
  // half table; kSt gathers in flight per thread before any is used
  for (int base = 0; base < NH * BN; base += kSt * NTH) {
    double2 v[kSt];
#pragma unroll
    for (int u = 0; u < kSt; ++u) {
      const int e = base + tid + u * NTH;
      const int c = e / NH, q = e - c * NH;
      v[u] = make_double2(0.0, 0.0);
      if (e < NH * BN && q < NR) {
        const int src = s_src[c];
        if (src >= 0) v[u] = *reinterpret_cast<const double2*>(M + size_t(src) * kp2 + 2 * q);
      }
    }
#pragma unroll
    for (int u = 0; u < kSt; ++u) {
      const int e = base + tid + u * NTH;
      if (e < NH * BN) {
        const int c = e / NH, q = e - c * NH;
        const double2 r = s_cs[s_m[q]];
        Br[q * kBPad + c] = v[u].x * r.x - v[u].y * r.y;
        Bi[q * kBPad + c] = v[u].x * r.y + v[u].y * r.x;
      }
    }
  }
  __syncthreads();

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int ks = 0; ks < nks; ++ks) {
    double an[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) an[i] = ks + 2 < nks ? __ldg(Arow + size_t(i * 8) * NH + 4 * (ks + 2)) : 0.0;
    double b[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) b[j] = B[(4 * ks + (lane & 3)) * kBPad + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a0[i], b[j]);
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      a0[i] = a1[i];
      a1[i] = an[i];
    }
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = j * 8 + (lane & 3) * 2 + h;
      if (c >= tile.z) continue;
      double* out = temp + size_t(col_pos[tile.y + c]) * KRp;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = row_w + i * 8 + (lane >> 2);
        if (!imw) {
          if (r < NR) out[r] = acc[i][j][h];
        } else if (r - NH < NI) {
          out[NR + r - NH] = acc[i][j][h];
        }
      }
    }
  }
}

template <int NH, int NW, int BN>
void split2_launch(const M2LPlan& P, const M2LChunk& C, const double* X, int kp2, int p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_split2<NH, NW, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const int NHI = split_nhi(p, NH);
  const int threads = (NH + NHI) / (NH / NW) * 32;
  const size_t smem = size_t(2 * NH * (BN + 4)) * sizeof(double);
  k_m2l_split2<NH, NW, BN><<<C.n_tiles, threads, smem, s>>>(NHI, P.sops, P.cs, p, C.tiles, C.col_src, C.col_pos,
                                                            X, kp2, P.KRp, P.temp);
}

template <int NH, int NW, int BN, int KC>
void split_launch(const M2LPlan& P, const M2LChunk& C, const double* X, int kp2, int p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_split<NH, NW, BN, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const int NHI = split_nhi(p, NH);
  const int threads = (NH + NHI) / (NH / NW) * 32;
  const size_t smem = size_t(2 * (NH + NHI) * (KC + 4) + 2 * 2 * KC * (BN + 4)) * sizeof(double);
  k_m2l_split<NH, NW, BN, KC><<<C.n_tiles, threads, smem, s>>>(NHI, P.sops, P.cs, p, C.tiles, C.col_src,
                                                               C.col_pos, C.col_scale, X, kp2, P.KRp, P.temp);
}


template <int NH>
void split_nh_launch(const M2LPlan& P, const M2LChunk& C, const double* X, int kp2, int p, cudaStream_t s) {
  static const bool v1 = std::getenv("QBXG_SPLIT_V1") != nullptr;
  if (v1)
    split_launch<NH, 6, 32, 16>(P, C, X, kp2, p, s);  // 6 Re warps + Im warps; 2 CTAs/SM up to NH = 144
  else
    split2_launch<NH, 6, kSplitBN>(P, C, X, kp2, p, s);
}

// Sum each target box's staged rows in List-2 CSR order and add to L~_b.
__global__ void __launch_bounds__(256) k_m2l_reduce(const int* __restrict__ boxes, const int64_t* __restrict__ v_starts,
                                                    int64_t chunk_base, int KR, int KRp,
                                                    const int* __restrict__ rmap, const double* __restrict__ temp,
                                                    const double4* __restrict__ box, double* __restrict__ L,
                                                    int kp2) {
  const int b = boxes[blockIdx.x];
  const int64_t a = v_starts[b] - chunk_base, e = v_starts[b + 1] - chunk_base;
  const double ih = 1.0 / box[b].w;
  for (int r = threadIdx.x; r < KR; r += blockDim.x) {
    double s = 0.0;
    for (int64_t pos = a; pos < e; ++pos) s += temp[pos * KRp + r];
    L[size_t(b) * kp2 + rmap[r]] += s * ih;
  }
}

// Split-M2L reduce: each staging row holds L' of one List-2 entry in its offset's
// rotated frame (Re block rows 0..NH-1, Im block rows NH..).  Rotate back
// (L = L' e^{-i m alpha}) and sum in CSR order; scale by 1/|b| once.
__global__ void __launch_bounds__(160) k_m2l_reduce_split(const int* __restrict__ boxes,
                                                          const int64_t* __restrict__ v_starts,
                                                          const int* __restrict__ ent_op,
                                                          const double2* __restrict__ cs, int p, int KRp,
                                                          int64_t chunk_base, const double* __restrict__ temp,
                                                          const double4* __restrict__ box, double* __restrict__ L,
                                                          int kp2) {
  const int b = boxes[blockIdx.x];
  const int64_t a = v_starts[b], e = v_starts[b + 1];
  const int NR = hsize(p);
  const double ih = 1.0 / box[b].w;
  for (int q = threadIdx.x; q < NR; q += blockDim.x) {
    int n, m;
    q_nm(q, n, m);
    double sx = 0.0, sy = 0.0;
    const int qi = m > 0 ? NR + n * (n - 1) / 2 + m - 1 : q;
    // kU entries' loads in flight per thread (the kernel is HBM-bound on the staging
    // rows); the sums still run in CSR order
    constexpr int kU = 4;
    int64_t pos = a;
    for (; pos + kU <= e; pos += kU) {
      double re[kU], im[kU];
      double2 r[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const double* row = temp + (pos + u - chunk_base) * KRp;
        re[u] = __ldcs(row + q);
        im[u] = m > 0 ? __ldcs(row + qi) : 0.0;
        r[u] = m > 0 ? cs[size_t(__ldg(ent_op + pos + u)) * (p + 1) + m] : make_double2(1.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (m == 0) {
          sx += re[u];
        } else {
          sx += re[u] * r[u].x + im[u] * r[u].y;
          sy += im[u] * r[u].x - re[u] * r[u].y;
        }
      }
    }
    for (; pos < e; ++pos) {
      const double* row = temp + (pos - chunk_base) * KRp;
      const double re = __ldcs(row + q);
      if (m == 0) {
        sx += re;
      } else {
        const double im = __ldcs(row + qi);
        const double2 r = cs[size_t(ent_op[pos]) * (p + 1) + m];
        sx += re * r.x + im * r.y;
        sy += im * r.x - re * r.y;
      }
    }
    L[size_t(b) * kp2 + 2 * q] += sx * ih;
    if (m > 0) L[size_t(b) * kp2 + 2 * q + 1] += sy * ih;
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

int launch_m2l_ops(const M2LPlan& P, int p, const int* used_slot, const int4* rdof, cudaStream_t s) {
  const size_t smem = hsize(2 * p) * sizeof(double2);
  cudaFuncSetAttribute(k_m2l_ops, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_m2l_ops<<<P.n_ops, 256, smem, s>>>(p, P.KR, P.KRp, used_slot, rdof, P.ops);
  return 1;
}

int split_nh(int p) { return (hsize(p) + 47) / 48 * 48; }
int split_nhi(int p, int NH) {  // Im block rows: whole warps of 8 * MT rows (MT = NH / 48)
  const int rows = 8 * (NH / 48), ni = hsize(p) - (p + 1);
  return (ni + rows - 1) / rows * rows;
}
int split_tile_cols() {
  const char* v1 = std::getenv("QBXG_SPLIT_V1");
  return v1 != nullptr ? 32 : kSplitBN;
}

int launch_m2l_ops_split(const M2LPlan& P, int p, const int* used_slot, cudaStream_t s) {
  const size_t smem = hsize(2 * p) * sizeof(double2);
  cudaFuncSetAttribute(k_m2l_ops_split, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_m2l_ops_split<<<P.n_ops, 256, smem, s>>>(p, split_nh(p), split_nhi(p, split_nh(p)), used_slot, P.sops, P.cs);
  return 1;
}

int launch_m2l_dense(const M2LPlan& P, const DevData& D, cudaStream_t s) {
  int k = 0;
  const int kp2 = 2 * D.kp;
  for (int c = 0; c < int(P.chunks.size()); ++c) {
    const M2LChunk& C = P.chunks[c];
    if (C.n_tiles == 0) continue;
    if (P.pas) {
      launch_m2l_pas(P, C, reinterpret_cast<const double*>(D.M), kp2, D.p, s);
    } else if (P.split) {
      const double* X = reinterpret_cast<const double*>(D.M);
      switch (split_nh(D.p)) {
        case 48: split_nh_launch<48>(P, C, X, kp2, D.p, s); break;
        case 96: split_nh_launch<96>(P, C, X, kp2, D.p, s); break;
        case 144: split_nh_launch<144>(P, C, X, kp2, D.p, s); break;
        case 192: split_nh_launch<192>(P, C, X, kp2, D.p, s); break;
        case 240: split_nh_launch<240>(P, C, X, kp2, D.p, s); break;
        default: return -1;
      }
    } else if (P.rot) {
      static const bool v3 = std::getenv("QBXG_M2L_ROTV") && std::getenv("QBXG_M2L_ROTV")[0] == '3';
      if (!v3 && m2l_rot4_ok(D.p))
        launch_m2l_rot4_chunk(P, C, D, s);
      else if (m2l_rot3_ok(D.p))
        launch_m2l_rot3_chunk(P, C, D, s);
      else
        launch_m2l_rot2_chunk(P, C, D, s);
    } else if (gemm_any(P.KRp, P.ops, C.n_tiles, C.tiles, C.col_src, C.col_pos, C.col_scale, P.rmap,
                        reinterpret_cast<const double*>(D.M), kp2, P.temp, s, P.bn) < 0) {
      return -1;
    }
    if (P.split)
      k_m2l_reduce_split<<<C.n_boxes, 160, 0, s>>>(C.boxes, D.v_starts, P.ent_op, P.cs, D.p, P.KRp, C.base,
                                                   P.temp, D.box, reinterpret_cast<double*>(D.L), kp2);
    else
      k_m2l_reduce<<<C.n_boxes, 256, 0, s>>>(C.boxes, D.v_starts, C.base, P.KR, P.KRp, P.rmap, P.temp, D.box,
                                              reinterpret_cast<double*>(D.L), kp2);
    k += 2;
  }
  return k;
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
