// Stage 4 M2L (List 2) as point-and-shoot in the azimuthal frame, on real
// half-table blocks.
//
// The split M2L (m2l_gemm.cu) rotates about z by alpha = atan2(dy, dx) so the
// offset v' = (2 rho, 0, 2 dz) lies in the xz-plane; there the operator is real
// and block diagonal in (Re, Im) -- two dense hsize(p)^2 blocks.  Rotating on
// about y by theta = angle(v', z) puts v' on +z, where the translation is
// diagonal in the order m.  For real data (M_n^{-m} = (-1)^m conj M_n^m) each of
// the three factors keeps Re and Im parts apart:
//   W (multipole rotation):  per degree j, a (j+1)^2 Re block and a j^2 Im block
//   Z (z-translation):       per order m, rows n / columns j in [m, p]:
//                            (-1)^{n+m} (j+n)! / |v'|^{j+n+1}, the same for Re and Im
//   V (local back-rotation): per degree n, like W
// 3 x 2,736 multiply-adds per List-2 entry at p = 15 instead of 32,896 for the two
// dense blocks: 4x less arithmetic (3x on the tensor pipe after padding blocks to
// 8-row / 4-column DMMA tiles).
// W and V are the real parts of the validated rotation blocks of rotation.cpp
// evaluated at v' (phi = 0, so their Re/Im cross terms vanish; checked at setup).
//
// Kernel: one CTA = one offset x 32 entries (tiles as the split M2L).  The
// gathered, alpha-rotated multipoles sit in shared memory as (p+1)^2 rows (Re in
// hidx order, Im in compacted order) x 32 columns.  In each phase every warp owns
// a fixed list of whole blocks (longest-processing-time balanced on the host), so
// the phase runs in place: the warp reads a block's operator (A fragments, from
// L2) and its rows (B fragments, from shared memory) into registers, runs the
// m8n8k4 DMMAs, then writes its rows.  Output rows use the split M2L's
// staging layout, so its CSR-order reduce (back-rotation by alpha, 1/|b|)
// finishes the job unchanged.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "harmonics.cuh"
#include "kernels.cuh"
#include "../host/rotation.hpp"

namespace qbxg {
namespace dev {

namespace {

constexpr int kPasPhases = 3;
constexpr int kWarps = 8, kBN = 32, kLD = kBN + 1;
constexpr int kWarps2 = 16;
__host__ __device__ constexpr int pas2_f(int n, int m) {
  return 4 * ((0x36 >> (2 * ((n + m) & 3))) & 3) + (((n + m) >> 2) & 3);
}
__host__ __device__ constexpr int pas2_code(int row, int n, int m) { return row * kBN | pas2_f(n, m); }

// shared-memory address of (row, column): plain rows of kLD doubles (row codes are row
// indices) or swizzled rows of 32 (row codes from pas2_code)
template <bool SWZ>
__device__ __forceinline__ int xa(int code, int c) {
  return SWZ ? (code & ~(kBN - 1)) + (c ^ (code & (kBN - 1))) : code * kLD + c;
}


// table layout (ints), per phase: [nblk+1 row offsets][nblk op offsets]
// [(p+1)^2 rows][kWarps+1 warp offsets][block ids]
struct TabHead {
  int base[kPasPhases];
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One block of size S in place on the fp64 tensor pipe (mma.sync m8n8k4): the
// operator (rows padded to 8, columns to 4, zeros) as A fragments from L2, the
// block's rows x 32 columns as B fragments from shared memory -- all read before
// any row is written, so the warp may overwrite its own block.
template <int S, bool SWZ>
__device__ __forceinline__ void pas_block(double* X, const int* rw, const double* __restrict__ Ob, int lane) {
  constexpr int MT = (S + 7) / 8, KS = (S + 3) / 4, K4 = 4 * KS, NT = kBN / 8;
  double a[MT][KS], b[KS][NT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[mt][ks] = __ldg(Ob + (mt * 8 + (lane >> 2)) * K4 + ks * 4 + (lane & 3));
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + (lane & 3);
    const int row = k < S ? rw[k] : 0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[ks][nt] = k < S ? X[xa<SWZ>(row, nt * 8 + (lane >> 2))] : 0.0;
  }
  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt][ks], b[ks][nt]);
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = mt * 8 + (lane >> 2);
    if (r < S) {
      const int row = rw[r];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        if (SWZ) {  // the swizzle keeps column pairs (2t, 2t+1) adjacent, possibly swapped
          const int msk = row & (kBN - 1);
          const int pos = (row & ~(kBN - 1)) + (((nt * 8 + (lane & 3) * 2) ^ msk) & ~1);
          *reinterpret_cast<double2*>(X + pos) = (msk & 1) ? make_double2(acc[mt][nt][1], acc[mt][nt][0])
                                                           : make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        } else {
          X[row * kLD + nt * 8 + (lane & 3) * 2] = acc[mt][nt][0];
          X[row * kLD + nt * 8 + (lane & 3) * 2 + 1] = acc[mt][nt][1];
        }
      }
    }
  }
}

template <int P, bool SWZ>
__global__ void __launch_bounds__(kWarps * 32, 3) k_m2l_pas(const int* __restrict__ tab, int tab_n, TabHead hd,
                                                           int nblk, const double* __restrict__ ops, int op_stride,
                                                           int phase_size, const double2* __restrict__ cs_all,
                                                           const int4* __restrict__ tiles,
                                                           const int* __restrict__ col_src,
                                                           const int* __restrict__ col_pos,
                                                           const double* __restrict__ M, int kp2, int KRp,
                                                           double* __restrict__ temp) {
  constexpr int NR = hsize(P), NROW = (P + 1) * (P + 1), NTH = kWarps * 32;
  extern __shared__ double smem[];
  double* X = smem;
  int* s_tab = reinterpret_cast<int*>(X + NROW * (SWZ ? kBN : kLD));
  __shared__ int s_src[kBN];
  __shared__ double2 s_cs[P + 1];
  // half-table index q: Re row | Im row << 10 (0 for m = 0) | m << 20 | swizzle << 25
  __shared__ int s_code[NR];
  __shared__ int s_rc[NROW];  // row code of each storage row (xa)
  __shared__ int s_pos[kBN];
  const int4 tile = tiles[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < tab_n; i += NTH) s_tab[i] = tab[i];
  if (tid < kBN) s_src[tid] = tid < tile.z ? col_src[tile.y + tid] : -1;
  if (tid < kBN) s_pos[tid] = tid < tile.z ? col_pos[tile.y + tid] : -1;
  if (tid <= P) s_cs[tid] = cs_all[size_t(tile.x) * (P + 1) + tid];
  for (int q = tid; q < NR; q += NTH) {
    int n = 0;
    while (hidx(n + 1, 0) <= q) ++n;
    const int m = q - hidx(n, 0);
    const int ri = m > 0 ? NR + n * (n - 1) / 2 + m - 1 : 0;
    s_code[q] = q | ri << 10 | m << 20 | (SWZ ? pas2_f(n, m) : 0) << 25;
    s_rc[q] = SWZ ? pas2_code(q, n, m) : q;
    if (m > 0) s_rc[ri] = SWZ ? pas2_code(ri, n, m) : ri;
  }
  __syncthreads();
  // gather M' = M e^{i k alpha}, coalesced along each multipole, kSt loads in flight per thread
  constexpr int kSt = 6;
  for (int base = 0; base < NR * kBN; base += kSt * NTH) {
    double2 v[kSt];
#pragma unroll
    for (int u = 0; u < kSt; ++u) {
      const int e = base + tid + u * NTH;
      v[u] = make_double2(0.0, 0.0);
      if (e < NR * kBN) {
        const int c = e / NR, q = e - c * NR;
        const int src = s_src[c];
        if (src >= 0) v[u] = __ldg(reinterpret_cast<const double2*>(M + size_t(src) * kp2) + q);
      }
    }
#pragma unroll
    for (int u = 0; u < kSt; ++u) {
      const int e = base + tid + u * NTH;
      if (e < NR * kBN) {
        const int c = e / NR, q = e - c * NR;
        const int code = s_code[q], ri = (code >> 10) & 1023;
        const double2 r = s_cs[(code >> 20) & 31];
        const int cs = SWZ ? c ^ (code >> 25) : c, ld = SWZ ? kBN : kLD;
        X[(code & 1023) * ld + cs] = v[u].x * r.x - v[u].y * r.y;
        if (ri) X[ri * ld + cs] = v[u].x * r.y + v[u].y * r.x;
      }
    }
  }
  __syncthreads();
  const double* opb = ops + size_t(tile.x) * op_stride;
#pragma unroll 1
  for (int ph = 0; ph < kPasPhases; ++ph) {
    const int* T = s_tab + hd.base[ph];
    const int* rowoff = T;
    const int* opoff = T + nblk + 1;
    const int* rows = opoff + nblk;
    const int* woff = rows + NROW;
    const int* wblk = woff + kWarps + 1;
    const double* Op = opb + size_t(ph) * phase_size;
#pragma unroll 1
    for (int i = woff[warp]; i < woff[warp + 1]; ++i) {
      const int b = wblk[i];
      const int* rw = rows + rowoff[b];
      const double* Ob = Op + opoff[b];
      switch (rowoff[b + 1] - rowoff[b]) {
#define QBXG_PAS_CASE(S) \
  case S:                \
    pas_block<S, SWZ>(X, rw, Ob, lane); \
    break;
        QBXG_PAS_CASE(1) QBXG_PAS_CASE(2) QBXG_PAS_CASE(3) QBXG_PAS_CASE(4) QBXG_PAS_CASE(5) QBXG_PAS_CASE(6)
        QBXG_PAS_CASE(7) QBXG_PAS_CASE(8) QBXG_PAS_CASE(9) QBXG_PAS_CASE(10) QBXG_PAS_CASE(11) QBXG_PAS_CASE(12)
        QBXG_PAS_CASE(13) QBXG_PAS_CASE(14) QBXG_PAS_CASE(15) QBXG_PAS_CASE(16)
#undef QBXG_PAS_CASE
        default: break;
      }
    }
    __syncthreads();
  }
  // staging row = Re (NR) then compacted Im, coalesced along each row
  // (row-outer: one row code per thread and row; consecutive lanes, consecutive rows)
  for (int r = tid; r < NROW; r += NTH) {
    const int code = s_rc[r];
    for (int c = 0; c < tile.z; ++c) temp[size_t(s_pos[c]) * KRp + r] = X[xa<SWZ>(code, c)];
  }
}

// ------------------------------------------------- v2: persistent, operator in smem
// One CTA per SM walks a contiguous run of the offset-sorted tiles.  The offset's
// operator [W | Z | V] (96 KB at p = 15) is copied into shared memory once per run
// of same-offset tiles (~460 tiles per offset at config 1) and read as DMMA A
// fragments in fragment order (conflict-free); the next tile's multipoles are
// loaded into registers while the current tile runs its three phases.  16 warps:
// warp w owns the blocks of LPT list w % 8 for columns 16 (w / 8) .. + 15.
//
// The tile is 32 columns per row with the columns XOR-swizzled per row by
// f(n + m) = 4 sigma + tau, sigma = (2, 1, 3, 0)[(n + m) & 3], tau = ((n + m) >> 2) & 3:
//  - any 4 consecutive rows of a W/V block (consecutive m) or Z block (consecutive
//    n) have distinct sigma: the B-fragment loads (4 rows x 4 columns per half warp)
//    are conflict-free;
//  - adjacent block rows differ in sigma's bit 1: the C-fragment stores (double2,
//    2 rows x 8 columns per quarter warp) are conflict-free;
//  - f is a bijection of (n + m) mod 16: the column passes (16 consecutive rows of one
//    column per half warp) conflict only where a degree ends inside the 16 rows.
template <int S>
__device__ __forceinline__ void pas2_block(double* X, const int* rw, const double* Ob, int lane, int colbase) {
  constexpr int MT = (S + 7) / 8, KS = (S + 3) / 4, NT = 2;
  double a[MT][KS], b[KS][NT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[mt][ks] = Ob[(mt * KS + ks) * 32 + lane];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + (lane & 3);
    const int code = k < S ? rw[k] : 0, base = code & ~(kBN - 1), msk = code & (kBN - 1);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[ks][nt] = k < S ? X[base + ((colbase + nt * 8 + (lane >> 2)) ^ msk)] : 0.0;
  }
  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt][ks], b[ks][nt]);
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = mt * 8 + (lane >> 2);
    if (r < S) {
      const int code = rw[r], base = code & ~(kBN - 1), msk = code & (kBN - 1);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int pos = ((colbase + nt * 8 + (lane & 3) * 2) ^ msk) & ~1;
        *reinterpret_cast<double2*>(X + base + pos) =
            (msk & 1) ? make_double2(acc[mt][nt][1], acc[mt][nt][0]) : make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      }
    }
  }
}

template <int P>
__global__ void __launch_bounds__(kWarps2 * 32, 1)
    k_m2l_pas2(const int* __restrict__ tab, int tab_n, TabHead hd, int nblk, const double* __restrict__ ops,
               int op_stride, int phase_size, const double2* __restrict__ cs_all, const int4* __restrict__ tiles,
               int n_tiles, const int* __restrict__ col_src, const int* __restrict__ col_pos,
               const double* __restrict__ M, int kp2, int KRp, double* __restrict__ temp) {
  constexpr int NR = hsize(P), NROW = (P + 1) * (P + 1), NTH = kWarps2 * 32;
  constexpr int NV = (NR * kBN + NTH - 1) / NTH;  // multipole coefficients prefetched per thread
  extern __shared__ double smem[];
  double* OPS = smem;
  double* X = OPS + op_stride;
  int* s_tab = reinterpret_cast<int*>(X + NROW * kBN);
  __shared__ double2 s_cs[P + 1];
  __shared__ int s_rc[NROW];  // row codes (row * 32 | swizzle) of the storage rows
  __shared__ int s_qi[NR];    // m | Im storage row << 8 of half-table index q
  __shared__ int s_pos[kBN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < tab_n; i += NTH) s_tab[i] = tab[i];
  for (int q = tid; q < NR; q += NTH) {
    int n = 0;
    while (hidx(n + 1, 0) <= q) ++n;
    const int m = q - hidx(n, 0), ri = m > 0 ? NR + n * (n - 1) / 2 + m - 1 : 0;
    s_qi[q] = m | ri << 8;
    s_rc[q] = pas2_code(q, n, m);
    if (m > 0) s_rc[ri] = pas2_code(ri, n, m);
  }
  const int t0 = int(int64_t(blockIdx.x) * n_tiles / gridDim.x);
  const int t1 = int(int64_t(blockIdx.x + 1) * n_tiles / gridDim.x);
  double2 v[NV];
  auto prefetch = [&](int t) {
    const int4 tl = tiles[t];
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int e = tid + u * NTH, c = e / NR, q = e - c * NR;
      v[u] = make_double2(0.0, 0.0);
      if (e < NR * kBN && c < tl.z)
        v[u] = __ldg(reinterpret_cast<const double2*>(M + size_t(__ldg(col_src + tl.y + c)) * kp2) + q);
    }
  };
  if (t0 < t1) prefetch(t0);
  int cur = -1;
#pragma unroll 1
  for (int t = t0; t < t1; ++t) {
    const int4 tile = tiles[t];
    __syncthreads();  // the previous tile's write-out has read X
    if (tile.x != cur) {
      cur = tile.x;
      const double2* src = reinterpret_cast<const double2*>(ops + size_t(cur) * op_stride);
      for (int i = tid; i < op_stride / 2; i += NTH) reinterpret_cast<double2*>(OPS)[i] = __ldg(src + i);
      if (tid <= P) s_cs[tid] = cs_all[size_t(cur) * (P + 1) + tid];
      __syncthreads();
    }
    if (tid < kBN) s_pos[tid] = tid < tile.z ? col_pos[tile.y + tid] : -1;
    // M' = M e^{i k alpha} into the tile
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      const int e = tid + u * NTH, c = e / NR, q = e - c * NR;
      if (e < NR * kBN) {
        const int qi = s_qi[q], m = qi & 255;
        const double2 r = s_cs[m];
        const int code = s_rc[q];
        X[(code & ~(kBN - 1)) + (c ^ (code & (kBN - 1)))] = v[u].x * r.x - v[u].y * r.y;
        if (m > 0) {
          const int ci = s_rc[qi >> 8];
          X[(ci & ~(kBN - 1)) + (c ^ (ci & (kBN - 1)))] = v[u].x * r.y + v[u].y * r.x;
        }
      }
    }
    __syncthreads();
    if (t + 1 < t1) prefetch(t + 1);  // in flight during the phases
    const int colbase = (warp >> 3) * 16, wq = warp & 7;
#pragma unroll 1
    for (int ph = 0; ph < kPasPhases; ++ph) {
      const int* T = s_tab + hd.base[ph];
      const int* rowoff = T;
      const int* opoff = T + nblk + 1;
      const int* rows = opoff + nblk;
      const int* woff = rows + NROW;
      const int* wblk = woff + kWarps + 1;
      const double* Op = OPS + size_t(ph) * phase_size;
#pragma unroll 1
      for (int i = woff[wq]; i < woff[wq + 1]; ++i) {
        const int b = wblk[i];
        const int* rw = rows + rowoff[b];
        const double* Ob = Op + opoff[b];
        switch (rowoff[b + 1] - rowoff[b]) {
#define QBXG_PAS2_CASE(S) \
  case S:                 \
    pas2_block<S>(X, rw, Ob, lane, colbase); \
    break;
          QBXG_PAS2_CASE(1) QBXG_PAS2_CASE(2) QBXG_PAS2_CASE(3) QBXG_PAS2_CASE(4) QBXG_PAS2_CASE(5)
          QBXG_PAS2_CASE(6) QBXG_PAS2_CASE(7) QBXG_PAS2_CASE(8) QBXG_PAS2_CASE(9) QBXG_PAS2_CASE(10)
          QBXG_PAS2_CASE(11) QBXG_PAS2_CASE(12) QBXG_PAS2_CASE(13) QBXG_PAS2_CASE(14) QBXG_PAS2_CASE(15)
          QBXG_PAS2_CASE(16)
#undef QBXG_PAS2_CASE
          default: break;
        }
      }
      __syncthreads();
    }
    // staging rows (Re, then compacted Im): consecutive lanes walk one column's rows
    for (int e = tid; e < NROW * kBN; e += NTH) {
      const int c = e / NROW, r = e - c * NROW, pos = s_pos[c];
      if (pos >= 0) {
        const int code = s_rc[r];
        temp[size_t(pos) * KRp + r] = X[(code & ~(kBN - 1)) + (c ^ (code & (kBN - 1)))];
      }
    }
  }
}

// ------------------------------------------- v3: persistent, warp-specialised pipeline
// One CTA per SM walks tiles blockIdx.x, blockIdx.x + grid, ... through two tile buffers.
// kMemW memory warps gather tile k+1 (and write out tile k-1's staging rows) while the
// compute warps run tile k's three phases; the hand-off uses named barriers
// (FULL[b]: memory -> compute, DONE[b]: compute -> memory; bar.arrive / bar.sync).
// CW = 8 compute warps own all 32 columns of their blocks, CW = 16 split them in halves.
constexpr int kMemW = 4;

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// block of size S on NT 8-column groups starting at column cb (padded rows of kLD)
template <int S, int NT>
__device__ __forceinline__ void pas3_block(double* X, const int* rw, const double* __restrict__ Ob, int lane, int cb) {
  constexpr int MT = (S + 7) / 8, KS = (S + 3) / 4, K4 = 4 * KS;
  double a[MT][KS], b[KS][NT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[mt][ks] = __ldg(Ob + (mt * 8 + (lane >> 2)) * K4 + ks * 4 + (lane & 3));
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = ks * 4 + (lane & 3);
    const int row = k < S ? rw[k] : 0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) b[ks][nt] = k < S ? X[row * kLD + cb + nt * 8 + (lane >> 2)] : 0.0;
  }
  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt][ks], b[ks][nt]);
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = mt * 8 + (lane >> 2);
    if (r < S) {
      double* x = X + rw[r] * kLD + cb + (lane & 3) * 2;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        x[nt * 8] = acc[mt][nt][0];
        x[nt * 8 + 1] = acc[mt][nt][1];
      }
    }
  }
}

template <int P, int CW>
__global__ void __launch_bounds__((CW + kMemW) * 32, 1)
    k_m2l_pas3(const int* __restrict__ tab, int tab_n, TabHead hd, int nblk, const double* __restrict__ ops,
               int op_stride, int phase_size, const double2* __restrict__ cs_all, const int4* __restrict__ tiles,
               int n_tiles, const int* __restrict__ col_src, const int* __restrict__ col_pos,
               const double* __restrict__ M, int kp2, int KRp, double* __restrict__ temp) {
  constexpr int NR = hsize(P), NROW = (P + 1) * (P + 1), CT = CW * 32, MEMT = kMemW * 32, NTHR = CT + MEMT;
  constexpr int NT = CW == 8 ? 4 : 2;
  extern __shared__ double smem[];
  double* Xb = smem;  // two tiles of NROW x kLD
  int* s_tab = reinterpret_cast<int*>(Xb + 2 * NROW * kLD);
  __shared__ int s_src[2][kBN], s_pos[2][kBN], s_op[2], s_cnt[2];
  __shared__ double2 s_cs[2][P + 1];
  __shared__ int s_code[NR];  // Re row | Im row << 10 (0 for m = 0) | m << 20 of half-table index q
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < tab_n; i += NTHR) s_tab[i] = tab[i];
  for (int q = tid; q < NR; q += NTHR) {
    int n = 0;
    while (hidx(n + 1, 0) <= q) ++n;
    const int m = q - hidx(n, 0);
    s_code[q] = q | (m > 0 ? NR + n * (n - 1) / 2 + m - 1 : 0) << 10 | m << 20;
  }
  __syncthreads();
  const int ntl = blockIdx.x < n_tiles ? (n_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  if (warp >= CW) {
    // ---- memory warps: write out tile k-2, gather tile k, into buffer k & 1
    const int mt = tid - CT;
    for (int k = 0; k < ntl + 2; ++k) {
      const int b = k & 1;
      double* X = Xb + b * NROW * kLD;
      if (k >= 2) {
        nb_sync(3 + b, NTHR);  // DONE[b]: tile k-2's phases are finished
        const int cnt = s_cnt[b];
        for (int r = mt; r < NROW; r += MEMT)
          for (int c = 0; c < cnt; ++c) temp[size_t(s_pos[b][c]) * KRp + r] = X[r * kLD + c];
        nb_sync(5, MEMT);
      }
      if (k < ntl) {
        const int4 tile = tiles[blockIdx.x + size_t(k) * gridDim.x];
        if (mt < kBN) {
          s_src[b][mt] = mt < tile.z ? col_src[tile.y + mt] : -1;
          s_pos[b][mt] = mt < tile.z ? col_pos[tile.y + mt] : -1;
        }
        if (mt <= P) s_cs[b][mt] = cs_all[size_t(tile.x) * (P + 1) + mt];
        if (mt == 0) {
          s_op[b] = tile.x;
          s_cnt[b] = tile.z;
        }
        nb_sync(5, MEMT);
        constexpr int kSt = 8;
        for (int base = 0; base < NR * kBN; base += kSt * MEMT) {
          double2 v[kSt];
#pragma unroll
          for (int u = 0; u < kSt; ++u) {
            const int e = base + mt + u * MEMT;
            v[u] = make_double2(0.0, 0.0);
            if (e < NR * kBN) {
              const int c = e / NR, q = e - c * NR;
              const int src = s_src[b][c];
              if (src >= 0) v[u] = __ldg(reinterpret_cast<const double2*>(M + size_t(src) * kp2) + q);
            }
          }
#pragma unroll
          for (int u = 0; u < kSt; ++u) {
            const int e = base + mt + u * MEMT;
            if (e < NR * kBN) {
              const int c = e / NR, q = e - c * NR;
              const int code = s_code[q], ri = (code >> 10) & 1023;
              const double2 r = s_cs[b][code >> 20];
              X[(code & 1023) * kLD + c] = v[u].x * r.x - v[u].y * r.y;
              if (ri) X[ri * kLD + c] = v[u].x * r.y + v[u].y * r.x;
            }
          }
        }
        nb_arrive(1 + b, NTHR);  // FULL[b]
      }
    }
  } else {
    // ---- compute warps: the three phases of tile k in buffer k & 1
    const int wq = warp % kWarps, cb = CW == 8 ? 0 : (warp / kWarps) * 16;
    for (int k = 0; k < ntl; ++k) {
      const int b = k & 1;
      double* X = Xb + b * NROW * kLD;
      nb_sync(1 + b, NTHR);  // FULL[b]
      const double* opb = ops + size_t(s_op[b]) * op_stride;
#pragma unroll 1
      for (int ph = 0; ph < kPasPhases; ++ph) {
        const int* T = s_tab + hd.base[ph];
        const int* rowoff = T;
        const int* opoff = T + nblk + 1;
        const int* rows = opoff + nblk;
        const int* woff = rows + NROW;
        const int* wblk = woff + kWarps + 1;
        const double* Op = opb + size_t(ph) * phase_size;
#pragma unroll 1
        for (int i = woff[wq]; i < woff[wq + 1]; ++i) {
          const int bl = wblk[i];
          const int* rw = rows + rowoff[bl];
          const double* Ob = Op + opoff[bl];
          switch (rowoff[bl + 1] - rowoff[bl]) {
#define QBXG_PAS3_CASE(S) \
  case S:                 \
    pas3_block<S, NT>(X, rw, Ob, lane, cb); \
    break;
            QBXG_PAS3_CASE(1) QBXG_PAS3_CASE(2) QBXG_PAS3_CASE(3) QBXG_PAS3_CASE(4) QBXG_PAS3_CASE(5)
            QBXG_PAS3_CASE(6) QBXG_PAS3_CASE(7) QBXG_PAS3_CASE(8) QBXG_PAS3_CASE(9) QBXG_PAS3_CASE(10)
            QBXG_PAS3_CASE(11) QBXG_PAS3_CASE(12) QBXG_PAS3_CASE(13) QBXG_PAS3_CASE(14) QBXG_PAS3_CASE(15)
            QBXG_PAS3_CASE(16)
#undef QBXG_PAS3_CASE
            default: break;
          }
        }
        nb_sync(6, CT);  // compute warps only
      }
      nb_arrive(3 + b, NTHR);  // DONE[b]
    }
  }
}

// ---------------------------------------------------------------- host side
struct PasLayout {
  int nblk = 0, phase_size = 0;
  std::vector<int> tab;
  TabHead hd{};
};

// blocks of one phase: storage rows (Re rows hidx(n, m); Im rows NR + n(n-1)/2 + m - 1),
// as row indices (v1) or as row codes with the v2 swizzle
void phase_blocks(int p, int ph, bool v2, std::vector<std::vector<int>>& blocks) {
  const int NR = hsize(p);
  auto re = [&](int n, int m) { return v2 ? pas2_code(hidx(n, m), n, m) : hidx(n, m); };
  auto im = [&](int n, int m) {
    const int r = NR + n * (n - 1) / 2 + m - 1;
    return v2 ? pas2_code(r, n, m) : r;
  };
  blocks.clear();
  for (int part = 0; part < 2; ++part)
    for (int a = part; a <= p; ++a) {
      std::vector<int> b;
      if (ph != 1)  // W, V: degree a, orders part..a
        for (int m = part; m <= a; ++m) b.push_back(part ? im(a, m) : re(a, m));
      else  // Z: order a, degrees a..p
        for (int n = a; n <= p; ++n) b.push_back(part ? im(n, a) : re(n, a));
      blocks.push_back(b);
    }
}

PasLayout make_layout(int p, bool v2) {
  PasLayout L;
  for (int ph = 0; ph < kPasPhases; ++ph) {
    std::vector<std::vector<int>> blocks;
    phase_blocks(p, ph, v2, blocks);
    L.nblk = int(blocks.size());
    L.hd.base[ph] = int(L.tab.size());
    std::vector<int> rowoff{0}, opoff, rows;
    int oo = 0;
    for (auto& b : blocks) {
      const int s = int(b.size());
      rows.insert(rows.end(), b.begin(), b.end());
      rowoff.push_back(int(rows.size()));
      opoff.push_back(oo);
      oo += (s + 7) / 8 * 8 * ((s + 3) / 4 * 4);  // rows padded to 8, columns to 4
    }
    L.phase_size = oo;  // the same for the three phases (same block sizes)
    // whole blocks per warp, longest processing time first
    std::vector<int> order(blocks.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = int(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return blocks[a].size() > blocks[b].size(); });
    std::vector<std::vector<int>> wl(kWarps);
    std::vector<long> load(kWarps, 0);
    for (int bi : order) {
      const int w = int(std::min_element(load.begin(), load.end()) - load.begin());
      load[w] += long(blocks[bi].size() * blocks[bi].size());
      wl[w].push_back(bi);
    }
    std::vector<int> woff{0}, wblk;
    for (auto& v : wl) {
      wblk.insert(wblk.end(), v.begin(), v.end());
      woff.push_back(int(wblk.size()));
    }
    for (auto* v : {&rowoff, &opoff, &rows, &woff, &wblk}) L.tab.insert(L.tab.end(), v->begin(), v->end());
  }
  return L;
}

// v1 (one tile per CTA, 3 CTAs per SM, operators read from L2) is the default: the
// persistent v2 (QBXG_PAS_V2=1, 1 CTA of 16 warps per SM, operator in shared memory)
// is parity-green but slower at config 1 (64.2 vs 45.8 ms for the M2L stage): with one
// CTA per SM nothing fills the phase barriers and the staging stores.
bool pas_v2() {
  static const bool v2 = std::getenv("QBXG_PAS_V2") != nullptr;
  return v2;
}
// v1 tile layout: padded rows of 33 (default) or swizzled rows of 32 (QBXG_PAS_SWZ=1).
// The swizzle removes the B-load / C-store bank conflicts (shared wavefronts 4.7G ->
// 3.3G per chunk-1 launch) but its per-access XOR addressing costs 36% more issued
// instructions, and the kernel is latency/issue-limited: 32.4 vs 25.7 ms (ncu).
bool pas_swz() {
  static const bool on = std::getenv("QBXG_PAS_SWZ") && std::getenv("QBXG_PAS_SWZ")[0] == '1';
  return on;
}

template <int P>
int pas2_launch_p(const M2LPlan& Pl, const M2LChunk& C, const double* X, int kp2, cudaStream_t s) {
  constexpr int NROW = (P + 1) * (P + 1);
  const size_t smem = size_t(Pl.pas_stride + NROW * kBN) * sizeof(double) + size_t(Pl.pas_tab_n) * sizeof(int);
  static size_t attr = 0;
  static int n_sm = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_m2l_pas2<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
      return -1;
    attr = smem;
  }
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  TabHead hd;
  for (int k = 0; k < 3; ++k) hd.base[k] = Pl.pas_base[k];
  const int grid = std::max(1, std::min(C.n_tiles, n_sm));
  k_m2l_pas2<P><<<grid, kWarps2 * 32, smem, s>>>(Pl.pas_tab, Pl.pas_tab_n, hd, Pl.pas_nblk, Pl.pas_ops, Pl.pas_stride,
                                                 Pl.pas_phase, Pl.cs, C.tiles, C.n_tiles, C.col_src, C.col_pos, X,
                                                 kp2, Pl.KRp, Pl.temp);
  return 1;
}

template <int P, bool SWZ>
int pas1_launch_p(const M2LPlan& Pl, const M2LChunk& C, const double* X, int kp2, cudaStream_t s);

// v3 (QBXG_PAS_V3=8 or 16 compute warps): the warp-specialised pipeline.  Parity-green but
// slower at config 1 (M2L 57.5 / 61.0 vs 42.9 ms): with one CTA per SM the phases of a
// single tile cannot hide the operator-fragment latency the three co-resident v1 CTAs hide.
// (A warp-owned-columns variant without any CTA barrier measured 82 ms: with one 8-column
// group per warp each operator fragment feeds one DMMA instead of four.)
int pas_v3() {
  static const int cw = std::getenv("QBXG_PAS_V3") ? std::atoi(std::getenv("QBXG_PAS_V3")) : 0;
  return cw == 8 || cw == 16 ? cw : 0;
}

template <int P, int CW>
int pas3_launch_p(const M2LPlan& Pl, const M2LChunk& C, const double* X, int kp2, cudaStream_t s) {
  constexpr int NROW = (P + 1) * (P + 1);
  const size_t smem = size_t(2 * NROW * kLD) * sizeof(double) + size_t(Pl.pas_tab_n) * sizeof(int);
  static size_t attr = 0;
  static int n_sm = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_m2l_pas3<P, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
        cudaSuccess)
      return -1;
    attr = smem;
  }
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  TabHead hd;
  for (int k = 0; k < 3; ++k) hd.base[k] = Pl.pas_base[k];
  const int grid = std::max(1, std::min(C.n_tiles, n_sm));
  k_m2l_pas3<P, CW><<<grid, (CW + kMemW) * 32, smem, s>>>(Pl.pas_tab, Pl.pas_tab_n, hd, Pl.pas_nblk, Pl.pas_ops,
                                                          Pl.pas_stride, Pl.pas_phase, Pl.cs, C.tiles, C.n_tiles,
                                                          C.col_src, C.col_pos, X, kp2, Pl.KRp, Pl.temp);
  return 1;
}

template <int P>
int pas_launch_p(const M2LPlan& Pl, const M2LChunk& C, const double* X, int kp2, cudaStream_t s) {
  if (pas_v2()) return pas2_launch_p<P>(Pl, C, X, kp2, s);
  if (pas_v3() == 8) return pas3_launch_p<P, 8>(Pl, C, X, kp2, s);
  if (pas_v3() == 16) return pas3_launch_p<P, 16>(Pl, C, X, kp2, s);
  return pas_swz() ? pas1_launch_p<P, true>(Pl, C, X, kp2, s) : pas1_launch_p<P, false>(Pl, C, X, kp2, s);
}

template <int P, bool SWZ>
int pas1_launch_p(const M2LPlan& Pl, const M2LChunk& C, const double* X, int kp2, cudaStream_t s) {
  constexpr int NROW = (P + 1) * (P + 1);
  const size_t smem = size_t(NROW * (SWZ ? kBN : kLD)) * sizeof(double) + size_t(Pl.pas_tab_n) * sizeof(int);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_m2l_pas<P, SWZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
      return -1;
    attr = smem;
  }
  TabHead hd;
  for (int k = 0; k < 3; ++k) hd.base[k] = Pl.pas_base[k];
  k_m2l_pas<P, SWZ><<<C.n_tiles, kWarps * 32, smem, s>>>(Pl.pas_tab, Pl.pas_tab_n, hd, Pl.pas_nblk, Pl.pas_ops,
                                                    Pl.pas_stride, Pl.pas_phase, Pl.cs, C.tiles, C.col_src,
                                                    C.col_pos, X, kp2, Pl.KRp, Pl.temp);
  return 1;
}

}  // namespace

bool pas_supported(int p) { return p >= 4 && p <= 15; }
int pas_tile_cols() { return kBN; }

// Per-offset operators: [W | Z | V], blocks in phase_blocks order, each with rows
// padded to 8 and columns to 4 (zeros): DMMA A fragments without guards.  v1: each
// block row-major; v2: each block in fragment order (8x4 fragment (mt, ks) as 32
// consecutive doubles, lane l holding element (mt*8 + l/4, ks*4 + l%4)).
void pas_build_ops(int p, int n_ops, const int* used_slot, std::vector<double>& ops, int& op_stride,
                   std::vector<int>& tab, int& nblk, int& phase_size, int (&base)[3]) {
  const bool v2 = pas_v2();
  const PasLayout L = make_layout(p, v2 || pas_swz());
  nblk = L.nblk;
  phase_size = L.phase_size;
  op_stride = kPasPhases * L.phase_size;
  tab = L.tab;
  for (int k = 0; k < 3; ++k) base[k] = L.hd.base[k];
  ops.assign(size_t(n_ops) * op_stride, 0.0);
  const size_t rs = rot_blocks_size(p);
  double worst = 0.0;
#pragma omp parallel for schedule(dynamic, 4) reduction(max : worst)
  for (int o = 0; o < n_ops; ++o) {
    const int sl = used_slot[o];
    const int dx = sl / 121 - 5, dy = (sl / 11) % 11 - 5, dz = sl % 11 - 5;
    const double v[3] = {2.0 * std::sqrt(double(dx * dx + dy * dy)), 0.0, 2.0 * dz};
    const double rho = std::sqrt(v[0] * v[0] + v[2] * v[2]);
    std::vector<double> Rf(rs), Rb(rs);
    m2l_rotation_blocks(p, v, Rf.data(), Rb.data());
    double* W = &ops[size_t(o) * op_stride];
    double* Z = W + L.phase_size;
    double* V = Z + L.phase_size;
    auto re = [](int m) { return m == 0 ? 0 : 2 * m - 1; };
    auto im = [](int m) { return 2 * m; };
    size_t w = 0, z = 0;
    for (int part = 0; part < 2; ++part)
      for (int a = part; a <= p; ++a) {
        // W, V: degree a (rows / columns = orders part..a); rows padded to 8, columns to 4
        const int d = 2 * a + 1, s = a + 1 - part, sr = (s + 7) / 8 * 8, sp = (s + 3) / 4 * 4;
        const double* F = &Rf[rot_block_offset(a)];
        const double* B = &Rb[rot_block_offset(a)];
        for (int i = 0; i < sr; ++i)
          for (int k = 0; k < sp; ++k) {
            const bool pad = i >= s || k >= s;
            const int mi = part + (pad ? 0 : i), mk = part + (pad ? 0 : k);
            const int ri = part ? im(mi) : re(mi), rk = part ? im(mk) : re(mk);
            W[w + size_t(i) * sp + k] = pad ? 0.0 : F[ri * d + rk];
            V[w + size_t(i) * sp + k] = pad ? 0.0 : B[ri * d + rk];
          }
        w += size_t(sr) * sp;
        for (int i = 0; i <= a; ++i)  // Re/Im cross terms vanish at phi = 0
          for (int k = 1; k <= a; ++k) {
            worst = std::max(worst, std::fabs(F[re(i) * d + im(k)]) + std::fabs(F[im(k) * d + re(i)]));
            worst = std::max(worst, std::fabs(B[re(i) * d + im(k)]) + std::fabs(B[im(k) * d + re(i)]));
          }
        // Z: order m = a, rows n / columns j in [m, p]: (-1)^{n+m} (j+n)! / rho^{j+n+1}
        const int m = a, sz = p - m + 1, szr = (sz + 7) / 8 * 8, szp = (sz + 3) / 4 * 4;
        for (int i = 0; i < szr; ++i)
          for (int k = 0; k < szp; ++k) {
            double val = 0.0;
            if (i < sz && k < sz) {
              const int n = m + i, j = m + k;
              double f = 1.0;
              for (int t = 2; t <= j + n; ++t) f *= t;
              val = (((n + m) & 1) ? -1.0 : 1.0) * f / std::pow(rho, j + n + 1);
            }
            Z[z + size_t(i) * szp + k] = val;
          }
        z += size_t(szr) * szp;
      }
  }
  if (worst > 1e-12) throw std::runtime_error("pas_build_ops: rotation blocks mix Re and Im at phi = 0");
  if (!v2) return;
  // row-major blocks -> fragment order, block by block (W and V share sizes, Z its own)
  std::vector<int> wsz, zsz;
  for (int part = 0; part < 2; ++part)
    for (int a = part; a <= p; ++a) {
      wsz.push_back(a + 1 - part);
      zsz.push_back(p - a + 1);
    }
#pragma omp parallel for schedule(static)
  for (int o = 0; o < n_ops; ++o) {
    std::vector<double> tmp(size_t(L.phase_size));
    for (int ph = 0; ph < kPasPhases; ++ph) {
      double* A = &ops[size_t(o) * op_stride + size_t(ph) * L.phase_size];
      const std::vector<int>& sz = ph == 1 ? zsz : wsz;
      size_t off = 0;
      for (int s : sz) {
        const int MT = (s + 7) / 8, KS = (s + 3) / 4, sp = KS * 4;
        for (int mt = 0; mt < MT; ++mt)
          for (int ks = 0; ks < KS; ++ks)
            for (int l = 0; l < 32; ++l)
              tmp[off + size_t(mt * KS + ks) * 32 + l] = A[off + size_t(mt * 8 + l / 4) * sp + ks * 4 + l % 4];
        off += size_t(MT) * 8 * sp;
      }
      std::copy(tmp.begin(), tmp.end(), A);
    }
  }
}

int launch_m2l_pas(const M2LPlan& P, const M2LChunk& C, const double* X, int kp2, int p, cudaStream_t s) {
  switch (p) {
    case 4: return pas_launch_p<4>(P, C, X, kp2, s);
    case 5: return pas_launch_p<5>(P, C, X, kp2, s);
    case 6: return pas_launch_p<6>(P, C, X, kp2, s);
    case 7: return pas_launch_p<7>(P, C, X, kp2, s);
    case 8: return pas_launch_p<8>(P, C, X, kp2, s);
    case 9: return pas_launch_p<9>(P, C, X, kp2, s);
    case 10: return pas_launch_p<10>(P, C, X, kp2, s);
    case 11: return pas_launch_p<11>(P, C, X, kp2, s);
    case 12: return pas_launch_p<12>(P, C, X, kp2, s);
    case 13: return pas_launch_p<13>(P, C, X, kp2, s);
    case 14: return pas_launch_p<14>(P, C, X, kp2, s);
    case 15: return pas_launch_p<15>(P, C, X, kp2, s);
    default: return -1;
  }
}

}  // namespace dev
}  // namespace qbxg
