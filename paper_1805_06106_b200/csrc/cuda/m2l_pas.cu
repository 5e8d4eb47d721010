// Stage 4 M2L (List 2) as point-and-shoot translations on real
// half-table blocks, accumulated per target box
// on chip.
//
// Operator.  With box-scaled coefficients the translation depends only on the offset
// delta = (c_b - c_d) / (2|b|) in [-5,5]^3.  Rotating the frame about z by
// alpha = atan2(dy, dx) puts v = 2 delta in the xz-plane (v' = (2 rho_xy, 0, 2 dz));
// with M' = M e^{i k alpha} and L = L' e^{-i m alpha} the remaining map is real and
// keeps Re and Im parts apart, and factors as
//   W (rotation about y by theta = angle(v', z)): per degree j, a (j+1)^2 Re block and a j^2 Im block
//   Z (translation along z by |v'|):             per order m, rows n / columns j in [m, p]:
//                                                (-1)^{n+m} (j+n)! / |v'|^{j+n+1}, the same for Re and Im
//   V (local rotation back):                    per degree n, like W
// 3 x 2,736 multiply-adds per List-2 entry at p = 15 instead of 32,896 for the two dense
// azimuthal blocks.  W, Z and V depend on (rho_xy^2, dz) only, and an offset below the
// xy-plane is the mirror image of one above it: T(rho, -dz) = S T(rho, dz) S with the
// diagonal sign S = (-1)^{n+m} on both expansions.  So the 1,206 offsets of [-5,5]^3 fall
// into 102 classes (rho_xy^2, |dz|), one operator set per class (~10 MB at p = 15); the
// signs are applied in the gather and the accumulate (kPasMirror column flag).  Classes on
// the z axis (rho_xy = 0) have W = V = identity: their tiles run the Z phase only.
//
// Work split (target-grouped).  One CTA owns a group of G target boxes (48 at p <= 16,
// consecutive in DFS order) and walks a host-built list of tiles: a tile is <= BN (40 at
// p <= 15) List-2 entries of the group that share an operator class, columns sorted by
// (target slot, offset).  Two CTAs of 8 warps share an SM (one CTA's gather, barriers
// and accumulate overlap the other's DMMA phases).  Per tile:
//   1. the columns' multipoles are read from L2 and rotated by e^{i k alpha} into the
//      (p+1)^2 x BN real tile X in shared memory (XOR-swizzled): a warp takes a column at
//      a time, lane l the coefficients l + 32 k (row codes packed in registers);
//   2. W, Z and V run in place on X as m8n8k4 DMMAs; each phase's blocks (sub-blocks
//      merged block-diagonally where that costs no extra fragments: 17 per phase at
//      p = 15) are balanced over the warps; operator blocks are stored in DMMA
//      fragment order and read from L2 as coalesced 256-byte fragments;
//   3. each column is rotated back by e^{-i m alpha} and added to its target's
//      accumulators, which live in tensor memory (tcgen05.ld / tcgen05.st; warp w owns
//      target slots w, w + 8, ..., lane l the coefficients q = l + 32 k).
// At the end every target's local gets L += acc / |b|, once.  A target's entries are
// summed in (class, offset) order whatever the group composition: the result is
// bitwise reproducible run to run and identical between sharded and
// single-GPU applies, and no staging rows leave the SM (the round-1 offset-grouped
// kernel wrote and re-read 2 KB per List-2 entry: 95 GB per apply at config 1).
// Measured and not kept (profiles/r02_ncu_m2l.json): one CTA of 16 warps per SM with
// the multipoles and operators staged in shared memory by TMA bulk copies on
// mbarriers (44.8 vs 43.1 ms), register accumulators, double-buffered tiles with the
// gather overlapped in the phases, L1 prefetch of operator fragments.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "harmonics.cuh"
#include "kernels.cuh"
#include "../host/rotation.hpp"

namespace qbxg {
namespace dev {

namespace {

#ifndef QBXG_M2L_BN40
#define QBXG_M2L_BN40 1
#endif
constexpr int kPasPhases = 3;
constexpr int kWarps = 8, kNTh = kWarps * 32;  // two CTAs per SM
#ifndef QBXG_M2L_GATCOLS
#define QBXG_M2L_GATCOLS 1  // measured at config 1: 1 -> 36.1 ms, 2 -> 41.8 (spills), 3 -> 49.0; flat 4-deep gather 40.8
#endif
constexpr int kGatCols = QBXG_M2L_GATCOLS;       // columns a warp gathers at a time (KA loads each in flight per lane)
constexpr size_t kSmemMax = 232448 / 2 - 2048;  // two CTAs per SM (sm_100: 228 KB), less static

// per-phase operator size bound (doubles): blocks of sizes 1..p+1 (Re) and 1..p (Im),
// rows padded to 8 and columns to 4 -- the same multiset for W, Z and V (merging
// blocks, below, never makes a phase larger)
__host__ __device__ constexpr int pad_blk(int s) { return (s + 7) / 8 * 8 * ((s + 3) / 4 * 4); }
__host__ __device__ constexpr int phase_doubles(int p) {
  int t = 0;
  for (int s = 1; s <= p + 1; ++s) t += pad_blk(s);
  for (int s = 1; s <= p; ++s) t += pad_blk(s);
  return t;
}
// block table ints per phase (bound): [nblk][nblk+1 row offsets][nblk op offsets]
// [(p+1)^2 rows][kWarps+1 warp offsets][nblk block ids]
__host__ __device__ constexpr int tab_ints(int p) {
  return kPasPhases * (1 + 3 * (2 * p + 1) + 1 + (p + 1) * (p + 1) + kWarps + 1);
}
constexpr int kMaxBlock = 22;  // largest (merged) block the kernel instantiates

template <int P>
struct Tg {
  static constexpr int NR = hsize(P), NROW = (P + 1) * (P + 1), KP2 = 2 * NR;
  static constexpr int KA = (NR + 31) / 32;                // coefficients per lane in the accumulate
  static constexpr int TPW = 32 / KA < 6 ? 32 / KA : 6;    // target boxes per warp
  static constexpr int G = kWarps * TPW;                   // target boxes per CTA
  static constexpr int TW = 4 * KA;                        // TMEM words (columns) per target per lane
  // TMEM: warps w, w + 4 share lane quadrant w % 4, each its own column range
  static constexpr int TCOLS = (kWarps / 4) * TPW * TW;
  static constexpr int TALLOC = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128 : TCOLS <= 256 ? 256 : 512;
  static_assert(TCOLS <= 256, "TMEM accumulators exceed half of tensor memory");
  static constexpr size_t bytes(int bn) {
    return size_t(NROW + 1) * bn * 8              // X (+ a zero row), swizzled
           + size_t(2) * bn * (P + 1) * 16        // (cos, sin) per column, two tiles
           + size_t(6) * bn * 4                   // column meta, three tiles
           + size_t(tab_ints(P)) * 4;             // block table
  }
  static constexpr int BN = (QBXG_M2L_BN40 && bytes(40) <= kSmemMax) ? 40 : bytes(32) <= kSmemMax ? 32 : 16;  // tile columns
  static constexpr size_t SMEM = bytes(BN);
};

// X element (row r, column c) lives at r * BN + (c ^ swz<BN>(r)): the B-fragment loads
// (4 consecutive rows x 8 columns), the accumulate's reads (32 consecutive rows, one
// column) and the fragment stores all spread over the banks.  A row stride of 40 doubles
// already puts consecutive rows 8 banks apart, so only the low three column bits are
// permuted there (and column groups of 8 are reached by addition, not XOR).
template <int BN>
__device__ __forceinline__ int swz(int r) {
  if constexpr ((BN & (BN - 1)) == 0) return ((r & 1) << 3) | ((r >> 1) & 7);
  else return (r >> 1) & 7;
}
template <int BN>
__device__ __forceinline__ int col_group(int x, int j) {  // element x of column group 0 -> group j
  if constexpr ((BN & (BN - 1)) == 0) return x ^ (j * 8);
  else return x + j * 8;
}

struct TabHead {
  int base[kPasPhases];
};

// ---- PTX helpers: cp.async, DMMA, tensor memory
__device__ __forceinline__ unsigned sm_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sm_addr(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sm_addr(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// (x, y) or -(x, y): sign bits flipped by integer XOR
__device__ __forceinline__ double2 flip(double2 v, int neg) {
  const int sb = neg << 31;
  return make_double2(__hiloint2double(__double2hiint(v.x) ^ sb, __double2loint(v.x)),
                      __hiloint2double(__double2hiint(v.y) ^ sb, __double2loint(v.y)));
}

// TMEM: 4K consecutive 32-bit columns of this lane -> K (re, im) double pairs, one wait
template <int K>
__device__ __forceinline__ void tm_ld(unsigned ta, double* re, double* im) {
  unsigned r[4 * K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[4 * k]), "=r"(r[4 * k + 1]), "=r"(r[4 * k + 2]), "=r"(r[4 * k + 3])
                 : "r"(ta + 4 * k)
                 : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int k = 0; k < K; ++k) {
    re[k] = __hiloint2double(int(r[4 * k + 1]), int(r[4 * k]));
    im[k] = __hiloint2double(int(r[4 * k + 3]), int(r[4 * k + 2]));
  }
}
// TMEM: 4 consecutive 32-bit columns of this lane <- two doubles
__device__ __forceinline__ void tm_st4(unsigned ta, double x, double y) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(ta),
               "r"(__double2loint(x)), "r"(__double2hiint(x)), "r"(__double2loint(y)), "r"(__double2hiint(y))
               : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// One block of size S in place on the fp64 tensor pipe: the operator as A fragments
// (fragment order: 32 consecutive doubles per (mt, ks), zero padded) held in registers,
// then per 8-column tile j < nt the block's rows as B fragments from X (padding rows
// k >= S read the zero row), the DMMAs, and the rows written back.  Tile j's reads
// feed its DMMAs, which precede its writes; other tiles touch other columns.
template <int S, int BN, int ZR>
__device__ __forceinline__ void pas_block(double* X, const int* rw, const double* Ob, int lane, int nt, bool dual) {
  constexpr int MT = (S + 7) / 8, KS = (S + 3) / 4;
  double a[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[mt][ks] = Ob[(mt * KS + ks) * 32 + lane];
  // a dual block (Z of order m >= 1) applies the same fragments to a second row set
#pragma unroll 1
  for (int part = 0; part < (dual ? 2 : 1); ++part, rw += S) {
    int rb[KS], ro[MT];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + (lane & 3);
      const int t = k < S ? rw[k] : ZR * BN;  // row offset | swizzle << 16
      rb[ks] = (t & 0xffff) + ((lane >> 2) ^ (t >> 16));
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int i = mt * 8 + (lane >> 2);
      const int t = i < S ? rw[i] : -1;
      ro[mt] = t < 0 ? -1 : (t & 0xffff) + (((lane & 3) * 2) ^ (t >> 16));
    }
#pragma unroll 1
    for (int j = 0; j < nt; ++j) {
      double b[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) b[ks] = X[col_group<BN>(rb[ks], j)];
      double acc[MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma(acc[mt][0], acc[mt][1], a[mt][ks], b[ks]);
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
        if (ro[mt] >= 0) {
          X[col_group<BN>(ro[mt], j)] = acc[mt][0];
          X[col_group<BN>(ro[mt], j) ^ 1] = acc[mt][1];
        }
    }
  }
}

template <int P>
__global__ void __launch_bounds__(kNTh, 2)
    k_m2l_tg(const int* __restrict__ tab, int tab_n, TabHead hd, const double* __restrict__ ops, int op_stride,
             int phase_size, const double2* __restrict__ cs_all, const int* __restrict__ grp_order,
             const int* __restrict__ grp_tiles, const int* __restrict__ grp_box, const int4* __restrict__ tiles,
             const int* __restrict__ col_src, const int* __restrict__ col_meta, const double2* __restrict__ M,
             const double4* __restrict__ box, double* __restrict__ L) {
  using C = Tg<P>;
  constexpr int NR = C::NR, NROW = C::NROW, KP2 = C::KP2, BN = C::BN;
  constexpr int KA = C::KA, TPW = C::TPW, TW = C::TW;
  extern __shared__ __align__(16) unsigned char smem[];
  double* X = reinterpret_cast<double*>(smem);
  double2* s_cs = reinterpret_cast<double2*>(X + (NROW + 1) * BN);  // [2][BN][P+1]
  int* s_meta = reinterpret_cast<int*>(s_cs + 2 * BN * (P + 1));   // [3][BN]: target slot | offset << 8
  int* s_msrc = s_meta + 3 * BN;                                    // [3][BN]: source box
  int* s_tab = s_msrc + 3 * BN;
  __shared__ int s_code[NR];  // half-table q: Re row | Im row << 10 (zero row if m = 0) | m << 20
  __shared__ unsigned s_tmem;

  // (a parameter array indexed by a runtime phase would be copied to local memory)
  auto tab_base = [&](int ph) { return ph == 0 ? hd.base[0] : ph == 1 ? hd.base[1] : hd.base[2]; };
  const int g = grp_order[blockIdx.x];
  const int t_begin = grp_tiles[g], t_end = grp_tiles[g + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {  // accumulators of the group's target boxes live in tensor memory
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sm_addr(&s_tmem)),
                 "n"(C::TALLOC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  {  // block table; the blocks' row lists become X row offset | swizzle << 16
    int rs[kPasPhases];
#pragma unroll
    for (int ph = 0; ph < kPasPhases; ++ph) rs[ph] = hd.base[ph] + 2 + 2 * tab[hd.base[ph]];
    for (int i = tid; i < tab_n; i += kNTh) {
      int v = tab[i];
#pragma unroll
      for (int ph = 0; ph < kPasPhases; ++ph)
        if (i >= rs[ph] && i < rs[ph] + NROW) v = v * BN | swz<BN>(v) << 16;
      s_tab[i] = v;
    }
  }
  for (int q = tid; q < NR; q += kNTh) {
    int n = 0;
    while (hidx(n + 1, 0) <= q) ++n;
    const int m = q - hidx(n, 0);
    s_code[q] = q | (m > 0 ? NR + n * (n - 1) / 2 + m - 1 : NROW) << 10 | m << 20;
  }
  for (int c = tid; c < BN; c += kNTh) X[NROW * BN + c] = 0.0;
  // Tile metadata runs ahead by cp.async: column (slot | offset, source) two tiles
  // ahead (buffer it % 3), the columns' (cos, sin) rows one tile ahead (buffer it & 1),
  // so no thread waits on a global load between barriers.
  auto load_cols = [&](const int4 tl, int buf) {
    for (int i = tid; i < tl.z; i += kNTh) {
      cp_async4(s_meta + buf * BN + i, col_meta + tl.y + i);
      cp_async4(s_msrc + buf * BN + i, col_src + tl.y + i);
    }
  };
  auto load_cs = [&](int ncols, int mbuf, int cbuf) {
    double2* sc = s_cs + cbuf * BN * (P + 1);
    for (int i = tid; i < ncols * (P + 1); i += kNTh) {
      const int c = i / (P + 1), m = i - c * (P + 1);
      cp_async16(sc + i, cs_all + size_t((s_meta[mbuf * BN + c] & (kPasMirror - 1)) >> 8) * (P + 1) + m);
    }
  };
  int4 tl = make_int4(0, 0, 0, 0), tn = tl;
  if (t_begin < t_end) {
    tl = tiles[t_begin];
    load_cols(tl, 0);
    if (t_begin + 1 < t_end) {
      tn = tiles[t_begin + 1];
      load_cols(tn, 1);
    }
  }
  cp_async_wait_all();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (t_begin < t_end) load_cs(tl.z, 0, 0);
  // lane l owns the half-table coefficients q = l + 32 k in the gather and the accumulate:
  // X row offset | swizzle << 16 (| m << 20) of their Re and Im rows (Im of m = 0: zero row)
  int q_re[KA], q_im[KA];
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const int q = lane + 32 * k;
    const int code = q < NR ? s_code[q] : (NROW | NROW << 10);
    const int re = code & 1023, im = (code >> 10) & 1023, m = code >> 20;
    int n = 0;
    while (q < NR && hidx(n + 1, 0) <= q) ++n;
    q_re[k] = re * BN | swz<BN>(re) << 16 | m << 20 | ((n + m) & 1) << 25;  // bit 25: sign under z -> -z
    q_im[k] = im * BN | swz<BN>(im) << 16;
  }
  // this warp's accumulators: lane quadrant warp % 4, columns of its TPW targets
  const unsigned tm = s_tmem + (unsigned(32 * (warp & 3)) << 16) + unsigned((warp >> 2) * TPW * TW);
#pragma unroll 1
  for (int w = 0; w < TPW * KA; ++w) tm_st4(tm + 4 * w, 0.0, 0.0);
  tm_wait_st();
  cp_async_wait_all();
  __syncthreads();

#pragma unroll 1
  for (int t = t_begin, it = 0; t < t_end; ++t, ++it) {
    const bool more = t + 1 < t_end;
    const int4 tn2 = t + 2 < t_end ? tiles[t + 2] : make_int4(0, 0, 0, 0);
    const int ncols = tl.z, nt = (ncols + 7) >> 3;
    const int mb = it % 3, mb1 = (it + 1) % 3, mb2 = (it + 2) % 3, cb = it & 1;
    const int* sm = s_meta + mb * BN;
    const double2* sc = s_cs + cb * BN * (P + 1);
    {  // 1. multipoles straight from L2, rotated by e^{i k alpha} into X: a warp takes
       // kGatCols columns at a time, lane l the coefficients q = l + 32 k (coalesced
       // 512-byte reads, all of them in flight before the first use)
      const int* src = s_msrc + mb * BN;
#pragma unroll 1
      for (int c0 = warp * kGatCols; c0 < ncols; c0 += kWarps * kGatCols) {
        double2 v[kGatCols][KA];
#pragma unroll
        for (int u = 0; u < kGatCols; ++u)
          if (c0 + u < ncols) {
            const double2* Mb = M + size_t(src[c0 + u]) * NR + lane;
#pragma unroll
            for (int k = 0; k < KA; ++k)
              if (lane + 32 * k < NR) v[u][k] = __ldg(Mb + 32 * k);
          }
#pragma unroll
        for (int u = 0; u < kGatCols; ++u)
          if (c0 + u < ncols) {
            const int c = c0 + u;
            const double2* rc = sc + c * (P + 1);
            const int mir = (sm[c] >> 30) & 1;  // offset below the xy-plane: M_n^m -> (-1)^{n+m} M_n^m
#pragma unroll
            for (int k = 0; k < KA; ++k)
              if (lane + 32 * k < NR) {
                const int m = (q_re[k] >> 20) & 31;
                const double2 r = flip(rc[m], (q_re[k] >> 25) & mir);
                X[(q_re[k] & 0xffff) + (c ^ ((q_re[k] >> 16) & 15))] = v[u][k].x * r.x - v[u][k].y * r.y;
                if (m) X[(q_im[k] & 0xffff) + (c ^ (q_im[k] >> 16))] = v[u][k].x * r.y + v[u][k].y * r.x;
              }
          }
      }
    }
    __syncthreads();
    if (more) {  // the next tiles' metadata in flight
      load_cs(tn.z, mb1, cb ^ 1);
      if (t + 2 < t_end) load_cols(tn2, mb2);
    }
    // 2. W, Z, V in place
#pragma unroll 1
    for (int ph = 0; ph < kPasPhases; ++ph) {
      if (tl.w && ph != 1) continue;  // offset along +z (after mirroring): the rotations are the identity
      const double* Op = ops + size_t(tl.x) * op_stride + size_t(ph) * phase_size;
      const int* T = s_tab + tab_base(ph);
      const int nblk = T[0];
      const int* rowoff = T + 1;
      const int* opoff = rowoff + nblk + 1;
      const int* rows = opoff + nblk;
      const int* woff = rows + NROW;
      const int* wblk = woff + kWarps + 1;
#define QBXG_PAS_CASE(S) \
  case S:                \
    if (S <= kMaxBlock) pas_block<S, BN, NROW>(X, rw, Ob, lane, nt, dual); \
    break;
      const int i_end = woff[warp + 1];
#pragma unroll 1
      for (int i = woff[warp]; i < i_end; ++i) {
        const int b = wblk[i];
        const int* rw = rows + rowoff[b];
        const double* Ob = Op + opoff[b];
        const bool dual = ph == 1 && b > 0;  // Z of order m >= 1: Re rows, then Im rows
        switch ((rowoff[b + 1] - rowoff[b]) >> (dual ? 1 : 0)) {
          QBXG_PAS_CASE(1) QBXG_PAS_CASE(2) QBXG_PAS_CASE(3) QBXG_PAS_CASE(4) QBXG_PAS_CASE(5) QBXG_PAS_CASE(6)
          QBXG_PAS_CASE(7) QBXG_PAS_CASE(8) QBXG_PAS_CASE(9) QBXG_PAS_CASE(10) QBXG_PAS_CASE(11)
          QBXG_PAS_CASE(12) QBXG_PAS_CASE(13) QBXG_PAS_CASE(14) QBXG_PAS_CASE(15) QBXG_PAS_CASE(16)
          QBXG_PAS_CASE(17) QBXG_PAS_CASE(18) QBXG_PAS_CASE(19) QBXG_PAS_CASE(20) QBXG_PAS_CASE(21)
          QBXG_PAS_CASE(22)
          default: break;
        }
      }
#undef QBXG_PAS_CASE
      __syncthreads();
    }
    // 3. rotate back by e^{-i m alpha} and add to the owning warp's accumulators (TMEM),
    // in column order; a target's columns are consecutive, so its accumulators are read
    // and written once per tile
    {
#pragma unroll 1
      for (int cb = 0; cb < ncols; cb += 32) {  // (BN may exceed the 32 lanes of the ballot)
        const int mine = cb + lane < ncols && ((sm[cb + lane] & 255) % kWarps) == warp;
        unsigned mask = __ballot_sync(0xffffffffu, mine);
        if (cb && mask) tm_wait_st();  // a target's run may continue from the previous 32 columns
        while (mask) {
          const int slot = sm[cb + __ffs(mask) - 1] & 255, u = slot / kWarps;
          double are[KA], aim[KA];
          tm_ld<KA>(tm + u * TW, are, aim);
          while (mask && (sm[cb + __ffs(mask) - 1] & 255) == slot) {
            const int c = cb + __ffs(mask) - 1;
            mask &= mask - 1;
            const double2* r = sc + c * (P + 1);
            const int mir = (sm[c] >> 30) & 1;  // L_n^m <- (-1)^{n+m} L_n^m of the mirrored translation
#pragma unroll
            for (int k = 0; k < KA; ++k) {
              const double xr = X[(q_re[k] & 0xffff) + (c ^ ((q_re[k] >> 16) & 15))];
              const double xi = X[(q_im[k] & 0xffff) + (c ^ (q_im[k] >> 16))];
              const double2 rr = flip(r[(q_re[k] >> 20) & 31], (q_re[k] >> 25) & mir);
              are[k] += xr * rr.x + xi * rr.y;
              aim[k] += xi * rr.x - xr * rr.y;
            }
          }
#pragma unroll
          for (int k = 0; k < KA; ++k) tm_st4(tm + (u * KA + k) * 4, are[k], aim[k]);
        }
      }
      tm_wait_st();  // each run wrote a different target's columns; one wait for all
    }
    cp_async_wait_all();  // next tiles' metadata landed
    __syncthreads();      // X and this tile's buffers free
    tl = tn;
    tn = tn2;
  }
#pragma unroll 1
  for (int u = 0; u < TPW; ++u) {
    const int b = grp_box[size_t(g) * C::G + u * kWarps + warp];
    if (b < 0) continue;
    const double ih = 1.0 / box[b].w;
    double* Lb = L + size_t(b) * KP2;
    double xr[KA], xi[KA];
    tm_ld<KA>(tm + u * TW, xr, xi);
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const int q = lane + 32 * k;
      if (q < NR) {
        Lb[2 * q] += xr[k] * ih;
        if (s_code[q] >> 20) Lb[2 * q + 1] += xi[k] * ih;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem), "n"(C::TALLOC) : "memory");
}

// ---------------------------------------------------------------- host side
// sub-blocks of one phase as storage rows (Re rows hidx(n, m); Im rows
// NR + n(n-1)/2 + m - 1): W, V per degree a (orders part..a), Z per order a
// (degrees a..p), part 0 = Re, 1 = Im
struct SubBlock {
  int part, a;
  std::vector<int> rows;
  std::vector<int> rows2;  // Z phase, m >= 1: the Im rows that take the same operator (dual block)
};
std::vector<SubBlock> phase_subblocks(int p, int ph) {
  const int NR = hsize(p);
  auto re = [&](int n, int m) { return hidx(n, m); };
  auto im = [&](int n, int m) { return NR + n * (n - 1) / 2 + m - 1; };
  std::vector<SubBlock> out;
  if (ph == 1) {
    // Z_m is the same for the Re and the Im rows of order m: sub-block m >= 1 is dual (its
    // operator fragments are loaded once and applied to both row sets); m = 0 has Re rows only
    for (int a = 0; a <= p; ++a) {
      SubBlock b{0, a, {}, {}};
      for (int n = a; n <= p; ++n) {
        b.rows.push_back(re(n, a));
        if (a > 0) b.rows2.push_back(im(n, a));
      }
      out.push_back(b);
    }
    return out;
  }
  for (int part = 0; part < 2; ++part)
    for (int a = part; a <= p; ++a) {
      SubBlock b{part, a, {}, {}};
      for (int m = part; m <= a; ++m) b.rows.push_back(part ? im(a, m) : re(a, m));
      out.push_back(b);
    }
  return out;
}

// Merged blocks: sub-blocks placed block-diagonally in one operator when that costs no
// more DMMA fragments than running them apart (the padding of a large block absorbs a
// small one), so a phase is ~17 near-square blocks instead of 2p + 1 at p = 15.
// (a sub-block without a second row set is never merged with dual ones)
std::vector<std::vector<int>> merge_subblocks(const std::vector<SubBlock>& sb) {
  std::vector<int> order(sb.size());
  for (size_t i = 0; i < sb.size(); ++i) order[i] = int(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sb[a].rows.size() > sb[b].rows.size(); });
  std::vector<char> used(sb.size(), 0);
  std::vector<std::vector<int>> groups;
  // (merged sizes may exceed 2p + 2 when several small blocks chain: every size up to
  // kMaxBlock is instantiated)
  for (int i : order) {
    if (used[i]) continue;
    used[i] = 1;
    std::vector<int> gr{i};
    int s = int(sb[i].rows.size()), cost = pad_blk(s);
    for (bool grew = true; grew;) {
      grew = false;
      for (int j : order) {  // largest sub-block that fits for free
        if (used[j]) continue;
        const int u = int(sb[j].rows.size());
        if (sb[j].rows2.empty() != sb[i].rows2.empty()) continue;
        if (s + u > kMaxBlock || pad_blk(s + u) > cost + pad_blk(u)) continue;
        used[j] = 1;
        gr.push_back(j);
        s += u;
        cost = pad_blk(s);
        grew = true;
        break;
      }
    }
    groups.push_back(gr);
  }
  return groups;
}

struct PasLayout {
  int phase_size = 0;
  std::vector<int> tab;
  TabHead hd{};
  std::vector<std::vector<SubBlock>> sub;             // per phase
  std::vector<std::vector<std::vector<int>>> groups;  // per phase: merged blocks
  std::vector<std::vector<int>> opoff;                // per phase
};

PasLayout make_layout(int p) {
  PasLayout L;
  L.sub.resize(kPasPhases);
  L.groups.resize(kPasPhases);
  L.opoff.resize(kPasPhases);
  for (int ph = 0; ph < kPasPhases; ++ph) {
    L.sub[ph] = phase_subblocks(p, ph);
    L.groups[ph] = merge_subblocks(L.sub[ph]);
    const auto& G = L.groups[ph];
    const int nblk = int(G.size());
    L.hd.base[ph] = int(L.tab.size());
    std::vector<int> rowoff{0}, rows, sizes;
    int oo = 0;
    std::vector<char> dual;
    for (const auto& gr : G) {
      int sz = 0;
      for (int i : gr) {
        rows.insert(rows.end(), L.sub[ph][i].rows.begin(), L.sub[ph][i].rows.end());
        sz += int(L.sub[ph][i].rows.size());
      }
      // a dual block lists its second row set after the first (the kernel runs the block
      // twice with the operator fragments in registers)
      dual.push_back(!L.sub[ph][gr[0]].rows2.empty());
      for (int i : gr) rows.insert(rows.end(), L.sub[ph][i].rows2.begin(), L.sub[ph][i].rows2.end());
      rowoff.push_back(int(rows.size()));
      sizes.push_back(sz);
      L.opoff[ph].push_back(oo);
      oo += pad_blk(sz);
    }
    // the kernel tells dual blocks by position: Z phase, every block but the first
    for (int b = 0; b < nblk; ++b)
      if (bool(dual[b]) != (ph == 1 && b > 0)) throw std::logic_error("m2l_pas: unexpected dual block order");
    L.phase_size = std::max(L.phase_size, oo);
    // whole blocks per warp, longest processing time first; a block costs its DMMA
    // fragments plus a fixed latency share
    std::vector<int> order(nblk);
    for (int i = 0; i < nblk; ++i) order[i] = i;
    auto cost = [&](int b) { return long(pad_blk(sizes[b])) * (dual[b] ? 2 : 1) + 96; };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
    std::vector<std::vector<int>> wl(kWarps);
    std::vector<long> load(kWarps, 0);
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
    L.tab.push_back(nblk);
    for (auto* v : {&rowoff, &L.opoff[ph], &rows, &woff, &wblk}) L.tab.insert(L.tab.end(), v->begin(), v->end());
  }
  if (int(L.tab.size()) > tab_ints(p) || L.phase_size > phase_doubles(p))
    throw std::logic_error("m2l_pas: block table exceeds its bound");
  return L;
}

template <int P>
int tg_launch(const M2LPlan& Pl, const DevData& D, cudaStream_t s) {
  using C = Tg<P>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_m2l_tg<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)) != cudaSuccess)
      return -1;
    attr = true;
  }
  TabHead hd;
  for (int k = 0; k < 3; ++k) hd.base[k] = Pl.pas_base[k];
  k_m2l_tg<P><<<Pl.n_groups, kNTh, C::SMEM, s>>>(Pl.pas_tab, Pl.pas_tab_n, hd, Pl.pas_ops, Pl.pas_stride,
                                                   Pl.pas_phase, Pl.cs, Pl.grp_order, Pl.grp_tiles, Pl.grp_box,
                                                   Pl.tiles, Pl.col_src, Pl.col_meta,
                                                   D.M, D.box,
                                                   reinterpret_cast<double*>(D.L));
  return 1;
}

#define QBXG_PAS_ORDERS(X)                                                                                   \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18) X(19) \
      X(20) X(21)

}  // namespace

bool pas_supported(int p) { return p >= 1 && p <= kMaxPasOrder; }

int pas_tile_cols(int p) {
  switch (p) {
#define QBXG_TG_BN(N) \
  case N:             \
    return Tg<N>::BN;
    QBXG_PAS_ORDERS(QBXG_TG_BN)
#undef QBXG_TG_BN
    default: return 0;
  }
}

int pas_group_size(int p) {
  switch (p) {
#define QBXG_TG_G(N) \
  case N:            \
    return Tg<N>::G;
    QBXG_PAS_ORDERS(QBXG_TG_G)
#undef QBXG_TG_G
    default: return 0;
  }
}

// Per-class operators [W | Z | V], blocks in phase_blocks order, each stored in DMMA
// A-fragment order: for every (row tile mt, k step ks) the 32 lanes' elements
// A[8 mt + lane/4][4 ks + lane%4] are consecutive (rows padded to 8 and columns to 4
// with zeros).  A class is (rho_xy^2, dz); v' = (2 rho_xy, 0, 2 dz) is the same for all
// its offsets.
void pas_build_ops(int p, int n_cls, const int* cls_rxy2, const int* cls_dz, std::vector<double>& ops,
                   int& op_stride, std::vector<int>& tab, int& nblk, int& phase_size, int (&base)[3]) {
  const PasLayout L = make_layout(p);
  nblk = int(L.groups[0].size());
  phase_size = L.phase_size;
  op_stride = kPasPhases * L.phase_size;
  tab = L.tab;
  for (int k = 0; k < 3; ++k) base[k] = L.hd.base[k];
  ops.assign(size_t(n_cls) * op_stride, 0.0);
  const size_t rs = rot_blocks_size(p);
  // element (i, k) of a block with padded column count sp, in fragment order
  auto frag = [](int i, int k, int sp) {
    const int ks_n = sp / 4, mt = i / 8, ks = k / 4, lane = (i % 8) * 4 + k % 4;
    return size_t(mt * ks_n + ks) * 32 + lane;
  };
  auto re = [](int m) { return m == 0 ? 0 : 2 * m - 1; };
  auto im = [](int m) { return 2 * m; };
  double worst = 0.0;
#pragma omp parallel for schedule(dynamic, 4) reduction(max : worst)
  for (int o = 0; o < n_cls; ++o) {
    const double v[3] = {2.0 * std::sqrt(double(cls_rxy2[o])), 0.0, 2.0 * cls_dz[o]};
    const double rho = std::sqrt(v[0] * v[0] + v[2] * v[2]);
    std::vector<double> Rf(rs), Rb(rs);
    m2l_rotation_blocks(p, v, Rf.data(), Rb.data());
    for (int a = 0; a <= p; ++a) {  // Re/Im cross terms vanish at phi = 0
      const int d = 2 * a + 1;
      const double* F = &Rf[rot_block_offset(a)];
      const double* B = &Rb[rot_block_offset(a)];
      for (int i = 0; i <= a; ++i)
        for (int k = 1; k <= a; ++k) {
          worst = std::max(worst, std::fabs(F[re(i) * d + im(k)]) + std::fabs(F[im(k) * d + re(i)]));
          worst = std::max(worst, std::fabs(B[re(i) * d + im(k)]) + std::fabs(B[im(k) * d + re(i)]));
        }
    }
    for (int ph = 0; ph < kPasPhases; ++ph) {
      double* Op = &ops[size_t(o) * op_stride + size_t(ph) * L.phase_size];
      const auto& sub = L.sub[ph];
      for (size_t b = 0; b < L.groups[ph].size(); ++b) {
        const auto& gr = L.groups[ph][b];
        int S = 0;
        for (int i : gr) S += int(sub[i].rows.size());
        const int sp = (S + 3) / 4 * 4;
        double* Ob = Op + L.opoff[ph][b];
        int off = 0;  // sub-blocks block-diagonally
        for (int si : gr) {
          const int part = sub[si].part, a = sub[si].a, sz = int(sub[si].rows.size());
          for (int i = 0; i < sz; ++i)
            for (int k = 0; k < sz; ++k) {
              double val;
              if (ph != 1) {  // W (rotation of the multipole), V (back-rotation of the local)
                const int d = 2 * a + 1, mi = part + i, mk = part + k;
                const int ri = part ? im(mi) : re(mi), rk = part ? im(mk) : re(mk);
                val = (ph == 0 ? Rf : Rb)[rot_block_offset(a) + size_t(ri) * d + rk];
              } else {  // Z: order m = a, rows n / columns j in [m, p]: (-1)^{n+m} (j+n)! / rho^{j+n+1}
                const int m = a, n = m + i, j = m + k;
                double f = 1.0;
                for (int t = 2; t <= j + n; ++t) f *= t;
                val = (((n + m) & 1) ? -1.0 : 1.0) * f / std::pow(rho, j + n + 1);
              }
              Ob[frag(off + i, off + k, sp)] = val;
            }
          off += sz;
        }
      }
    }
  }
  if (worst > 1e-12) throw std::runtime_error("pas_build_ops: rotation blocks mix Re and Im at phi = 0");
}

int launch_m2l(const M2LPlan& P, const DevData& D, cudaStream_t s) {
  if (P.n_groups == 0) return 0;
  switch (D.p) {
#define QBXG_TG_P(N) \
  case N:            \
    return tg_launch<N>(P, D, s);
    QBXG_PAS_ORDERS(QBXG_TG_P)
#undef QBXG_TG_P
    default: return -1;
  }
}

}  // namespace dev
}  // namespace qbxg
