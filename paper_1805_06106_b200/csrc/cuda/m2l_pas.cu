// Stage 4 M2L (List 2) as point-and-shoot translations on real
// half-table blocks.
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
// azimuthal blocks.  W, Z and V depend on (rho_xy^2, dz) only: the 1,206 offsets of
// [-5,5]^3 fall into 190 classes, so one operator set per class (~19 MB at p = 15).
//
// Kernel: one CTA = one offset x <= 32 List-2 entries (3 CTAs per SM).  The gathered,
// alpha-rotated multipoles sit in shared memory as (p+1)^2 rows (Re in half-table order,
// Im in compacted order) x 32 columns.  In each phase every warp owns a fixed list of
// whole blocks (longest processing time balanced on the host), so the phase runs in
// place: the warp reads a block's operator (A fragments, from L2) and its rows (B
// fragments, from shared memory) into registers, runs the m8n8k4 DMMAs, then writes its
// rows.  Each entry's output row (still in the offset's frame) goes to a staging row at
// its List-2 CSR position; k_m2l_reduce then rotates each row back by alpha and sums a
// box's rows in CSR order (fixed order: bitwise reproducible), x 1/|b|.
//
// Measured and not kept (profiles/r02_summary.md): fusing the reduction into this kernel
// (target-superblock tile order, per-entry alpha, last-arriving CTA reduces from L2):
// 50-55 ms vs 43 at config 1 -- the kernel is latency-bound, and the per-entry rotations
// and the 1.17x tiles cost more than the 37 GB staging round trip they save; a fully
// unrolled compile-time block schedule per warp: 30% fewer instructions but 49 ms, half
// the warp stalls on instruction fetch (the per-warp code no longer fits the I-cache).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "harmonics.cuh"
#include "kernels.cuh"
#include "../host/rotation.hpp"

namespace qbxg {
namespace dev {

namespace {

constexpr int kPasPhases = 3;
constexpr int kWarps = 8, kBN = 32, kLD = kBN + 1, kNTh = kWarps * 32;

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

// One block of size S in place on the fp64 tensor pipe: the operator (rows padded to
// 8, columns to 4, zeros) as A fragments from L2, the block's rows x the tile's first
// 8*NT columns as B fragments from shared memory -- all read before any row is
// written, so the warp may overwrite its own block.
template <int S, int NT>
__device__ __forceinline__ void pas_block(double* X, const int* rw, const double* __restrict__ Ob, int lane) {
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
    for (int nt = 0; nt < NT; ++nt) b[ks][nt] = k < S ? X[row * kLD + nt * 8 + (lane >> 2)] : 0.0;
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
        X[row * kLD + nt * 8 + (lane & 3) * 2] = acc[mt][nt][0];
        X[row * kLD + nt * 8 + (lane & 3) * 2 + 1] = acc[mt][nt][1];
      }
    }
  }
}

template <int P>
__global__ void __launch_bounds__(kNTh, P <= 15 ? 3 : (P <= 18 ? 2 : 1))
    k_m2l_pas(const int* __restrict__ tab, int tab_n, TabHead hd, int nblk, const double* __restrict__ ops,
              int op_stride, int phase_size, const double2* __restrict__ cs_all, const int4* __restrict__ tiles,
              const int* __restrict__ col_src, const int* __restrict__ col_pos, const double* __restrict__ M, int kp2,
              int row_stride, double* __restrict__ temp) {
  constexpr int NR = hsize(P), NROW = (P + 1) * (P + 1);
  extern __shared__ double smem[];
  double* X = smem;
  int* s_tab = reinterpret_cast<int*>(X + NROW * kLD);
  __shared__ int s_src[kBN];
  __shared__ int s_pos[kBN];
  __shared__ double2 s_cs[P + 1];
  // half-table index q: Re row | Im row << 10 (0 for m = 0) | m << 20
  __shared__ int s_code[NR];
  const int4 tile = tiles[blockIdx.x];  // (offset, first column, columns, class)
  const int ncol = tile.z;
  const bool half = ncol <= kBN / 2;  // tiles of <= 16 columns run 2 of the 4 DMMA n-tiles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < tab_n; i += kNTh) s_tab[i] = tab[i];
  if (tid < kBN) s_src[tid] = tid < ncol ? col_src[tile.y + tid] : -1;
  if (tid < kBN) s_pos[tid] = tid < ncol ? col_pos[tile.y + tid] : -1;
  if (tid <= P) s_cs[tid] = cs_all[size_t(tile.x) * (P + 1) + tid];
  for (int q = tid; q < NR; q += kNTh) {
    int n = 0;
    while (hidx(n + 1, 0) <= q) ++n;
    const int m = q - hidx(n, 0);
    s_code[q] = q | (m > 0 ? NR + n * (n - 1) / 2 + m - 1 : 0) << 10 | m << 20;
  }
  __syncthreads();
  // gather M' = M e^{i k alpha}, coalesced along each multipole, kSt loads in flight per
  // thread; columns past the tile are zero
  constexpr int kSt = 6;
  const int nel = NR * (half ? kBN / 2 : kBN);
  for (int e0 = 0; e0 < nel; e0 += kSt * kNTh) {
    double2 v[kSt];
#pragma unroll
    for (int u = 0; u < kSt; ++u) {
      const int e = e0 + tid + u * kNTh;
      v[u] = make_double2(0.0, 0.0);
      if (e < nel) {
        const int c = e / NR, q = e - c * NR;
        const int src = s_src[c];
        if (src >= 0) v[u] = __ldg(reinterpret_cast<const double2*>(M + size_t(src) * kp2) + q);
      }
    }
#pragma unroll
    for (int u = 0; u < kSt; ++u) {
      const int e = e0 + tid + u * kNTh;
      if (e < nel) {
        const int c = e / NR, q = e - c * NR;
        const int code = s_code[q], ri = (code >> 10) & 1023;
        const double2 r = s_cs[(code >> 20) & 63];
        X[(code & 1023) * kLD + c] = v[u].x * r.x - v[u].y * r.y;
        if (ri) X[ri * kLD + c] = v[u].x * r.y + v[u].y * r.x;
      }
    }
  }
  __syncthreads();
  const double* opb = ops + size_t(tile.w) * op_stride;
#pragma unroll 1
  for (int ph = 0; ph < kPasPhases; ++ph) {
    const int* T = s_tab + hd.base[ph];
    const int* rowoff = T;
    const int* opoff = T + nblk + 1;
    const int* rows = opoff + nblk;
    const int* woff = rows + NROW;
    const int* wblk = woff + kWarps + 1;
    const double* Op = opb + size_t(ph) * phase_size;
#define QBXG_PAS_CASES(NT)                                                                                     \
  QBXG_PAS_CASE(1, NT) QBXG_PAS_CASE(2, NT) QBXG_PAS_CASE(3, NT) QBXG_PAS_CASE(4, NT) QBXG_PAS_CASE(5, NT)         \
  QBXG_PAS_CASE(6, NT) QBXG_PAS_CASE(7, NT) QBXG_PAS_CASE(8, NT) QBXG_PAS_CASE(9, NT) QBXG_PAS_CASE(10, NT)        \
  QBXG_PAS_CASE(11, NT) QBXG_PAS_CASE(12, NT) QBXG_PAS_CASE(13, NT) QBXG_PAS_CASE(14, NT) QBXG_PAS_CASE(15, NT)    \
  QBXG_PAS_CASE(16, NT) QBXG_PAS_CASE(17, NT) QBXG_PAS_CASE(18, NT) QBXG_PAS_CASE(19, NT) QBXG_PAS_CASE(20, NT)    \
  QBXG_PAS_CASE(21, NT) QBXG_PAS_CASE(22, NT)
#define QBXG_PAS_CASE(S, NT) \
  case S:                    \
    if (S <= P + 1) pas_block<S, NT>(X, rw, Ob, lane); \
    break;
#pragma unroll 1
    for (int i = woff[warp]; i < woff[warp + 1]; ++i) {
      const int b = wblk[i];
      const int* rw = rows + rowoff[b];
      const double* Ob = Op + opoff[b];
      if (half) {
        switch (rowoff[b + 1] - rowoff[b]) {
          QBXG_PAS_CASES(2)
          default: break;
        }
      } else {
        switch (rowoff[b + 1] - rowoff[b]) {
          QBXG_PAS_CASES(4)
          default: break;
        }
      }
    }
#undef QBXG_PAS_CASE
#undef QBXG_PAS_CASES
    __syncthreads();
  }
  // staging row = Re (NR) then compacted Im, coalesced along each row (row-outer: one
  // row per thread and column; consecutive lanes, consecutive rows); streaming stores,
  // so the rows do not evict the multipoles and operators from L2
  for (int r = tid; r < NROW; r += kNTh)
    for (int c = 0; c < ncol; ++c) __stcs(temp + size_t(s_pos[c]) * row_stride + r, X[r * kLD + c]);
}

// Each staging row holds L' of one List-2 entry in its offset's rotated frame (Re rows
// in half-table order, then compacted Im rows).  Rotate back (L = L' e^{-i m alpha}) and
// sum a box's rows in CSR order; scale by 1/|b| once.
__global__ void __launch_bounds__(160) k_m2l_reduce(const int* __restrict__ boxes, const int64_t* __restrict__ v_starts,
                                                    const int* __restrict__ ent_op, const double2* __restrict__ cs,
                                                    int p, int row_stride, int64_t chunk_base,
                                                    const double* __restrict__ temp, const double4* __restrict__ box,
                                                    double* __restrict__ L, int kp2) {
  const int b = boxes[blockIdx.x];
  const int64_t a = v_starts[b], e = v_starts[b + 1];
  const int NR = hsize(p);
  const double ih = 1.0 / box[b].w;
  for (int q = threadIdx.x; q < NR; q += blockDim.x) {
    int n = int((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while (hidx(n + 1, 0) <= q) ++n;
    while (hidx(n, 0) > q) --n;
    const int m = q - hidx(n, 0);
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
        const double* row = temp + (pos + u - chunk_base) * row_stride;
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
      const double* row = temp + (pos - chunk_base) * row_stride;
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

// ---------------------------------------------------------------- host side
struct PasLayout {
  int nblk = 0, phase_size = 0;
  std::vector<int> tab;
  TabHead hd{};
};

// blocks of one phase as storage rows (Re rows hidx(n, m); Im rows NR + n(n-1)/2 + m - 1)
void phase_blocks(int p, int ph, std::vector<std::vector<int>>& blocks) {
  const int NR = hsize(p);
  auto re = [&](int n, int m) { return hidx(n, m); };
  auto im = [&](int n, int m) { return NR + n * (n - 1) / 2 + m - 1; };
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

PasLayout make_layout(int p) {
  PasLayout L;
  for (int ph = 0; ph < kPasPhases; ++ph) {
    std::vector<std::vector<int>> blocks;
    phase_blocks(p, ph, blocks);
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

template <int P>
int pas_launch_p(const M2LPlan& Pl, const M2LChunk& C, const double* X, int kp2, double* stage, cudaStream_t s) {
  constexpr int NROW = (P + 1) * (P + 1);
  const size_t smem = size_t(NROW * kLD) * sizeof(double) + size_t(Pl.pas_tab_n) * sizeof(int);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_m2l_pas<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
      return -1;
    attr = smem;
  }
  TabHead hd;
  for (int k = 0; k < 3; ++k) hd.base[k] = Pl.pas_base[k];
  k_m2l_pas<P><<<C.n_tiles, kNTh, smem, s>>>(Pl.pas_tab, Pl.pas_tab_n, hd, Pl.pas_nblk, Pl.pas_ops, Pl.pas_stride,
                                             Pl.pas_phase, Pl.cs, C.tiles, C.col_src, C.col_pos, X, kp2, Pl.srow,
                                             stage);
  return 1;
}

}  // namespace

bool pas_supported(int p) { return p >= 1 && p <= kMaxPasOrder; }
int pas_tile_cols() { return kBN; }

// Per-class operators [W | Z | V], blocks in phase_blocks order, each row-major with
// rows padded to 8 and columns to 4 (zeros): DMMA A fragments without guards.  A
// class is (rho_xy^2, dz); v' = (2 rho_xy, 0, 2 dz) is the same for all its offsets.
void pas_build_ops(int p, int n_cls, const int* cls_rxy2, const int* cls_dz, std::vector<double>& ops,
                   int& op_stride, std::vector<int>& tab, int& nblk, int& phase_size, int (&base)[3]) {
  const PasLayout L = make_layout(p);
  nblk = L.nblk;
  phase_size = L.phase_size;
  op_stride = kPasPhases * L.phase_size;
  tab = L.tab;
  for (int k = 0; k < 3; ++k) base[k] = L.hd.base[k];
  ops.assign(size_t(n_cls) * op_stride, 0.0);
  const size_t rs = rot_blocks_size(p);
  double worst = 0.0;
#pragma omp parallel for schedule(dynamic, 4) reduction(max : worst)
  for (int o = 0; o < n_cls; ++o) {
    const double v[3] = {2.0 * std::sqrt(double(cls_rxy2[o])), 0.0, 2.0 * cls_dz[o]};
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
}

int launch_m2l_pas(const M2LPlan& P, const M2LChunk& C, const DevData& D, double* stage, cudaStream_t s) {
  const double* X = reinterpret_cast<const double*>(D.M);
  const int kp2 = 2 * D.kp;
  int r = -1;
  switch (D.p) {
#define QBXG_PAS_P(N) \
  case N:             \
    r = pas_launch_p<N>(P, C, X, kp2, stage, s); \
    break;
    QBXG_PAS_P(1) QBXG_PAS_P(2) QBXG_PAS_P(3) QBXG_PAS_P(4) QBXG_PAS_P(5) QBXG_PAS_P(6) QBXG_PAS_P(7)
    QBXG_PAS_P(8) QBXG_PAS_P(9) QBXG_PAS_P(10) QBXG_PAS_P(11) QBXG_PAS_P(12) QBXG_PAS_P(13) QBXG_PAS_P(14)
    QBXG_PAS_P(15) QBXG_PAS_P(16) QBXG_PAS_P(17) QBXG_PAS_P(18) QBXG_PAS_P(19) QBXG_PAS_P(20) QBXG_PAS_P(21)
#undef QBXG_PAS_P
    default: return -1;
  }
  return r;
}

int launch_m2l_reduce(const M2LPlan& P, const M2LChunk& C, const DevData& D, const double* stage, cudaStream_t s) {
  if (C.n_boxes == 0) return 0;
  k_m2l_reduce<<<C.n_boxes, 160, 0, s>>>(C.boxes, D.v_starts, P.ent_op, P.cs, D.p, P.srow, C.base, stage, D.box,
                                         reinterpret_cast<double*>(D.L), 2 * D.kp);
  return 1;
}

}  // namespace dev
}  // namespace qbxg
