// Kernel interface shared by the stage kernels (kernels.cu) and the device
// handle (handle.cu).  One struct of device pointers, passed by value.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace qbxg {
namespace dev {

struct DevData {
  int p, q;          // FMM / QBX order
  int kp, kq;        // half-table sizes hsize(p), hsize(q)
  int ktab_m2l;      // hsize(2p): M2L offset table row length
  int dipole;        // 1 for Laplace SL+DL
  // tree (DFS-preorder boxes)
  const double4* box;  // (cx, cy, cz, |b|)
  const int* child_starts;
  const int* children;
  const int* parent;
  const int* src_own_start;
  const int* src_own_count;
  const int* ctr_own_start;
  const int* ctr_own_count;
  const int* tgt_own_start;
  const int* tgt_own_count;
  // box-sorted particles
  double4* src;        // (x, y, z, w)
  double4* mu;         // (mx, my, mz, 0) or null
  const double4* ctr;  // (x, y, z, r)
  const double4* tgt;  // conventional targets (x, y, z, 0)
  // expansions
  double2* M;   // nb x kp   box multipoles (box-scaled)
  double2* L;   // nb x kp   box locals (box-scaled)
  double2* Lc;  // nc x kq   QBX locals (radius-scaled), sorted centre order
  double* phi;  // nconv     near + W-far point potential (no 1/4pi)
  // lists (device CSR)
  const int64_t* near_starts;  // per box -> segments (src_start, src_count) of U u W_close u X_close
  const int2* near_seg;
  const int* near_nsrc;        // per box: sources over its near segments
  const int64_t* near_off;     // per box: offset of its flattened near-source list in near_src
  const int* near_src;         // flattened near-source lists (box-sorted source indices)
  const int64_t* xfar_starts;  // per box -> segments of X_far
  const int2* xfar_seg;
  const int64_t* v_starts;     // per box -> (source box, offset index)
  const int2* v_ent;
  const int64_t* wfar_starts;  // per box -> source box
  const int* wfar_box;
  // operator tables
  const double2* m2l_tab;  // 1331 x ktab_m2l: I(2*delta) for box offsets delta in [-5,5]^3
  const double2* oct_m2m;  // 8 x kp: R((child-parent)/|child|)
  const double2* oct_l2l;  // 8 x kp: R((child-parent)/|parent|)
  unsigned int* bad;       // set by Stage 9 when a potential / centre coefficient is non-finite
};

// Stage 4 M2L (m2l_pas.cu): point-and-shoot on real half-table blocks, one operator
// set per offset class (rho_xy^2, dz).  Target-grouped: one CTA owns a group of G
// target boxes and accumulates their List-2 contributions on chip; its work is a
// list of tiles, each <= pas_tile_cols() entries of one class (columns sorted by
// (target slot, offset)), so every box local is written once, in a fixed order.
constexpr int kMaxPasOrder = 21;
constexpr int kPasMirror = 1 << 30;  // column flag: offset below the xy-plane, operator of (rho_xy^2, |dz|) mirrored
struct M2LPlan {
  int KR = 0, KRp = 0;         // (p+1)^2 real DOF, padded to a multiple of 64 (tree-shift GEMMs)
  int* rmap = nullptr;         // real DOF -> double offset in a complex half table (-1 = pad)
  double* temp = nullptr;      // staging rows of the tree shifts (KRp doubles each)
  int n_offsets = 0, n_classes = 0;
  double2* cs = nullptr;       // n_offsets x (p+1): (cos k alpha, sin k alpha)
  double* pas_ops = nullptr;   // n_classes x pas_stride: [W | Z | V], blocks in DMMA fragment order
  int pas_stride = 0, pas_phase = 0, pas_nblk = 0;
  int* pas_tab = nullptr;      // block row sets and per-warp block lists of the three phases
  int pas_tab_n = 0;
  int pas_base[3] = {0, 0, 0};
  // target groups
  int n_groups = 0, group = 0; // groups, target boxes per group (G)
  int* grp_order = nullptr;    // launch order (heaviest first)
  int* grp_tiles = nullptr;    // n_groups + 1 tile offsets
  int* grp_box = nullptr;      // n_groups x G target boxes (-1: none)
  int4* tiles = nullptr;       // (class, first column, columns, 1 if the class lies on the z axis: W = V = identity)
  int* col_src = nullptr;      // source box of each column
  int* col_meta = nullptr;     // target slot | offset id << 8 | kPasMirror if dz < 0
};
bool pas_supported(int p);
int pas_tile_cols(int p);
int pas_group_size(int p);
void pas_build_ops(int p, int n_cls, const int* cls_rxy2, const int* cls_dz, std::vector<double>& ops,
                   int& op_stride, std::vector<int>& tab, int& nblk, int& phase_size, int (&base)[3]);
int launch_m2l(const M2LPlan& P, const DevData& D, cudaStream_t s);  // Stage 4

// Tree shifts (Stage 2 M2M, Stage 7 L2L) as DMMA GEMMs over 8 octant operators:
// one level = tiles of same-octant columns, staged rows, segmented reduce.
struct ShiftLevel {
  int n_tiles = 0;
  int4* tiles = nullptr;
  int* col_src = nullptr;       // box whose expansion is shifted
  int* col_pos = nullptr;       // staging row
  double* col_scale = nullptr;  // 1
  int n_out = 0;
  int* out_boxes = nullptr;     // receiving boxes
  int2* out_seg = nullptr;      // staging rows [first, last) of each receiver
};
int launch_shift_ops(int mode, int p, int KR, int KRp, const int4* rdof, double* ops, cudaStream_t s);
int launch_shift_level(const M2LPlan& P, const ShiftLevel& S, const double* ops, double2* X, int kp, bool accumulate,
                       cudaStream_t s);

// Thread-per-centre translations (centre_trans.cu)
int launch_m2p(const DevData& D, const int* tgt_boxes, int n_tgt, cudaStream_t s);  // List 3 far, conventional targets
// M2QBXL over (centre, List-3-far box) pairs, chunked by centres.
struct PairChunk {
  int n_pairs = 0;
  int2* pairs = nullptr;   // (sorted centre, source box), centre-major
  int pair_base = 0;       // index of the chunk's first pair (starts are global)
  int n_centres = 0;
  int* centres = nullptr;  // sorted centre ids of the chunk
  int* starts = nullptr;   // n_centres + 1 global pair offsets
  int* perm = nullptr;     // chunk pair indices in source-box order (stable)
  int2* ctas = nullptr;    // box-major CTA descriptors (first perm index, count)
  int n_ctas = 0;
};
constexpr int kW3Threads = 128;
constexpr int kW3Boxes = 4;
struct PairPlan {
  double2* temp = nullptr;  // max chunk pairs x kq
  std::vector<PairChunk> chunks;
};
int launch_m2qbxl_pairs(const DevData& D, const PairPlan& P, cudaStream_t s);
// L2QBXL over host-built CTA descriptors (first item, count): <= kL3Threads
// consecutive centres from <= kL3Boxes boxes, box tables staged in shared memory.
constexpr int kL3Threads = 128;
constexpr int kL3Boxes = 8;
int launch_l2qbxl3(const DevData& D, const int* items, const int2* ctas, int n_ctas, const int* ctr_box,
                   cudaStream_t s);

// launchers (return number of kernels launched)
int launch_gather(const DevData& D, int ns, const int* perm, const double* w, const double* mu, cudaStream_t s);
int launch_p2m(const DevData& D, const int* boxes, int n, cudaStream_t s);
// batched densities (R right-hand sides): sorted weights / dipoles, and the
// near-field P2QBXL for NR = near_batch_width(q) densities per pass
int launch_gather_batch(const DevData& D, int ns, int R, const int* perm, const double* w, const double* mu,
                        double* bw, double4* bmu, cudaStream_t s);
int near_batch_width(int q);
int launch_near_qbx_batch(const DevData& D, const int* boxes, int n, int NR, const double* bw, const double4* bmu,
                          int64_t ns, double2* bLc, int64_t nc, cudaStream_t s);
int launch_near_qbx(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_near_p2p(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_p2l(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_eval(const DevData& D, int n_assoc, const int* assoc_items, const double* tpos, const int* assoc,
                const int* ctr_sorted, int n_conv, const int* conv_items, const int* tgt_perm, const int* tgt_box,
                double* pot, cudaStream_t s);
int launch_centre_out(const DevData& D, int nc, const int* items, const int* ctr_perm, double* out, cudaStream_t s);
// gather rows (pack: buf[k] = full[idx[k]]) or scatter them back (unpack), `width` doubles each
int launch_pack(int n, const int* idx, int width, double* full, double* buf, bool unpack, cudaStream_t s);
// Error path after a non-finite result: the first (kind, particle, source) triple whose
// near-field pair is coincident, packed (kind << 62 | original id << 31 | original source id),
// kind 0 = QBX centre, 1 = conventional target; ~0ull when there is none.
int launch_find_coincident(const DevData& D, int nc, const int* ctr_box, const int* ctr_perm, int n_conv,
                           const int* tgt_box, const int* tgt_perm, const int* src_perm, unsigned long long* out,
                           cudaStream_t s);
int launch_tables(const DevData& D, double2* m2l_tab, double2* oct_m2m, double2* oct_l2l, cudaStream_t s);
int launch_direct_sum(int ns, const double4* src, const double4* mu, int nt, const double4* tgt, double* pot,
                      unsigned long long* bad, cudaStream_t s);
int launch_direct_qbx(int q, int ns, const double4* src, const double4* mu, int nc, const double4* ctr,
                      double2* Lc, cudaStream_t s);
int launch_direct_qbx_eval(int q, int n, const double* tpos, const int* assoc, const double4* ctr,
                           const double2* Lc, double* pot, cudaStream_t s);
// Helmholtz single (+ double) layer, unaccelerated (helm.cu): complex weights / dipoles / potentials
int launch_helm_direct_sum(double k, int ns, const double4* src, const double2* w, const double2* mu, int nt,
                           const double4* tgt, double2* pot, unsigned long long* bad, cudaStream_t s);
int launch_helm_direct_qbx(double k, int q, int ns, const double4* src, const double2* w, const double2* mu, int nc,
                           const double4* ctr, double2* Lc, int nt, const double* tpos, const int* assoc,
                           double2* pot, cudaStream_t s);
void upload_constants();
void set_smem_limits();

}  // namespace dev
}  // namespace qbxg
