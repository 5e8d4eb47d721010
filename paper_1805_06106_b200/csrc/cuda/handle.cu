// Device handle: qbxg_create / qbxg_apply / qbxg_apply_device / qbxg_destroy
// and qbxg_direct_sum.  Replaces the reference's declared execute() driver
// (src/fmm.cpp, proj/CMakeLists.txt:27) and direct_sum
// (proj/src/kernels.cpp:46-73) with one sm_100a pass over Stages 2-9.
//
// HBM layout (all box-sorted in the plan's DFS preorder):
//   sources  double4 (x, y, z, w) [+ double4 dipole]      32 B (64 B SL+DL) per source
//   centres  double4 (x, y, z, r)                          32 B per centre
//   targets  double4 (x, y, z, 0) for conventional targets
//   boxes    double4 (cx, cy, cz, |b|)
//   M, L     nb x K_p complex (half table), box-scaled
//   L_c      nc x K_q complex (half table), radius-scaled
// Lists are CSR; near-field lists are flattened into source segments.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "harmonics.cuh"
#include "helm.cuh"
#include "../host/helm_rot.hpp"
#include "kernels.cuh"
#include "../host/rotation.hpp"

namespace qbxg {

#define QCK(call)                                                                                    \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      throw ::qbxg::CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);         \
  } while (0)

namespace {

template <class T>
T* dalloc(std::vector<void*>& owned, size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  QCK(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

template <class T>
T* dupload(std::vector<void*>& owned, const std::vector<T>& v, cudaStream_t s) {
  T* p = dalloc<T>(owned, v.size());
  if (!v.empty()) QCK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

void check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device available (the qbxg GPU path has no CPU fallback)");
  }
}

}  // namespace

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;   // near field forked beside the far-field chain (NEAR_SIDE)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaEvent_t evx[4] = {};       // near begin/end (side stream), P2L end, L2L end
  bool overlap = false, timed_overlap = false;
  bool debug_sync = false;    // QBXG_DEBUG_SYNC (read once at create): sync after every launch group
  // sharded result all-gather: packed segments per rank (targets; centre rows of 2 kq)
  std::vector<int64_t> res_off, cres_off;
  int* d_res_idx = nullptr;   // original target id of each packed slot
  double* d_res_buf = nullptr;
  int* d_cres_idx = nullptr;  // original centre id of each packed row
  double* d_cres_buf = nullptr;
  cudaEvent_t ev[QBXG_NUM_TIMERS + 2] = {};
  qbxg_config cfg{};
  int64_t ns = 0, nc = 0, nt = 0, nconv = 0;
  int nb = 0, nlev = 0;
  dev::DevData D{};
  std::vector<void*> owned;
  // index arrays
  int* d_src_perm = nullptr;
  int* d_ctr_perm = nullptr;
  int* d_tgt_perm = nullptr;
  int* d_tgt_box = nullptr;
  int* d_ctr_sorted = nullptr;
  int* d_assoc = nullptr;
  double* d_tpos = nullptr;
  // work lists
  int* d_leaves = nullptr;
  int n_leaves = 0;
  int* d_ctr_boxes = nullptr;
  int n_ctr_boxes = 0;
  int* d_near_boxes = nullptr;  // d_ctr_boxes, heaviest near field first (no tail of big boxes)
  int* d_tgt_boxes = nullptr;
  int n_tgt_boxes = 0;
  int* d_v_boxes = nullptr;
  int n_v_boxes = 0;
  int* d_wfar_boxes = nullptr;   // boxes with List 3 far entries and centres
  int n_wfar_boxes = 0;
  int* d_wfar_tboxes = nullptr;  // boxes with List 3 far entries and conventional targets
  int n_wfar_tboxes = 0;
  int* d_xfar_boxes = nullptr;
  int n_xfar_boxes = 0;
  int* d_ctr_box = nullptr;      // owning box of each sorted centre
  int* d_flat_all = nullptr;     // 0..nc-1
  int* d_flat_wfar = nullptr;    // sorted centres of boxes with List 3 far entries
  int n_flat_wfar = 0;
  int2* d_l3_ctas = nullptr;     // L2QBXL CTA descriptors (first item in d_flat_all, count)
  int n_l3_ctas = 0;
  dev::PairPlan wpairs;          // M2QBXL (centre, W_far box) pairs
  double* ops_m2m = nullptr;     // 8 octant operators (real DOF)
  double* ops_l2l = nullptr;
  std::vector<dev::ShiftLevel> m2m_levels, l2l_levels;
  std::vector<dev::ShiftLevel> m2m_straddle;  // per level, recomputed after the exchange
  // sharding: rank's role bits per box and the global cuts
  int nranks = 1, rank = 0;
  // results packed per rank and gathered (sharded handles; also a one-rank handle made by
  // qbxg_create_sharded, which runs the whole NCCL protocol on a communicator of one)
  bool gather = false;
  std::vector<uint8_t> mask;
  std::vector<int32_t> cuts;
  int* d_eval_assoc = nullptr;   // owned associated targets (original index)
  int n_eval_assoc = 0;
  int* d_eval_conv = nullptr;    // owned conventional targets (sorted index)
  int n_eval_conv = 0;
  int* d_own_ctr = nullptr;      // owned centres (sorted index)
  int n_own_ctr = 0;
  void* nccl_comm = nullptr;     // ncclComm_t when attached
  // staging for host applies
  double* d_w = nullptr;
  double* d_mu_in = nullptr;
  double* d_pot = nullptr;
  double* d_coeffs = nullptr;
  dev::M2LPlan m2l;
  int last_launches = 0;
  unsigned int* h_bad = nullptr;  // pinned copy of D.bad, read after every apply
  // Helmholtz single layer (cfg.kernel == QBXG_KERNEL_HELMHOLTZ_SL): helm_setup / run_helm
  bool helm = false;
  dev::HelmData HD{};
  std::vector<double2*> h_ops_m2m, h_ops_l2l;  // per level: 8 octant operators
  // batched shifts: (src, dst) pairs grouped by (level, octant)
  int2* h_m2m_pairs = nullptr;
  int2* h_l2l_pairs = nullptr;
  std::vector<int> h_m2m_off, h_l2l_off;  // (nlev x 8 + 1) offsets
  int2* h_m2m_spairs = nullptr;           // sharded: M2M pairs into boxes whose subtree spans ranks
  std::vector<int> h_m2m_soff;
  double2* h_cs = nullptr;                     // per operator e^{i m alpha}, m <= p (split form)
  int* h_ent_op = nullptr;                     // operator of every List-2 CSR entry (split form)
  double* h_zops = nullptr;   // per operator: Z blocks (fragment order)
  double* h_wvops = nullptr;  // per polar-angle class: W and V blocks
  int* h_op_cls = nullptr;    // operator -> polar-angle class
  int* h_pas_tab = nullptr;
  int h_pas_tab_n = 0, h_zstride = 0, h_wvstride = 0;
  int h_pas_base[2][3] = {};
  struct HelmM2LChunk {
    int n_tiles = 0;
    int4* tiles = nullptr;
    int* col_src = nullptr;
    int* col_pos = nullptr;
    int n_boxes = 0;
    int* boxes = nullptr;
    int64_t base = 0;
  };
  std::vector<HelmM2LChunk> h_m2l;
  double2* h_temp = nullptr;                   // M2L staging rows (KP complex)
  int h_n_wctas = 0, h_n_wcentres = 0;         // M2QBXL: box-major CTAs, centre-major reduce
  int4* h_wctas = nullptr;
  int *h_wctr = nullptr, *h_wrow = nullptr, *h_wcentres = nullptr, *h_wstarts = nullptr;
  double2* h_wrows = nullptr;
  int n_tgt_boxes_eval = 0;                    // boxes owning conventional targets (L2P)
  int* d_tgt_boxes_eval = nullptr;
  int h_n_lctas = 0;                           // L2QBXL CTAs over each box's centres
  int4* h_lctas = nullptr;
  int* h_lctr = nullptr;
  double* d_wc = nullptr;                      // host-apply staging: complex weights, potentials
  double* d_muc = nullptr;                     // host-apply staging: complex dipoles (SL+DL)
  double* d_potc = nullptr;
  double* d_coeffc = nullptr;
  // batched densities (qbxg_apply_batch*): NR-wide near-field buffers, grown on demand
  int bnr = 0;                   // densities per near-field pass (0: not allocated)
  double* d_bw = nullptr;        // bnr x ns sorted weights
  double4* d_bmu = nullptr;      // bnr x ns sorted dipoles
  double2* d_bLc = nullptr;      // bnr x nc x kq centre locals (near part, then completed in place)
  int64_t bhost_cap = 0;         // densities the host staging below can hold
  int64_t bcoeff_cap = 0;        // densities d_bcoeffs can hold
  double *d_bw_in = nullptr, *d_bmu_in = nullptr, *d_bpot = nullptr, *d_bcoeffs = nullptr;

  ~Handle() {
    if (stream) cudaStreamSynchronize(stream);
    if (nccl_comm) {
      void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (lib) {
        auto destroy = reinterpret_cast<ncclResult_t (*)(ncclComm_t)>(dlsym(lib, "ncclCommDestroy"));
        if (destroy) destroy(static_cast<ncclComm_t>(nccl_comm));
      }
    }
    for (void* p : owned) cudaFree(p);
    if (h_bad) cudaFreeHost(h_bad);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (side) cudaStreamDestroy(side);
    if (fork_ev) cudaEventDestroy(fork_ev);
    for (auto& e : evx)
      if (e) cudaEventDestroy(e);
    if (join_ev) cudaEventDestroy(join_ev);
  }
};

namespace {

// Tree-shift levels (M2M / L2L DMMA GEMMs, m2l_gemm.cu) and the Stage 4 M2L work:
// point-and-shoot operators per offset class and target groups with their tiles
// (m2l_pas.cu).
void build_m2l(Handle& H, const qbxg_plan_view& V, const std::vector<int64_t>& vstarts,
               const std::vector<int2>& vent, cudaStream_t s) {
  auto& O = H.owned;
  dev::M2LPlan& P = H.m2l;
  const int p = H.cfg.p_fmm;
  P.KR = (p + 1) * (p + 1);
  P.KRp = (P.KR + 63) / 64 * 64;
  std::vector<int4> rdof(P.KRp, make_int4(0, 0, 0, 0));
  std::vector<int> rmap(P.KRp, -1);
  {
    int r = 0;
    for (int n = 0; n <= p; ++n)
      for (int m = 0; m <= n; ++m)
        for (int part = 0; part < (m == 0 ? 1 : 2); ++part) {
          rdof[r] = make_int4(n, m, part, 0);
          rmap[r] = 2 * dev::hidx(n, m) + part;
          ++r;
        }
  }
  P.rmap = dupload(O, rmap, s);
  int4* d_rdof = dupload(O, rdof, s);
  const int nb = V.n_boxes;
  // the rank's (filtered) List-2 CSR: entries (source box, offset slot)
  const int64_t* vs = vstarts.data();
  const int64_t nent = vs[nb];
  std::vector<int> vb(nent), slot(nent);
  std::vector<int> slot_to_op(1331, -1), used;
  for (int64_t e = 0; e < nent; ++e) {
    vb[e] = vent[e].x;
    const int sl = vent[e].y;
    slot[e] = sl;
    if (slot_to_op[sl] < 0) {
      slot_to_op[sl] = int(used.size());
      used.push_back(sl);
    }
  }
  const auto& mk = H.mask;

  // --- tree shifts: octant operators and per-level tiles
  int64_t max_level_rows = 1;
  {
    H.ops_m2m = dalloc<double>(O, size_t(8) * P.KRp * P.KRp);
    H.ops_l2l = dalloc<double>(O, size_t(8) * P.KRp * P.KRp);
    dev::launch_shift_ops(1, p, P.KR, P.KRp, d_rdof, H.ops_m2m, s);
    dev::launch_shift_ops(2, p, P.KR, P.KRp, d_rdof, H.ops_l2l, s);
    auto octant = [&](int c, int par) {
      return (V.box_center[3 * c] > V.box_center[3 * par] ? 1 : 0) |
             (V.box_center[3 * c + 1] > V.box_center[3 * par + 1] ? 2 : 0) |
             (V.box_center[3 * c + 2] > V.box_center[3 * par + 2] ? 4 : 0);
    };
    // cols: (octant, src, pos) -> tiles of <= 64 same-octant columns
    auto make_level = [&](const std::vector<int3>& cols, const std::vector<int>& outb,
                          const std::vector<int2>& seg) {
      dev::ShiftLevel L;
      if (cols.empty()) return L;
      std::vector<int> csrc, cpos;
      std::vector<double> cscale;
      std::vector<int4> tiles;
      for (int o = 0; o < 8; ++o) {
        const int first = int(csrc.size());
        for (const int3& c : cols)
          if (c.x == o) {
            csrc.push_back(c.y);
            cpos.push_back(c.z);
            cscale.push_back(1.0);
          }
        for (int i = first; i < int(csrc.size()); i += 64)
          tiles.push_back(make_int4(o, i, std::min(64, int(csrc.size()) - i), 0));
      }
      L.n_tiles = int(tiles.size());
      L.tiles = dupload(O, tiles, s);
      L.col_src = dupload(O, csrc, s);
      L.col_pos = dupload(O, cpos, s);
      L.col_scale = dupload(O, cscale, s);
      L.n_out = int(outb.size());
      L.out_boxes = dupload(O, outb, s);
      L.out_seg = dupload(O, seg, s);
      max_level_rows = std::max<int64_t>(max_level_rows, int64_t(cols.size()));
      return L;
    };
    H.m2m_levels.assign(H.nlev, dev::ShiftLevel());
    H.m2m_straddle.assign(H.nlev, dev::ShiftLevel());
    H.l2l_levels.assign(H.nlev, dev::ShiftLevel());
    for (int l = 0; l < H.nlev; ++l) {
      std::vector<int3> cols;
      std::vector<int> outb;
      std::vector<int2> seg;
      // upward: boxes whose subtree is the rank's (pass 0) or spans ranks (pass 1, after the exchange)
      for (int pass = 0; pass < 2; ++pass) {
        const uint8_t want = pass == 0 ? QBXG_SHARD_SUBTREE : QBXG_SHARD_STRADDLE;
        cols.clear();
        outb.clear();
        seg.clear();
        for (int i = V.level_starts[l]; i < V.level_starts[l + 1]; ++i) {
          const int b = V.level_boxes[i];
          if ((V.box_flags[b] & QBXG_BOX_LEAF) || !(V.box_flags[b] & QBXG_BOX_HAS_SOURCES)) continue;
          if (!(mk[b] & want)) continue;
          const int first = int(cols.size());
          for (int k = V.child_starts[b]; k < V.child_starts[b + 1]; ++k) {
            const int c = V.children[k];
            if (V.src_sub_count[c] == 0) continue;
            cols.push_back(make_int3(octant(c, b), c, int(cols.size())));
          }
          outb.push_back(b);
          seg.push_back(make_int2(first, int(cols.size())));
        }
        (pass == 0 ? H.m2m_levels : H.m2m_straddle)[l] = make_level(cols, outb, seg);
      }
      cols.clear();
      outb.clear();
      seg.clear();
      if (l == 0) continue;
      for (int i = V.level_starts[l]; i < V.level_starts[l + 1]; ++i) {
        const int b = V.level_boxes[i];
        if (!(V.box_flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR))) continue;
        if (!(mk[b] & QBXG_SHARD_DOWN)) continue;
        const int par = V.box_parent[b];
        const int pos = int(cols.size());
        cols.push_back(make_int3(octant(b, par), par, pos));
        outb.push_back(b);
        seg.push_back(make_int2(pos, pos + 1));
      }
      H.l2l_levels[l] = make_level(cols, outb, seg);
    }
  }
  if (nent == 0) {
    P.temp = dalloc<double>(O, size_t(max_level_rows) * P.KRp);
    return;
  }
  if (!dev::pas_supported(p)) throw InvalidArgument("qbxg_create: the M2L supports 1 <= p_fmm <= 21");
  // --- Stage 4 operators: one [W | Z | V] set per class (rho_xy^2, |dz|), classes
  // numbered in key order (independent of which offsets a rank uses); per offset only
  // the azimuth alpha = atan2(dy, dx) remains, as the (cos k alpha, sin k alpha) table
  P.n_offsets = int(used.size());
  std::vector<int> cls_of_op(P.n_offsets), cls_rxy2, cls_dz;
  std::vector<double2> cs(size_t(P.n_offsets) * (p + 1));
  {
    auto key_of = [&](int sl) {
      const int dx = sl / 121 - 5, dy = (sl / 11) % 11 - 5, dz = sl % 11 - 5;
      return (dx * dx + dy * dy) * 11 + std::abs(dz);  // dz < 0: the mirrored operator (m2l_pas.cu)
    };
    std::vector<int> key_to_cls(51 * 11, -1);
    for (int o = 0; o < P.n_offsets; ++o) key_to_cls[key_of(used[o])] = 0;
    for (int k = 0; k < 51 * 11; ++k)
      if (key_to_cls[k] == 0) {
        key_to_cls[k] = int(cls_rxy2.size());
        cls_rxy2.push_back(k / 11);
        cls_dz.push_back(k % 11);
      } else {
        key_to_cls[k] = -1;
      }
    for (int o = 0; o < P.n_offsets; ++o) {
      const int sl = used[o], dx = sl / 121 - 5, dy = (sl / 11) % 11 - 5;
      cls_of_op[o] = key_to_cls[key_of(sl)];
      const double alpha = (dx == 0 && dy == 0) ? 0.0 : std::atan2(double(dy), double(dx));
      for (int k = 0; k <= p; ++k) cs[size_t(o) * (p + 1) + k] = make_double2(std::cos(k * alpha), std::sin(k * alpha));
    }
  }
  P.n_classes = int(cls_rxy2.size());
  P.cs = dupload(O, cs, s);
  {
    std::vector<double> pops;
    std::vector<int> tab;
    dev::pas_build_ops(p, P.n_classes, cls_rxy2.data(), cls_dz.data(), pops, P.pas_stride, tab, P.pas_nblk,
                       P.pas_phase, P.pas_base);
    P.pas_ops = dupload(O, pops, s);
    P.pas_tab = dupload(O, tab, s);
    P.pas_tab_n = int(tab.size());
    QCK(cudaStreamSynchronize(s));  // host vectors go out of scope
  }

  // --- work order: groups of G consecutive target boxes (DFS order); a group's entries
  // sorted by (class, target slot, offset) and cut into tiles of <= BN same-class
  // columns.  Groups launch heaviest first.
  const int G = dev::pas_group_size(p), BN = dev::pas_tile_cols(p);
  std::vector<int> tb;
  for (int b = 0; b < nb; ++b)
    if (vs[b + 1] > vs[b]) tb.push_back(b);
  const int ng = int((tb.size() + G - 1) / G);
  std::vector<int> col_src(nent), col_meta(nent), grp_box(size_t(ng) * G, -1);
  std::vector<std::vector<int4>> gtiles(ng);
  std::vector<int64_t> gwork(ng, 0);
#pragma omp parallel for schedule(dynamic, 16)
  for (int g = 0; g < ng; ++g) {
    const int i0 = g * G, i1 = std::min<int>(int(tb.size()), i0 + G);
    const int64_t e0 = vs[tb[i0]], e1 = vs[tb[i1 - 1] + 1];
    std::vector<uint64_t> key;
    key.reserve(size_t(e1 - e0));
    for (int i = i0; i < i1; ++i) {
      grp_box[size_t(g) * G + (i - i0)] = tb[i];
      for (int64_t e = vs[tb[i]]; e < vs[tb[i] + 1]; ++e)
        key.push_back(uint64_t(cls_of_op[slot_to_op[slot[e]]]) << 44 | uint64_t(i - i0) << 36 |
                      uint64_t(slot[e]) << 24 | uint64_t(e - e0));
    }
    std::sort(key.begin(), key.end());
    auto& T = gtiles[g];
    int64_t work = 0;
    for (size_t k = 0; k < key.size();) {
      const int cls = int(key[k] >> 44);
      size_t k1 = k;
      while (k1 < key.size() && int(key[k1] >> 44) == cls && k1 - k < size_t(BN)) ++k1;
      T.push_back(make_int4(cls, int(k), int(k1 - k), cls_rxy2[cls] == 0 ? 1 : 0));  // .w: offset on the z axis
      work += 64 + int64_t((k1 - k + 7) / 8) * 256;
      k = k1;
    }
    for (size_t k = 0; k < key.size(); ++k) {
      const int64_t e = e0 + int64_t(key[k] & 0xFFFFFF);
      col_src[e0 + int64_t(k)] = vb[e];
      col_meta[e0 + int64_t(k)] =
          int((key[k] >> 36) & 255) | slot_to_op[slot[e]] << 8 | (slot[e] % 11 < 5 ? dev::kPasMirror : 0);
    }
    gwork[g] = work;
  }
  std::vector<int4> tiles;
  std::vector<int> grp_tiles{0};
  for (int g = 0; g < ng; ++g) {
    const int64_t e0 = vs[tb[size_t(g) * G]];
    for (int4 t : gtiles[g]) tiles.push_back(make_int4(t.x, int(e0 + t.y), t.z, t.w));
    grp_tiles.push_back(int(tiles.size()));
  }
  std::vector<int> order(ng);
  for (int g = 0; g < ng; ++g) order[g] = g;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return gwork[a] > gwork[b]; });
  P.n_groups = ng;
  P.group = G;
  P.grp_order = dupload(O, order, s);
  P.grp_tiles = dupload(O, grp_tiles, s);
  P.grp_box = dupload(O, grp_box, s);
  P.tiles = dupload(O, tiles, s);
  P.col_src = dupload(O, col_src, s);
  P.col_meta = dupload(O, col_meta, s);
  QCK(cudaStreamSynchronize(s));
  P.temp = dalloc<double>(O, size_t(max_level_rows) * P.KRp);
}

// ---- Helmholtz single layer: device data, operators and work lists --------
void helm_setup(Handle& H, const qbxg_plan_view& V, const std::vector<int64_t>& vs, const std::vector<int2>& vent,
                cudaStream_t s) {
  auto& O = H.owned;
  dev::DevData& D = H.D;
  dev::HelmData& HD = H.HD;
  const int p = H.cfg.p_fmm, q = H.cfg.p_qbx, nb = H.nb;
  HD.k = H.cfg.helmholtz_k;
  HD.P = p;
  HD.Q = q;
  HD.KP = (p + 1) * (p + 1);
  HD.KQ = (q + 1) * (q + 1);
  HD.GL = p + 1;
  HD.box = D.box;
  HD.child_starts = D.child_starts;
  HD.children = D.children;
  HD.parent = D.parent;
  HD.src_own_start = D.src_own_start;
  HD.src_own_count = D.src_own_count;
  HD.ctr_own_start = D.ctr_own_start;
  HD.ctr_own_count = D.ctr_own_count;
  HD.tgt_own_start = D.tgt_own_start;
  HD.tgt_own_count = D.tgt_own_count;
  HD.src = D.src;
  HD.ctr = D.ctr;
  HD.tgt = D.tgt;
  HD.near_starts = D.near_starts;
  HD.bad = D.bad;
  HD.near_seg = D.near_seg;
  HD.xfar_starts = D.xfar_starts;
  HD.xfar_seg = D.xfar_seg;
  HD.v_starts = D.v_starts;
  HD.wfar_starts = D.wfar_starts;
  HD.wfar_box = D.wfar_box;
  HD.hw = dalloc<double2>(O, std::max<int64_t>(H.ns, 1));
  HD.hmu = H.cfg.kernel == QBXG_KERNEL_HELMHOLTZ_SL_DL ? dalloc<double2>(O, 3 * std::max<int64_t>(H.ns, 1)) : nullptr;
  H.d_muc = HD.hmu ? dalloc<double>(O, 6 * std::max<int64_t>(H.ns, 1)) : nullptr;
  HD.M = dalloc<double2>(O, size_t(nb) * HD.KP);
  HD.L = dalloc<double2>(O, size_t(nb) * HD.KP);
  HD.Lc = dalloc<double2>(O, size_t(std::max<int64_t>(H.nc, 1)) * HD.KQ);
  // sharded: only the rank's centres are ever written; the others read as zero in the centre output
  if (H.gather) QCK(cudaMemsetAsync(HD.Lc, 0, size_t(std::max<int64_t>(H.nc, 1)) * HD.KQ * sizeof(double2), s));
  HD.phi = dalloc<double2>(O, std::max<int64_t>(H.nconv, 1));
  HD.gaunt = dupload(O, helm_gaunt_table(p), s);
  dev::helm_upload_constants();
  {
    double* gc = dalloc<double>(O, dev::helm_gaunt_ctr_size(p, q));
    HD.gaunt_ctr = gc;
    dev::helm_build_gaunt_ctr(HD, gc, s);
  }
  H.d_wc = dalloc<double>(O, 2 * std::max<int64_t>(H.ns, 1));
  H.d_potc = dalloc<double>(O, 2 * std::max<int64_t>(H.nt, 1));
  H.d_coeffc = dalloc<double>(O, 2 * std::max<int64_t>(H.nc, 1) * HD.KQ);
  const size_t opsz = size_t(HD.KP) * HD.KP;

  // level radii and M2M / L2L octant operators (child offset d_o = (+-h, +-h, +-h))
  std::vector<double> hl(H.nlev, 0.0);
  for (int l = 0; l < H.nlev; ++l)
    if (V.level_starts[l + 1] > V.level_starts[l]) hl[l] = V.box_radius[V.level_boxes[V.level_starts[l]]];
  std::vector<double4> shifts;
  auto octv = [](int o, double h, double sg) {
    return make_double4(sg * ((o & 4) ? h : -h), sg * ((o & 2) ? h : -h), sg * ((o & 1) ? h : -h), 0.0);
  };
  for (int l = 0; l + 1 < H.nlev; ++l)  // M2M into parents at level l: t = parent - child
    for (int o = 0; o < 8; ++o) shifts.push_back(octv(o, hl[l + 1], -1.0));
  for (int l = 1; l < H.nlev; ++l)  // L2L into children at level l: t = child - parent
    for (int o = 0; o < 8; ++o) shifts.push_back(octv(o, hl[l], 1.0));
  double2* shift_ops = dalloc<double2>(O, std::max<size_t>(shifts.size(), 1) * opsz);
  if (!shifts.empty()) dev::helm_build_ops(HD, int(shifts.size()), dupload(O, shifts, s), shift_ops, s);
  H.h_ops_m2m.assign(H.nlev, nullptr);
  H.h_ops_l2l.assign(H.nlev, nullptr);
  {
    size_t k = 0;
    for (int l = 0; l + 1 < H.nlev; ++l, k += 8) H.h_ops_m2m[l] = shift_ops + k * opsz;
    for (int l = 1; l < H.nlev; ++l, k += 8) H.h_ops_l2l[l] = shift_ops + k * opsz;
  }
  {
    // (src, dst) pairs per (level, octant) with the operators' octant convention (x 4, y 2, z 1)
    auto hoct = [&](int c, int par) {
      return (V.box_center[3 * c] > V.box_center[3 * par] ? 4 : 0) +
             (V.box_center[3 * c + 1] > V.box_center[3 * par + 1] ? 2 : 0) +
             (V.box_center[3 * c + 2] > V.box_center[3 * par + 2] ? 1 : 0);
    };
    const auto& mk = H.mask;
    std::vector<std::vector<int2>> m2m(size_t(H.nlev) * 8), l2l(size_t(H.nlev) * 8), m2ms(size_t(H.nlev) * 8);
    for (int l = 0; l < H.nlev; ++l)
      for (int i = V.level_starts[l]; i < V.level_starts[l + 1]; ++i) {
        const int b = V.level_boxes[i];
        // upward: boxes whose subtree is the rank's, and (after the exchange) those spanning ranks
        if (!(V.box_flags[b] & QBXG_BOX_LEAF) && (V.box_flags[b] & QBXG_BOX_HAS_SOURCES) &&
            (mk[b] & (QBXG_SHARD_SUBTREE | QBXG_SHARD_STRADDLE)))
          for (int k = V.child_starts[b]; k < V.child_starts[b + 1]; ++k) {
            const int c = V.children[k];
            if (V.src_sub_count[c] > 0)
              ((mk[b] & QBXG_SHARD_SUBTREE) ? m2m : m2ms)[size_t(l) * 8 + hoct(c, b)].push_back(make_int2(c, b));
          }
        if (l > 0 && (V.box_flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR)) && (mk[b] & QBXG_SHARD_DOWN)) {
          const int a = V.box_parent[b];
          l2l[size_t(l) * 8 + hoct(b, a)].push_back(make_int2(a, b));
        }
      }
    std::vector<int2> pm, pl, ps;
    H.h_m2m_off.assign(size_t(H.nlev) * 8 + 1, 0);
    H.h_l2l_off.assign(size_t(H.nlev) * 8 + 1, 0);
    H.h_m2m_soff.assign(size_t(H.nlev) * 8 + 1, 0);
    for (size_t g = 0; g < m2m.size(); ++g) {
      pm.insert(pm.end(), m2m[g].begin(), m2m[g].end());
      H.h_m2m_off[g + 1] = int(pm.size());
      ps.insert(ps.end(), m2ms[g].begin(), m2ms[g].end());
      H.h_m2m_soff[g + 1] = int(ps.size());
      pl.insert(pl.end(), l2l[g].begin(), l2l[g].end());
      H.h_l2l_off[g + 1] = int(pl.size());
    }
    H.h_m2m_pairs = dupload(O, pm, s);
    H.h_l2l_pairs = dupload(O, pl, s);
    if (!ps.empty()) H.h_m2m_spairs = dupload(O, ps, s);
    QCK(cudaStreamSynchronize(s));
  }

  // M2L operators per (level, offset slot) in use: t = c_b - c_d = 2 h_l delta
  const int64_t nent = vs[nb];
  std::vector<int> key_op;
  std::vector<int> op_of_entry(nent);
  {
    std::vector<int> key_to_op(size_t(H.nlev) * 1331, -1);
    std::vector<double4> msh;
    for (int b = 0; b < nb; ++b)
      for (int64_t e = vs[b]; e < vs[b + 1]; ++e) {
        const int l = V.box_level[b], sl = vent[e].y;
        int& op = key_to_op[size_t(l) * 1331 + sl];
        if (op < 0) {
          op = int(msh.size());
          const double dx = sl / 121 - 5, dy = (sl / 11) % 11 - 5, dz = sl % 11 - 5;
          msh.push_back(make_double4(2 * hl[l] * dx, 2 * hl[l] * dy, 2 * hl[l] * dz, 1.0));
        }
        op_of_entry[e] = op;
      }
    if (!dev::helm_pas_supported(p)) throw InvalidArgument("qbxg_create: the Helmholtz M2L supports p_fmm <= 20");
    {  // point-and-shoot: W, V per polar angle of the integer offset (level independent), Z per (level, offset)
      const HpasLayout PL = hpas_layout(p);
      std::vector<int> cls(msh.size()), key_cls;
      std::vector<double> thetas;
      {
        std::vector<int> key_to_cls(51 * 11, -1);
        for (int l = 0; l < H.nlev; ++l)
          for (int sl = 0; sl < 1331; ++sl) {
            const int op = key_to_op[size_t(l) * 1331 + sl];
            if (op < 0) continue;
            const int dx = sl / 121 - 5, dy = (sl / 11) % 11 - 5, dz = sl % 11 - 5;
            int& c = key_to_cls[size_t(dx * dx + dy * dy) * 11 + (dz + 5)];
            if (c < 0) {
              c = int(thetas.size());
              thetas.push_back(std::atan2(std::sqrt(double(dx * dx + dy * dy)), double(dz)));
            }
            cls[op] = c;
          }
      }
      std::vector<double> wv;
      hpas_build_wv(p, thetas, wv);
      H.h_wvops = dupload(O, wv, s);
      H.h_op_cls = dupload(O, cls, s);
      H.h_wvstride = int(PL.wv_stride);
      H.h_zstride = int(PL.z_stride);
      H.h_zops = dalloc<double>(O, std::max<size_t>(msh.size(), 1) * PL.z_stride);
      H.h_cs = dalloc<double2>(O, std::max<size_t>(msh.size(), 1) * (p + 1));
      for (auto& v : msh) v.w = 0.0;
      std::vector<int> zoff(PL.z_off.begin(), PL.z_off.end());
      if (!msh.empty())
        dev::helm_build_zpas(HD, int(msh.size()), dupload(O, msh, s), zoff.data(), H.h_zstride, H.h_zops, H.h_cs, s);
      std::vector<int> tab;
      dev::helm_pas_tables(p, PL.wv_off[0][0].data(), PL.wv_off[0][1].data(), PL.wv_off[1][0].data(),
                           PL.wv_off[1][1].data(), PL.z_off.data(), tab, H.h_pas_base);
      H.h_pas_tab = dupload(O, tab, s);
      H.h_pas_tab_n = int(tab.size());
      H.h_ent_op = dupload(O, op_of_entry, s);
      QCK(cudaStreamSynchronize(s));  // host vectors go out of scope
    }
    // tiles of same-operator entries, chunked over contiguous target boxes
    const int cols = dev::helm_m2l_split_cols();
    size_t free2 = 0, total_b = 0;
    QCK(cudaMemGetInfo(&free2, &total_b));
    const int64_t cap = std::max<int64_t>(
        int64_t(std::min<size_t>(size_t(8) << 30, size_t(double(free2) * 0.4)) / (HD.KP * sizeof(double2))), 1024);
    int64_t max_chunk = 0;
    int b0 = 0;
    const int n_ops = int(msh.size());
    while (b0 < nb) {
      int b1 = b0;
      while (b1 < nb && (vs[b1 + 1] - vs[b0] <= cap || b1 == b0)) ++b1;
      const int64_t base = vs[b0], cnt = vs[b1] - vs[b0];
      if (cnt > 0) {
        Handle::HelmM2LChunk C;
        C.base = base;
        std::vector<int> boxes;
        for (int b = b0; b < b1; ++b)
          if (vs[b + 1] > vs[b]) boxes.push_back(b);
        std::vector<int64_t> cnt_op(n_ops + 1, 0);
        for (int64_t e = base; e < base + cnt; ++e) cnt_op[op_of_entry[e] + 1]++;
        for (int o = 0; o < n_ops; ++o) cnt_op[o + 1] += cnt_op[o];
        std::vector<int> csrc(cnt), cpos(cnt);
        std::vector<int64_t> fill(cnt_op.begin(), cnt_op.end() - 1);
        for (int64_t e = base; e < base + cnt; ++e) {
          const int64_t i = fill[op_of_entry[e]]++;
          csrc[i] = vent[e].x;
          cpos[i] = int(e - base);
        }
        std::vector<int4> tiles;
        for (int o = 0; o < n_ops; ++o)
          for (int64_t i = cnt_op[o]; i < cnt_op[o + 1]; i += cols)
            tiles.push_back(make_int4(o, int(i), int(std::min<int64_t>(cols, cnt_op[o + 1] - i)), 0));
        C.n_tiles = int(tiles.size());
        C.tiles = dupload(O, tiles, s);
        C.col_src = dupload(O, csrc, s);
        C.col_pos = dupload(O, cpos, s);
        C.n_boxes = int(boxes.size());
        C.boxes = dupload(O, boxes, s);
        H.h_m2l.push_back(C);
        max_chunk = std::max(max_chunk, cnt);
        QCK(cudaStreamSynchronize(s));
      }
      b0 = b1;
    }
    H.h_temp = dalloc<double2>(O, size_t(std::max<int64_t>(max_chunk, 1)) * HD.KP);
  }

  // M2QBXL pairs (centre, W_far box): centre-major index for the reduce, box-major CTAs
  {
    std::vector<int2> pr;  // (sorted centre, box), centre-major
    std::vector<int> centres, starts;
    for (int b = 0; b < nb; ++b) {
      const int64_t a = V.list_starts[QBXG_LIST_W_FAR][b], e = V.list_starts[QBXG_LIST_W_FAR][b + 1];
      if (a == e || !(V.box_flags[b] & QBXG_BOX_TARGET)) continue;
      for (int j = 0; j < V.ctr_own_count[b]; ++j) {
        const int cs = V.ctr_own_start[b] + j;
        centres.push_back(cs);
        starts.push_back(int(pr.size()));
        for (int64_t i = a; i < e; ++i) pr.push_back(make_int2(cs, V.list_boxes[QBXG_LIST_W_FAR][i]));
      }
    }
    starts.push_back(int(pr.size()));
    std::vector<int> perm(pr.size());
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = int(i);
    std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return pr[x].y < pr[y].y; });
    std::vector<int> wctr(pr.size()), wrow(pr.size());
    std::vector<int4> ctas;
    for (size_t i = 0; i < perm.size(); ++i) {
      wctr[i] = pr[perm[i]].x;
      wrow[i] = perm[i];
    }
    size_t i = 0;
    while (i < perm.size()) {
      const int box = pr[perm[i]].y;
      size_t j = i;
      while (j < perm.size() && pr[perm[j]].y == box && j - i < size_t(dev::kHCtrMax)) ++j;
      ctas.push_back(make_int4(box, int(i), int(j - i), 0));
      i = j;
    }
    H.h_n_wctas = int(ctas.size());
    H.h_wctas = dupload(O, ctas, s);
    H.h_wctr = dupload(O, wctr, s);
    H.h_wrow = dupload(O, wrow, s);
    H.h_n_wcentres = int(centres.size());
    H.h_wcentres = dupload(O, centres, s);
    H.h_wstarts = dupload(O, starts, s);
    H.h_wrows = dalloc<double2>(O, std::max<size_t>(pr.size(), 1) * HD.KQ);
  }
  {
    std::vector<int> tb;
    for (int b = 0; b < nb; ++b)
      if (V.tgt_own_count[b] > 0) tb.push_back(b);
    H.n_tgt_boxes_eval = int(tb.size());
    H.d_tgt_boxes_eval = dupload(O, tb, s);
  }
  // L2QBXL: each box's centres in CTAs of <= kHCtrMax
  {
    std::vector<int4> ctas;
    std::vector<int> lctr;
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < V.ctr_own_count[b]; j += dev::kHCtrMax) {
        const int n = std::min(dev::kHCtrMax, V.ctr_own_count[b] - j);
        ctas.push_back(make_int4(b, int(lctr.size()), n, 0));
        for (int k = 0; k < n; ++k) lctr.push_back(V.ctr_own_start[b] + j + k);
      }
    H.h_n_lctas = int(ctas.size());
    H.h_lctas = dupload(O, ctas, s);
    H.h_lctr = dupload(O, lctr, s);
  }
  QCK(cudaStreamSynchronize(s));
}

// One Helmholtz apply: d_wc complex weights (caller order, interleaved), d_pot
// complex potentials (caller order), d_coeffs optional centre locals (caller order).
// phase bits as in run_device: 1 = density gather, P2M, M2M of the rank's subtrees;
// 2 = M2M of straddling boxes (sharded), then Stages 3-9 for the rank's boxes.
void run_helm(Handle& H, const double* d_wc, const double* d_muc, double* d_pot, double* d_coeffs, cudaStream_t s,
              int phase = 3) {
  dev::HelmData& HD = H.HD;
  auto& ev = H.ev;
  int L = (phase & 1) ? 0 : H.last_launches;
  const bool debug_sync = H.debug_sync;
  int stage_no = 0;
  auto chk = [&](int k) {
    if (k < 0) throw InvalidArgument("qbxg_apply: unsupported Helmholtz order");
    L += k;
    ++stage_no;
    cudaError_t e = cudaPeekAtLastError();
    if (e == cudaSuccess && debug_sync) {
      e = cudaStreamSynchronize(s);
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e != cudaSuccess)
      throw CudaError(std::string("CUDA error after Helmholtz launch group ") + std::to_string(stage_no) + ": " +
                      cudaGetErrorString(e));
  };
  if (phase & 1) {
    QCK(cudaEventRecord(ev[0], s));
    if (HD.hmu && !d_muc) throw InvalidArgument("qbxg_apply_complex: Helmholtz SL+DL requires dipole moments");
    if (!HD.hmu && d_muc) throw InvalidArgument("qbxg_apply_complex: dipoles given to a single-layer handle");
    chk(dev::helm_gather(HD, H.ns, H.d_src_perm, d_wc, d_muc, s));
    QCK(cudaMemsetAsync(HD.M, 0, size_t(H.nb) * HD.KP * sizeof(double2), s));
    QCK(cudaMemsetAsync(HD.L, 0, size_t(H.nb) * HD.KP * sizeof(double2), s));
    QCK(cudaMemsetAsync(HD.phi, 0, size_t(std::max<int64_t>(H.nconv, 1)) * sizeof(double2), s));
    QCK(cudaMemsetAsync(HD.bad, 0, sizeof(unsigned int), s));
    QCK(cudaEventRecord(ev[1], s));
    chk(dev::helm_p2m(HD, H.d_leaves, H.n_leaves, s));
    QCK(cudaEventRecord(ev[2], s));
    for (int l = H.nlev - 2; l >= 0; --l) {
      for (int o = 0; o < 8; ++o) {  // octants in a fixed order: deterministic sums into the parents
        const int a = H.h_m2m_off[size_t(l) * 8 + o], e = H.h_m2m_off[size_t(l) * 8 + o + 1];
        chk(dev::helm_shift_pairs(HD, 0, H.h_m2m_pairs + a, e - a, H.h_ops_m2m[l] + size_t(o) * HD.KP * HD.KP, s));
      }
    }
    H.last_launches = L;
  }
  if (!(phase & 2)) return;
  // boxes whose subtree spans ranks: every rank recomputes them, children in the same
  // octant order as the unsharded pass, once the owned multipoles have been exchanged
  if (H.nranks > 1 && H.h_m2m_spairs)
    for (int l = H.nlev - 2; l >= 0; --l)
      for (int o = 0; o < 8; ++o) {
        const int a = H.h_m2m_soff[size_t(l) * 8 + o], e = H.h_m2m_soff[size_t(l) * 8 + o + 1];
        chk(dev::helm_shift_pairs(HD, 0, H.h_m2m_spairs + a, e - a, H.h_ops_m2m[l] + size_t(o) * HD.KP * HD.KP, s));
      }
  QCK(cudaEventRecord(ev[3], s));
  chk(dev::helm_near(HD, H.d_near_boxes, H.n_ctr_boxes, s));
  chk(dev::helm_p2p(HD, H.d_tgt_boxes, H.n_tgt_boxes, s));
  QCK(cudaEventRecord(ev[4], s));
  for (const auto& C : H.h_m2l)
    chk(dev::helm_m2l_pas(HD, C.n_tiles, C.tiles, C.col_src, C.col_pos, H.h_pas_tab, H.h_pas_tab_n, H.h_pas_base,
                          H.h_zops, H.h_zstride, H.h_wvops, H.h_wvstride, H.h_op_cls, H.h_cs, H.h_temp, C.n_boxes,
                          C.boxes, C.base, H.h_ent_op, s));
  QCK(cudaEventRecord(ev[5], s));
  chk(dev::helm_p2l(HD, H.d_xfar_boxes, H.n_xfar_boxes, s));
  QCK(cudaEventRecord(H.evx[2], s));
  for (int l = 1; l < H.nlev; ++l) {
    for (int o = 0; o < 8; ++o) {
      const int a = H.h_l2l_off[size_t(l) * 8 + o], e = H.h_l2l_off[size_t(l) * 8 + o + 1];
      chk(dev::helm_shift_pairs(HD, 1, H.h_l2l_pairs + a, e - a, H.h_ops_l2l[l] + size_t(o) * HD.KP * HD.KP, s));
    }
  }
  QCK(cudaEventRecord(H.evx[3], s));
  chk(dev::helm_ctr(HD, 1, HD.M, H.h_n_wctas, H.h_wctas, H.h_wctr, H.h_wrow, H.h_wrows, 0, s));
  chk(dev::helm_pair_reduce(HD, H.h_wcentres, H.h_wstarts, H.h_n_wcentres, H.h_wrows, s));
  chk(dev::helm_m2p(HD, H.d_wfar_tboxes, H.n_wfar_tboxes, s));
  QCK(cudaEventRecord(ev[6], s));
  chk(dev::helm_ctr(HD, 0, HD.L, H.h_n_lctas, H.h_lctas, H.h_lctr, H.h_lctr, HD.Lc, 1, s));
  QCK(cudaEventRecord(ev[9], s));
  if (H.gather)  // targets of other ranks stay zero until the result exchange
    QCK(cudaMemsetAsync(d_pot, 0, size_t(std::max<int64_t>(H.nt, 1)) * 2 * sizeof(double), s));
  chk(dev::helm_eval(HD, H.n_eval_assoc, H.d_eval_assoc, H.d_tpos, H.d_assoc, H.d_ctr_sorted, H.n_tgt_boxes_eval,
                     H.d_tgt_boxes_eval, H.d_tgt_perm, d_pot, s));
  // (sharded: the centre locals of other ranks' centres are zero from create on; nothing writes them)
  if (d_coeffs) chk(dev::helm_centre_out(HD, int(H.nc), H.d_ctr_perm, d_coeffs, s));
  if (H.gather) {  // the rank's results into its segment of the gather buffers
    const int64_t a = H.res_off[H.rank], e = H.res_off[H.rank + 1];
    chk(dev::launch_pack(int(e - a), H.d_res_idx + a, 2, d_pot, H.d_res_buf + 2 * a, false, s));
    if (d_coeffs) {
      const int64_t ca = H.cres_off[H.rank], ce = H.cres_off[H.rank + 1];
      chk(dev::launch_pack(int(ce - ca), H.d_cres_idx + ca, 2 * HD.KQ, d_coeffs, H.d_cres_buf + ca * 2 * HD.KQ, false,
                           s));
    }
  }
  QCK(cudaEventRecord(ev[10], s));
  QCK(cudaGetLastError());
  H.timed_overlap = false;
  H.last_launches = L;
}

void create(Handle& H, const qbxg_config& cfg, const qbxg_geometry& g, const qbxg_plan* plan, int device,
            int nranks = 1, int rank = 0, bool sharded = false) {
  check_device();
  H.gather = sharded || nranks > 1;
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("qbxg_create: bad rank / n_ranks");
  {
    qbxg_plan_view V0;
    if (qbxg_plan_view_get(plan, &V0) != QBXG_OK) throw InvalidArgument(get_last_error());
    H.nranks = nranks;
    H.rank = rank;
    H.cuts.assign(nranks + 1, 0);
    H.mask.assign(V0.n_boxes, 0);
    if (qbxg_plan_shard(plan, nranks, rank, H.cuts.data(), H.mask.data()) != QBXG_OK)
      throw InvalidArgument(get_last_error());
  }
  if (cfg.kernel != QBXG_KERNEL_LAPLACE_SL && cfg.kernel != QBXG_KERNEL_LAPLACE_SL_DL &&
      cfg.kernel != QBXG_KERNEL_HELMHOLTZ_SL && cfg.kernel != QBXG_KERNEL_HELMHOLTZ_SL_DL)
    throw InvalidArgument("qbxg_create: unknown kernel");
  H.helm = cfg.kernel == QBXG_KERNEL_HELMHOLTZ_SL || cfg.kernel == QBXG_KERNEL_HELMHOLTZ_SL_DL;
  if (H.helm && (cfg.p_fmm > 20 || cfg.p_qbx > 6))
    throw InvalidArgument("qbxg_create: Helmholtz supports p_fmm <= 20, p_qbx <= 6");
  if (H.helm && !(cfg.helmholtz_k > 0 && std::isfinite(cfg.helmholtz_k)))
    throw InvalidArgument("qbxg_create: Helmholtz needs a positive wavenumber");
  if (cfg.p_fmm > 21) throw InvalidArgument("qbxg_create: p_fmm > 21 not supported on the GPU path");
  if (cfg.p_qbx > 8) throw InvalidArgument("qbxg_create: p_qbx > 8 not supported on the GPU path");
  qbxg_plan_view V;
  if (qbxg_plan_view_get(plan, &V) != QBXG_OK) throw InvalidArgument(get_last_error());
  if (V.n_sources != g.n_sources || V.n_centers != g.n_centers || V.n_targets != g.n_targets)
    throw InvalidArgument("qbxg_create: plan was built from a different geometry");
  H.device = device;
  QCK(cudaSetDevice(device));
  dev::upload_constants();
  dev::set_smem_limits();
  // the main stream outranks the side stream: with the near field forked beside the
  // far-field chain, the chain's CTAs are placed first as SMs free up and the near field's
  // many short CTAs fill what the chain leaves idle (small tree-shift levels, kernel tails)
  int prio_lo = 0, prio_hi = 0;
  QCK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  QCK(cudaStreamCreateWithPriority(&H.stream, cudaStreamNonBlocking, prio_hi));
  for (auto& e : H.ev) QCK(cudaEventCreate(&e));
  for (auto& e : H.evx) QCK(cudaEventCreate(&e));
  // near field beside the far-field chain: off by default on one GPU (both live on the
  // fp64 pipe; the sequential apply measured as fast), always on for sharded applies
  // (it hides the multipole exchange); qbxg_set_overlap opts in
  H.overlap = false;
  H.debug_sync = std::getenv("QBXG_DEBUG_SYNC") != nullptr;
  QCK(cudaStreamCreateWithPriority(&H.side, cudaStreamNonBlocking, prio_lo));
  QCK(cudaEventCreateWithFlags(&H.fork_ev, cudaEventDisableTiming));
  QCK(cudaEventCreateWithFlags(&H.join_ev, cudaEventDisableTiming));
  cudaStream_t s = H.stream;
  auto& O = H.owned;
  H.cfg = cfg;
  H.ns = g.n_sources;
  H.nc = g.n_centers;
  H.nt = g.n_targets;
  H.nconv = V.n_conv_targets;
  H.nb = V.n_boxes;
  H.nlev = V.n_levels;
  const int nb = H.nb;
  const int p = cfg.p_fmm, q = cfg.p_qbx;
  dev::DevData& D = H.D;
  D.p = p;
  D.q = q;
  D.kp = dev::hsize(p);
  D.kq = dev::hsize(q);
  D.ktab_m2l = dev::hsize(2 * p);
  D.dipole = cfg.kernel == QBXG_KERNEL_LAPLACE_SL_DL ? 1 : 0;

  // --- tree
  std::vector<double4> box(nb);
  for (int b = 0; b < nb; ++b)
    box[b] = make_double4(V.box_center[3 * b], V.box_center[3 * b + 1], V.box_center[3 * b + 2], V.box_radius[b]);
  D.box = dupload(O, box, s);
  D.child_starts = dupload(O, std::vector<int>(V.child_starts, V.child_starts + nb + 1), s);
  D.children = dupload(O, std::vector<int>(V.children, V.children + V.child_starts[nb]), s);
  D.parent = dupload(O, std::vector<int>(V.box_parent, V.box_parent + nb), s);
  auto up_i = [&](const int32_t* a) { return dupload(O, std::vector<int>(a, a + nb), s); };
  D.src_own_start = up_i(V.src_own_start);
  D.src_own_count = up_i(V.src_own_count);
  D.ctr_own_start = up_i(V.ctr_own_start);
  D.ctr_own_count = up_i(V.ctr_own_count);
  D.tgt_own_start = up_i(V.tgt_own_start);
  D.tgt_own_count = up_i(V.tgt_own_count);

  // --- particles (box-sorted)
  std::vector<double4> src(H.ns), ctr(H.nc), tgt(H.nconv);
  for (int64_t i = 0; i < H.ns; ++i) {
    const int64_t o = V.src_perm[i];
    src[i] = make_double4(g.source_pos[3 * o], g.source_pos[3 * o + 1], g.source_pos[3 * o + 2], 0.0);
  }
  for (int64_t i = 0; i < H.nc; ++i) {
    const int64_t o = V.ctr_perm[i];
    ctr[i] = make_double4(g.center_pos[3 * o], g.center_pos[3 * o + 1], g.center_pos[3 * o + 2], g.center_radius[o]);
  }
  for (int64_t i = 0; i < H.nconv; ++i) {
    const int64_t o = V.tgt_perm[i];
    tgt[i] = make_double4(g.target_pos[3 * o], g.target_pos[3 * o + 1], g.target_pos[3 * o + 2], 0.0);
  }
  D.src = dupload(O, src, s);
  D.mu = D.dipole ? dalloc<double4>(O, H.ns) : nullptr;
  D.ctr = dupload(O, ctr, s);
  D.tgt = dupload(O, tgt, s);
  H.d_src_perm = dupload(O, std::vector<int>(V.src_perm, V.src_perm + H.ns), s);
  H.d_ctr_perm = dupload(O, std::vector<int>(V.ctr_perm, V.ctr_perm + H.nc), s);
  H.d_tgt_perm = dupload(O, std::vector<int>(V.tgt_perm, V.tgt_perm + H.nconv), s);
  {
    std::vector<int> tb(H.nconv), cs(H.nc);
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < V.tgt_own_count[b]; ++j) tb[V.tgt_own_start[b] + j] = b;
    for (int64_t i = 0; i < H.nc; ++i) cs[V.ctr_perm[i]] = int(i);
    H.d_tgt_box = dupload(O, tb, s);
    H.d_ctr_sorted = dupload(O, cs, s);
    H.d_assoc = dupload(O, std::vector<int>(g.association, g.association + H.nt), s);
    H.d_tpos = dupload(O, std::vector<double>(g.target_pos, g.target_pos + 3 * H.nt), s);
  }

  // --- expansions
  D.M = dalloc<double2>(O, size_t(nb) * D.kp);
  D.L = dalloc<double2>(O, size_t(nb) * D.kp);
  D.Lc = dalloc<double2>(O, size_t(H.nc) * D.kq);
  D.phi = dalloc<double>(O, H.nconv);
  D.bad = dalloc<unsigned int>(O, 1);
  QCK(cudaMemsetAsync(D.bad, 0, sizeof(unsigned int), s));
  QCK(cudaMallocHost(&H.h_bad, sizeof(unsigned int)));

  // --- lists
  auto lrow = [&](int k, int b, int64_t& a, int64_t& e) {
    a = V.list_starts[k][b];
    e = V.list_starts[k][b + 1];
  };
  std::vector<int64_t> vs(nb + 1, 0);
  std::vector<int2> vent;
  {
    std::vector<int64_t> ns_(nb + 1, 0), xs(nb + 1, 0), ws(nb + 1, 0);
    std::vector<int2> nseg, xseg;
    std::vector<int> wbox;
    const auto& mk = H.mask;
    const int near_lists[3] = {QBXG_LIST_U, QBXG_LIST_W_CLOSE, QBXG_LIST_X_CLOSE};
    for (int b = 0; b < nb; ++b) {
      int64_t a, e;
      if ((V.box_flags[b] & QBXG_BOX_TARGET) && (mk[b] & QBXG_SHARD_OWN)) {
        for (int li : near_lists) {
          lrow(li, b, a, e);
          for (int64_t i = a; i < e; ++i) {
            const int d = V.list_boxes[li][i];
            if (V.src_own_count[d] > 0) nseg.push_back(make_int2(V.src_own_start[d], V.src_own_count[d]));
          }
        }
      }
      ns_[b + 1] = int64_t(nseg.size());
      lrow(QBXG_LIST_X_FAR, b, a, e);
      if (!(mk[b] & QBXG_SHARD_DOWN)) e = a;
      for (int64_t i = a; i < e; ++i) {
        const int d = V.list_boxes[QBXG_LIST_X_FAR][i];
        if (V.src_own_count[d] > 0) xseg.push_back(make_int2(V.src_own_start[d], V.src_own_count[d]));
      }
      xs[b + 1] = int64_t(xseg.size());
      lrow(QBXG_LIST_V, b, a, e);
      if (!(mk[b] & QBXG_SHARD_DOWN)) e = a;
      for (int64_t i = a; i < e; ++i) {
        const int d = V.list_boxes[QBXG_LIST_V][i];
        int dd[3];
        for (int k = 0; k < 3; ++k)
          dd[k] = int(std::lround((V.box_center[3 * b + k] - V.box_center[3 * d + k]) / (2.0 * V.box_radius[b])));
        if (std::abs(dd[0]) > 5 || std::abs(dd[1]) > 5 || std::abs(dd[2]) > 5)
          throw InvalidArgument("qbxg_create: List 2 offset outside [-5,5]^3");
        vent.push_back(make_int2(d, ((dd[0] + 5) * 11 + (dd[1] + 5)) * 11 + (dd[2] + 5)));
      }
      vs[b + 1] = int64_t(vent.size());
      lrow(QBXG_LIST_W_FAR, b, a, e);
      if (!(mk[b] & QBXG_SHARD_OWN)) e = a;
      for (int64_t i = a; i < e; ++i) wbox.push_back(V.list_boxes[QBXG_LIST_W_FAR][i]);
      ws[b + 1] = int64_t(wbox.size());
    }
    D.near_starts = dupload(O, ns_, s);
    D.near_seg = dupload(O, nseg, s);
    {
      // flattened near-source list of each box with centres (the P2QBXL kernel's input)
      std::vector<int> nn(nb, 0);
      std::vector<int64_t> off(nb + 1, 0);
      for (int b = 0; b < nb; ++b) {
        for (int64_t i = ns_[b]; i < ns_[b + 1]; ++i) nn[b] += nseg[i].y;
        off[b + 1] = off[b] + (V.ctr_own_count[b] > 0 ? nn[b] : 0);
      }
      std::vector<int> flat(std::max<int64_t>(off[nb], 1));
#pragma omp parallel for schedule(dynamic, 64)
      for (int b = 0; b < nb; ++b) {
        if (V.ctr_own_count[b] == 0) continue;
        int64_t o = off[b];
        for (int64_t i = ns_[b]; i < ns_[b + 1]; ++i)
          for (int j = 0; j < nseg[i].y; ++j) flat[o++] = nseg[i].x + j;
      }
      D.near_nsrc = dupload(O, nn, s);
      D.near_off = dupload(O, off, s);
      D.near_src = dupload(O, flat, s);
      QCK(cudaStreamSynchronize(s));
    }
    D.xfar_starts = dupload(O, xs, s);
    D.xfar_seg = dupload(O, xseg, s);
    D.v_starts = dupload(O, vs, s);
    D.v_ent = dupload(O, vent, s);
    D.wfar_starts = dupload(O, ws, s);
    D.wfar_box = dupload(O, wbox, s);

    // work lists
    std::vector<int> leaves, cb, tb, vb, wb, wtb, xb;
    for (int b = 0; b < nb; ++b) {
      const bool leaf = V.box_flags[b] & QBXG_BOX_LEAF;
      const bool own = mk[b] & QBXG_SHARD_OWN;
      if (leaf && V.src_own_count[b] > 0 && own) leaves.push_back(b);
      if (V.ctr_own_count[b] > 0 && own) cb.push_back(b);
      if (V.tgt_own_count[b] > 0 && ns_[b + 1] > ns_[b] && own) tb.push_back(b);
      if (vs[b + 1] > vs[b]) vb.push_back(b);
      if (ws[b + 1] > ws[b] && V.ctr_own_count[b] > 0) wb.push_back(b);
      if (ws[b + 1] > ws[b] && V.tgt_own_count[b] > 0) wtb.push_back(b);
      if (xs[b + 1] > xs[b]) xb.push_back(b);
    }
    // conventional targets with an empty near list still need phi = 0
    H.d_leaves = dupload(O, leaves, s);
    H.n_leaves = int(leaves.size());
    H.d_ctr_boxes = dupload(O, cb, s);
    H.n_ctr_boxes = int(cb.size());
    {
      // near-field launch order: decreasing (centres x near sources), ties in box order;
      // every CTA owns its centres, so the order changes no result
      std::vector<int64_t> cost(nb, 0);
      for (int b : cb) {
        int64_t nsrc = 0;
        for (int64_t i = ns_[b]; i < ns_[b + 1]; ++i) nsrc += nseg[i].y;
        cost[b] = nsrc * int64_t(V.ctr_own_count[b]);
      }
      std::vector<int> nbx(cb);
      std::stable_sort(nbx.begin(), nbx.end(), [&](int a, int b) { return cost[a] > cost[b]; });
      H.d_near_boxes = dupload(O, nbx, s);
    }
    H.d_tgt_boxes = dupload(O, tb, s);
    H.n_tgt_boxes = int(tb.size());
    H.d_v_boxes = dupload(O, vb, s);
    H.n_v_boxes = int(vb.size());
    H.d_wfar_boxes = dupload(O, wb, s);
    H.n_wfar_boxes = int(wb.size());
    H.d_wfar_tboxes = dupload(O, wtb, s);
    H.n_wfar_tboxes = int(wtb.size());
    std::vector<int> cbox(H.nc), all, fw, eval_assoc, eval_conv;
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < V.ctr_own_count[b]; ++j) cbox[V.ctr_own_start[b] + j] = b;
    for (int b : cb)
      for (int j = 0; j < V.ctr_own_count[b]; ++j) all.push_back(V.ctr_own_start[b] + j);
    {
      std::vector<int> cs_of(H.nc);
      for (int64_t i = 0; i < H.nc; ++i) cs_of[V.ctr_perm[i]] = int(i);
      for (int64_t t = 0; t < H.nt; ++t)
        if (g.association[t] >= 0 && (mk[cbox[cs_of[g.association[t]]]] & QBXG_SHARD_OWN)) eval_assoc.push_back(int(t));
      for (int b = 0; b < nb; ++b)
        if (mk[b] & QBXG_SHARD_OWN)
          for (int j = 0; j < V.tgt_own_count[b]; ++j) eval_conv.push_back(V.tgt_own_start[b] + j);
    }
    H.d_eval_assoc = dupload(O, eval_assoc, s);
    H.n_eval_assoc = int(eval_assoc.size());
    H.d_eval_conv = dupload(O, eval_conv, s);
    H.n_eval_conv = int(eval_conv.size());
    H.n_own_ctr = int(all.size());
    for (int b : wb)
      for (int j = 0; j < V.ctr_own_count[b]; ++j) fw.push_back(V.ctr_own_start[b] + j);
    H.d_ctr_box = dupload(O, cbox, s);
    H.d_flat_all = dupload(O, all, s);
    if (H.gather) {
      // result all-gather layout: rank-major segments of every rank's owned targets
      // (associated in target order, then conventional in box order) and centres
      auto owner = [&](int b) {
        return int(std::upper_bound(H.cuts.begin(), H.cuts.end(), int32_t(b)) - H.cuts.begin()) - 1;
      };
      std::vector<int> cs_of(H.nc);
      for (int64_t i = 0; i < H.nc; ++i) cs_of[V.ctr_perm[i]] = int(i);
      std::vector<std::vector<int>> rt(nranks), rc(nranks);
      for (int64_t t = 0; t < H.nt; ++t)
        if (g.association[t] >= 0) rt[owner(cbox[cs_of[g.association[t]]])].push_back(int(t));
      for (int b = 0; b < nb; ++b) {
        const int r = owner(b);
        for (int j = 0; j < V.tgt_own_count[b]; ++j) rt[r].push_back(V.tgt_perm[V.tgt_own_start[b] + j]);
        for (int j = 0; j < V.ctr_own_count[b]; ++j) rc[r].push_back(V.ctr_perm[V.ctr_own_start[b] + j]);
      }
      std::vector<int> ti, ci;
      H.res_off.assign(1, 0);
      H.cres_off.assign(1, 0);
      for (int r = 0; r < nranks; ++r) {
        ti.insert(ti.end(), rt[r].begin(), rt[r].end());
        ci.insert(ci.end(), rc[r].begin(), rc[r].end());
        H.res_off.push_back(int64_t(ti.size()));
        H.cres_off.push_back(int64_t(ci.size()));
      }
      if (int64_t(ti.size()) != H.nt || int64_t(ci.size()) != H.nc)
        throw InvalidArgument("qbxg_create_sharded: targets / centres not partitioned by the shard cuts");
      H.d_res_idx = dupload(O, ti, s);
      H.d_cres_idx = dupload(O, ci, s);
      // (Helmholtz: complex potentials, full (q+1)^2 tables of complex centre coefficients)
      H.d_res_buf = dalloc<double>(O, std::max<int64_t>(H.nt, 1) * (H.helm ? 2 : 1));
      H.d_cres_buf = dalloc<double>(O, std::max<int64_t>(H.nc, 1) * 2 * (H.helm ? (H.cfg.p_qbx + 1) * (H.cfg.p_qbx + 1) : D.kq));
      QCK(cudaStreamSynchronize(s));
    }
    {
      std::vector<int2> l3;
      size_t i = 0;
      while (i < all.size()) {
        const size_t first = i;
        int nbx = 0, last = -1;
        while (i < all.size() && i - first < size_t(dev::kL3Threads)) {
          const int bx = cbox[all[i]];
          if (bx != last) {
            if (nbx == dev::kL3Boxes) break;
            ++nbx;
            last = bx;
          }
          ++i;
        }
        l3.push_back(make_int2(int(first), int(i - first)));
      }
      H.d_l3_ctas = dupload(O, l3, s);
      H.n_l3_ctas = int(l3.size());
    }
    H.d_flat_wfar = dupload(O, fw, s);
    H.n_flat_wfar = int(fw.size());
    // (centre, W_far box) pairs, centre-major, chunked to bound the staging buffer
    {
      const int64_t cap_pairs = int64_t(1) << 24;
      std::vector<int2> pairs;
      std::vector<int> centres, starts;
      int64_t total = 0, max_chunk = 0;
      auto flush = [&]() {
        if (centres.empty()) return;
        dev::PairChunk C;
        C.n_pairs = int(pairs.size());
        C.pair_base = starts.front();
        C.n_centres = int(centres.size());
        starts.push_back(int(total));
        C.pairs = dupload(O, pairs, s);
        {
          std::vector<int> perm(pairs.size());
          for (size_t i = 0; i < perm.size(); ++i) perm[i] = int(i);
          std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return pairs[a].y < pairs[b].y; });
          std::vector<int2> ctas;
          size_t i = 0;
          while (i < perm.size()) {
            const size_t first = i;
            int nbx = 0, last = -1;
            while (i < perm.size() && i - first < size_t(dev::kW3Threads)) {
              const int bx = pairs[perm[i]].y;
              if (bx != last) {
                if (nbx == dev::kW3Boxes) break;
                ++nbx;
                last = bx;
              }
              ++i;
            }
            ctas.push_back(make_int2(int(first), int(i - first)));
          }
          C.perm = dupload(O, perm, s);
          C.ctas = dupload(O, ctas, s);
          C.n_ctas = int(ctas.size());
        }
        C.centres = dupload(O, centres, s);
        C.starts = dupload(O, starts, s);
        H.wpairs.chunks.push_back(C);
        max_chunk = std::max<int64_t>(max_chunk, int64_t(pairs.size()));
        pairs.clear();
        centres.clear();
        starts.clear();
      };
      for (int b : wb) {
        const int64_t a = ws[b], e = ws[b + 1];
        for (int j = 0; j < V.ctr_own_count[b]; ++j) {
          if (int64_t(pairs.size()) + (e - a) > cap_pairs) flush();
          const int cs = V.ctr_own_start[b] + j;
          centres.push_back(cs);
          starts.push_back(int(total));
          for (int64_t i = a; i < e; ++i) pairs.push_back(make_int2(cs, wbox[i]));
          total += e - a;
        }
      }
      flush();
      H.wpairs.temp = dalloc<double2>(O, size_t(std::max<int64_t>(max_chunk, 1)) * D.kq);
    }
    {
      // P2L launch order: decreasing X_far source count (one CTA per box, so the order
      // changes no result; no tail of heavy boxes)
      std::vector<int64_t> cost(nb, 0);
      for (int b : xb)
        for (int64_t i = xs[b]; i < xs[b + 1]; ++i) cost[b] += xseg[i].y;
      std::stable_sort(xb.begin(), xb.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    }
    H.d_xfar_boxes = dupload(O, xb, s);
    H.n_xfar_boxes = int(xb.size());
  }

  if (H.helm) {
    helm_setup(H, V, vs, vent, s);
    QCK(cudaGetLastError());
    QCK(cudaStreamSynchronize(s));
    return;
  }
  // --- operator tables
  double2* m2l_tab = dalloc<double2>(O, size_t(1331) * D.ktab_m2l);
  double2* oct_m2m = dalloc<double2>(O, size_t(8) * D.kp);
  double2* oct_l2l = dalloc<double2>(O, size_t(8) * D.kp);
  dev::launch_tables(D, m2l_tab, oct_m2m, oct_l2l, s);
  D.m2l_tab = m2l_tab;
  D.oct_m2m = oct_m2m;
  D.oct_l2l = oct_l2l;

  // --- host-apply staging
  H.d_w = dalloc<double>(O, H.ns);
  H.d_mu_in = D.dipole ? dalloc<double>(O, 3 * H.ns) : nullptr;
  H.d_pot = dalloc<double>(O, H.nt);
  H.d_coeffs = dalloc<double>(O, size_t(H.nc) * 2 * D.kq);

  build_m2l(H, V, vs, vent, s);
  QCK(cudaGetLastError());
  QCK(cudaStreamSynchronize(s));
}

// ---- NCCL, loaded at run time (libnccl.so.2: torch's or the system's) ----
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (n.lib) {
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.lib, "ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.lib, "ncclCommInitRank"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.lib, "ncclCommDestroy"));
      n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(dlsym(n.lib, "ncclBroadcast"));
      n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.lib, "ncclGroupStart"));
      n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.lib, "ncclGroupEnd"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.lib, "ncclGetErrorString"));
    }
  }
  if (!n.lib || !n.GetUniqueId || !n.CommInitRank || !n.Broadcast || !n.GroupStart || !n.GroupEnd)
    throw NcclError("libnccl.so.2 not loadable");
  return n;
}

// Box multipoles as rows of doubles (Laplace: half tables; Helmholtz: full complex tables)
double* m_ptr(Handle& H) { return reinterpret_cast<double*>(H.helm ? H.HD.M : H.D.M); }
size_t m_row(const Handle& H) { return size_t(2) * (H.helm ? H.HD.KP : H.D.kp); }
// doubles per target potential / per centre in the result exchange
int pot_w(const Handle& H) { return H.helm ? 2 : 1; }
int coef_w(const Handle& H) { return 2 * (H.helm ? H.HD.KQ : H.D.kq); }

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl().GetErrorString(r));
}

// Multipole exchange after the owned upward pass: rank r broadcasts the rows
// of its box range [cuts[r], cuts[r+1]) of M (in place) to every rank.
void exchange_nccl(Handle& H, cudaStream_t s) {
  Nccl& n = nccl();
  auto comm = static_cast<ncclComm_t>(H.nccl_comm);
  const size_t row = m_row(H);
  nck(n.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < H.nranks; ++r) {
    const size_t a = size_t(H.cuts[r]), b = size_t(H.cuts[r + 1]);
    if (b <= a) continue;
    double* p = m_ptr(H) + a * row;
    nck(n.Broadcast(p, p, (b - a) * row, ncclFloat64, r, comm, s), "ncclBroadcast");
  }
  nck(n.GroupEnd(), "ncclGroupEnd");
}

// phase bit 1: density gather, P2M, M2M of the rank's subtrees.
// phase bit 2: M2M of straddling boxes, then Stages 3-9 for the rank's boxes.
// near: NEAR_INLINE runs P2QBXL on s before M2L; NEAR_DONE skips it (the batched path
// ran it); NEAR_SIDE forks it onto the side stream right after the gather (phase 1) --
// it needs only the gathered sources -- and joins it before W far, the first stage
// that adds into the centre locals, so it overlaps the upward pass, the multipole
// exchange of a sharded apply and M2L / P2L / L2L.
enum NearMode { NEAR_INLINE = 0, NEAR_DONE = 1, NEAR_SIDE = 2 };

void run_device(Handle& H, const double* d_w, const double* d_mu, double* d_pot, double* d_coeffs, cudaStream_t s,
                int phase, NearMode near = NEAR_INLINE) {
  dev::DevData& D = H.D;
  if (D.dipole && !d_mu && (phase & 1)) throw InvalidArgument("qbxg_apply: Laplace SL+DL requires dipole moments");
  int L = (phase & 1) ? 0 : H.last_launches;
  int stage_no = 0;
  auto chk = [&](int k) {
    if (k < 0) throw InvalidArgument("qbxg_apply: unsupported order");
    L += k;
    ++stage_no;
    if (H.debug_sync) {  // localise asynchronous faults to the launch that caused them
      cudaError_t e = cudaStreamSynchronize(s);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error after launch group ") + std::to_string(stage_no) + " (phase " +
                        std::to_string(phase) + "): " + cudaGetErrorString(e));
    }
  };
  auto& ev = H.ev;
  if (phase & 1) {
    QCK(cudaEventRecord(ev[0], s));
    chk(dev::launch_gather(D, int(H.ns), H.d_src_perm, d_w, d_mu, s));
    if (near == NEAR_SIDE) {
      QCK(cudaEventRecord(H.fork_ev, s));
      QCK(cudaStreamWaitEvent(H.side, H.fork_ev, 0));
      QCK(cudaEventRecord(H.evx[0], H.side));
      chk(dev::launch_near_qbx(D, H.d_near_boxes, H.n_ctr_boxes, H.side));
      QCK(cudaEventRecord(H.evx[1], H.side));
      QCK(cudaEventRecord(H.join_ev, H.side));
    }
    QCK(cudaMemsetAsync(D.M, 0, size_t(H.nb) * D.kp * sizeof(double2), s));
    QCK(cudaMemsetAsync(D.L, 0, size_t(H.nb) * D.kp * sizeof(double2), s));
    QCK(cudaMemsetAsync(D.phi, 0, size_t(std::max<int64_t>(H.nconv, 1)) * sizeof(double), s));
    QCK(cudaMemsetAsync(D.bad, 0, sizeof(unsigned int), s));
    QCK(cudaEventRecord(ev[1], s));
    chk(dev::launch_p2m(D, H.d_leaves, H.n_leaves, s));
    QCK(cudaEventRecord(ev[2], s));
    for (int l = H.nlev - 2; l >= 0; --l)
      chk(dev::launch_shift_level(H.m2l, H.m2m_levels[l], H.ops_m2m, D.M, D.kp, false, s));
    H.last_launches = L;
  }
  if (!(phase & 2)) return;
  // boxes whose subtree spans ranks: recomputed identically by every rank once
  // the owned multipoles have been exchanged (no-op for a single rank)
  if (H.nranks > 1)
    for (int l = H.nlev - 2; l >= 0; --l)
      chk(dev::launch_shift_level(H.m2l, H.m2m_straddle[l], H.ops_m2m, D.M, D.kp, false, s));
  QCK(cudaEventRecord(ev[3], s));
  // Order: near field | M2L | P2L | L2L | W far | L2QBXL | eval
  if (near == NEAR_INLINE) chk(dev::launch_near_qbx(D, H.d_near_boxes, H.n_ctr_boxes, s));
  chk(dev::launch_near_p2p(D, H.d_tgt_boxes, H.n_tgt_boxes, s));
  QCK(cudaEventRecord(ev[4], s));
  chk(dev::launch_m2l(H.m2l, D, s));
  QCK(cudaEventRecord(ev[5], s));
  chk(dev::launch_p2l(D, H.d_xfar_boxes, H.n_xfar_boxes, s));
  QCK(cudaEventRecord(H.evx[2], s));
  for (int l = 1; l < H.nlev; ++l) chk(dev::launch_shift_level(H.m2l, H.l2l_levels[l], H.ops_l2l, D.L, D.kp, true, s));
  QCK(cudaEventRecord(H.evx[3], s));
  if (near == NEAR_SIDE) QCK(cudaStreamWaitEvent(s, H.join_ev, 0));
  chk(dev::launch_m2qbxl_pairs(D, H.wpairs, s));
  chk(dev::launch_m2p(D, H.d_wfar_tboxes, H.n_wfar_tboxes, s));
  QCK(cudaEventRecord(ev[6], s));
  H.timed_overlap = near == NEAR_SIDE;
  chk(dev::launch_l2qbxl3(D, H.d_flat_all, H.d_l3_ctas, H.n_l3_ctas, H.d_ctr_box, s));
  QCK(cudaEventRecord(ev[9], s));
  if (H.gather) {  // targets / centres of other ranks stay zero until the result exchange
    QCK(cudaMemsetAsync(d_pot, 0, size_t(std::max<int64_t>(H.nt, 1)) * sizeof(double), s));
    if (d_coeffs) QCK(cudaMemsetAsync(d_coeffs, 0, size_t(std::max<int64_t>(H.nc, 1)) * 2 * D.kq * sizeof(double), s));
  }
  chk(dev::launch_eval(D, H.n_eval_assoc, H.d_eval_assoc, H.d_tpos, H.d_assoc, H.d_ctr_sorted, H.n_eval_conv,
                       H.d_eval_conv, H.d_tgt_perm, H.d_tgt_box, d_pot, s));
  if (d_coeffs) chk(dev::launch_centre_out(D, H.n_own_ctr, H.d_flat_all, H.d_ctr_perm, d_coeffs, s));
  if (H.gather) {  // the rank's results into its segment of the gather buffers
    const int64_t a = H.res_off[H.rank], e = H.res_off[H.rank + 1];
    chk(dev::launch_pack(int(e - a), H.d_res_idx + a, 1, d_pot, H.d_res_buf + a, false, s));
    if (d_coeffs) {
      const int64_t ca = H.cres_off[H.rank], ce = H.cres_off[H.rank + 1];
      chk(dev::launch_pack(int(ce - ca), H.d_cres_idx + ca, 2 * D.kq, d_coeffs, H.d_cres_buf + ca * 2 * D.kq, false,
                           s));
    }
  }
  QCK(cudaEventRecord(ev[10], s));
  QCK(cudaGetLastError());
  H.last_launches = L;
}

// Results of a sharded apply: every rank broadcasts its packed segment of potentials
// (and centre coefficients) to all ranks in one NCCL group -- an all-gather of owned
// values, N_T doubles in total, instead of an all-reduce of N_T-long zero-padded
// vectors -- and scatters the gathered values into caller order.
void exchange_results_nccl(Handle& H, double* d_pot, double* d_coeffs, cudaStream_t s) {
  Nccl& n = nccl();
  auto comm = static_cast<ncclComm_t>(H.nccl_comm);
  const int w = coef_w(H), pw = pot_w(H);
  nck(n.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < H.nranks; ++r) {
    const int64_t a = H.res_off[r], e = H.res_off[r + 1];
    if (e > a)
      nck(n.Broadcast(H.d_res_buf + a * pw, H.d_res_buf + a * pw, size_t(e - a) * pw, ncclFloat64, r, comm, s),
          "ncclBroadcast");
    if (d_coeffs) {
      const int64_t ca = H.cres_off[r], ce = H.cres_off[r + 1];
      if (ce > ca)
        nck(n.Broadcast(H.d_cres_buf + ca * w, H.d_cres_buf + ca * w, size_t(ce - ca) * w, ncclFloat64, r, comm, s),
            "ncclBroadcast");
    }
  }
  nck(n.GroupEnd(), "ncclGroupEnd");
  dev::launch_pack(int(H.nt), H.d_res_idx, pw, d_pot, H.d_res_buf, true, s);
  if (d_coeffs) dev::launch_pack(int(H.nc), H.d_cres_idx, w, d_coeffs, H.d_cres_buf, true, s);
}

// One whole apply.  Sharded: owned upward pass (near field forked beside it), multipole
// exchange (NCCL), straddling M2M, downward + QBX stages, result all-gather.
void full_apply(Handle& H, const double* d_w, const double* d_mu, double* d_pot, double* d_coeffs, cudaStream_t s) {
  if (H.gather && !H.nccl_comm)
    throw InvalidArgument("sharded handle: attach NCCL (qbxg_nccl_attach) or drive qbxg_apply_phase");
  if (H.helm) {  // complex interleaved arrays; no side stream
    if (!H.gather) return run_helm(H, d_w, d_mu, d_pot, d_coeffs, s);
    run_helm(H, d_w, d_mu, d_pot, d_coeffs, s, 1);
    exchange_nccl(H, s);
    run_helm(H, d_w, d_mu, d_pot, d_coeffs, s, 2);
    exchange_results_nccl(H, d_pot, d_coeffs, s);
    return;
  }
  if (!H.gather) {
    run_device(H, d_w, d_mu, d_pot, d_coeffs, s, 3, H.overlap ? NEAR_SIDE : NEAR_INLINE);
    return;
  }
  run_device(H, d_w, d_mu, d_pot, d_coeffs, s, 1, NEAR_SIDE);
  exchange_nccl(H, s);
  run_device(H, d_w, d_mu, d_pot, d_coeffs, s, 2, NEAR_SIDE);
  exchange_results_nccl(H, d_pot, d_coeffs, s);
}

// Reference error semantics inside the apply (kernels.cpp:58-71): Stage 9
// flags any non-finite potential or centre coefficient; on the error path the near
// lists are scanned for the coincident (centre | target, source) pair, which is named
// the way the reference's direct_sum names it.  Costs one 4-byte read per apply.
void check_domain(Handle& H, cudaStream_t s) {
  dev::DevData& D = H.D;
  QCK(cudaMemcpyAsync(H.h_bad, D.bad, sizeof(unsigned int), cudaMemcpyDeviceToHost, s));
  QCK(cudaStreamSynchronize(s));
  if (*H.h_bad == 0) return;
  const unsigned kind = *H.h_bad;
  QCK(cudaMemsetAsync(D.bad, 0, sizeof(unsigned int), s));
  unsigned long long* d_key = dalloc<unsigned long long>(H.owned, 1);
  QCK(cudaMemsetAsync(d_key, 0xff, sizeof(unsigned long long), s));
  dev::launch_find_coincident(D, int(H.nc), H.d_ctr_box, H.d_ctr_perm, int(H.nconv), H.d_tgt_box, H.d_tgt_perm,
                              H.d_src_perm, d_key, s);
  unsigned long long key = 0;
  QCK(cudaMemcpyAsync(&key, d_key, sizeof(key), cudaMemcpyDeviceToHost, s));
  QCK(cudaStreamSynchronize(s));
  cudaFree(d_key);
  H.owned.erase(std::find(H.owned.begin(), H.owned.end(), static_cast<void*>(d_key)));
  if (key != ~0ull) {
    const bool ctr = (key >> 62) == 0;
    const long long id = (long long)((key >> 31) & 0x7fffffffull), src = (long long)(key & 0x7fffffffull);
    throw DomainError(std::string("qbxg_apply: ") + (ctr ? "QBX center " : "target ") + std::to_string(id) +
                      " coincides with source " + std::to_string(src));
  }
  throw DomainError(std::string("qbxg_apply: non-finite ") + ((kind & 1) ? "potential" : "center coefficient") +
                    " (no coincident near-field pair: overflow or non-finite input)");
}

// R densities (rhs-major device arrays).  Densities go through the near field NR
// at a time (one harmonic table per pair feeds NR densities); every other stage
// runs per density on its own completed centre locals.  Results equal R single
// applies up to rounding.  Sharded handles loop over full applies.
void batch_apply(Handle& H, int R, const double* d_w, const double* d_mu, double* d_pot, double* d_coeffs,
                 cudaStream_t s) {
  dev::DevData& D = H.D;
  // SL+DL: the single-density near field (V-form, kernels.cu near_pair_dip) costs less per
  // density than the shared harmonic table plus one contraction per density (76.9 vs 81.6 ms
  // per density at config 1), so only the single layer is batched through the near field
  const int NR = D.dipole ? 1 : dev::near_batch_width(D.q);
  if (H.gather || NR < 2 || R < 2) {
    for (int r = 0; r < R; ++r)
      full_apply(H, d_w + size_t(r) * H.ns, d_mu ? d_mu + size_t(r) * 3 * H.ns : nullptr, d_pot + size_t(r) * H.nt,
                 d_coeffs ? d_coeffs + size_t(r) * H.nc * 2 * D.kq : nullptr, s);
    return;
  }
  if (H.bnr < NR) {
    H.d_bw = dalloc<double>(H.owned, size_t(NR) * H.ns);
    H.d_bmu = dalloc<double4>(H.owned, size_t(NR) * H.ns);
    H.d_bLc = dalloc<double2>(H.owned, size_t(NR) * std::max<int64_t>(H.nc, 1) * D.kq);
    H.bnr = NR;
  }
  double2* const lc_single = D.Lc;
  int L = 0;
  int r0 = 0;
  for (; r0 + NR <= R; r0 += NR) {
    dev::launch_gather_batch(D, int(H.ns), NR, H.d_src_perm, d_w + size_t(r0) * H.ns,
                             d_mu ? d_mu + size_t(r0) * 3 * H.ns : nullptr, H.d_bw, H.d_bmu, s);
    if (dev::launch_near_qbx_batch(D, H.d_near_boxes, H.n_ctr_boxes, NR, H.d_bw, H.d_bmu, H.ns, H.d_bLc, H.nc, s) < 0)
      throw InvalidArgument("qbxg_apply_batch: unsupported order");
    L += 2;
    for (int k = 0; k < NR; ++k) {
      const int r = r0 + k;
      D.Lc = H.d_bLc + size_t(k) * H.nc * D.kq;
      try {
        run_device(H, d_w + size_t(r) * H.ns, d_mu ? d_mu + size_t(r) * 3 * H.ns : nullptr, d_pot + size_t(r) * H.nt,
                   d_coeffs ? d_coeffs + size_t(r) * H.nc * 2 * D.kq : nullptr, s, 3, NEAR_DONE);
      } catch (...) {
        D.Lc = lc_single;
        throw;
      }
      D.Lc = lc_single;
      L += H.last_launches;
    }
  }
  for (; r0 < R; ++r0) {
    full_apply(H, d_w + size_t(r0) * H.ns, d_mu ? d_mu + size_t(r0) * 3 * H.ns : nullptr, d_pot + size_t(r0) * H.nt,
               d_coeffs ? d_coeffs + size_t(r0) * H.nc * 2 * D.kq : nullptr, s);
    L += H.last_launches;
  }
  H.last_launches = L;
}

void fill_timings(Handle& H, qbxg_timings* t, bool host_copies, int64_t h2d, int64_t d2h) {
  QCK(cudaEventSynchronize(H.ev[host_copies ? 12 : 10]));
  if (!t) return;
  std::memset(t, 0, sizeof(*t));
  auto el = [&](int a, int b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, H.ev[a], H.ev[b]);
    return double(ms);
  };
  auto elx = [&](cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return double(ms);
  };
  t->ms[QBXG_T_P2M] = el(1, 2);
  t->ms[QBXG_T_M2M] = el(2, 3);
  // near: the P2QBXL kernel on whichever stream ran it, plus the conventional-target P2P
  t->ms[QBXG_T_NEAR] = el(3, 4) + (H.timed_overlap ? elx(H.evx[0], H.evx[1]) : 0.0);
  t->ms[QBXG_T_M2L] = el(4, 5);
  t->ms[QBXG_T_P2L] = elx(H.ev[5], H.evx[2]);
  t->ms[QBXG_T_L2L] = elx(H.evx[2], H.evx[3]);
  t->ms[QBXG_T_WFAR] = elx(H.evx[3], H.ev[6]);  // with overlap this includes any wait for the near field
  t->ms[QBXG_T_L2QBXL] = el(6, 9);
  t->ms[QBXG_T_EVAL] = el(9, 10);
  if (host_copies) {
    t->ms[QBXG_T_H2D] = el(11, 0) + el(0, 1);
    t->ms[QBXG_T_D2H] = el(10, 12);
    t->ms[QBXG_T_TOTAL] = el(11, 12);
  } else {
    t->ms[QBXG_T_H2D] = el(0, 1);
    t->ms[QBXG_T_TOTAL] = el(0, 10);
  }
  t->kernel_launches = H.last_launches;
  t->h2d_bytes = h2d;
  t->d2h_bytes = d2h;
}

void validate_sources(int64_t ns, const double* pos, const double* w, const double* mu) {
  for (int64_t i = 0; i < ns; ++i) {
    if (!std::isfinite(pos[3 * i]) || !std::isfinite(pos[3 * i + 1]) || !std::isfinite(pos[3 * i + 2]) ||
        !std::isfinite(w[i]))
      throw InvalidArgument("SourceEnsemble: non-finite entry at index " + std::to_string(i));
    if (mu && (!std::isfinite(mu[3 * i]) || !std::isfinite(mu[3 * i + 1]) || !std::isfinite(mu[3 * i + 2])))
      throw InvalidArgument("SourceEnsemble: non-finite dipole at index " + std::to_string(i));
  }
}

}  // namespace
}  // namespace qbxg

struct qbxg_handle {
  qbxg::Handle h;
};

extern "C" {

int qbxg_device_count(int32_t* out) {
  return qbxg::guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

int qbxg_create(const qbxg_config* cfg, const qbxg_geometry* geom, const qbxg_plan* plan, int32_t device,
                qbxg_handle** out) {
  int st = qbxg::guarded([&] {
    if (!cfg || !geom || !plan || !out) throw qbxg::InvalidArgument("qbxg_create: null argument");
    auto* h = new qbxg_handle;
    try {
      qbxg::create(h->h, *cfg, *geom, plan, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
  if (st == QBXG_ERR_CUDA) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return QBXG_ERR_NO_DEVICE;
    }
  }
  return st;
}

int qbxg_apply_device(qbxg_handle* hp, const double* d_weights, const double* d_dipoles, double* d_out_target_pot,
                      double* d_out_center_coeffs, void* cuda_stream, qbxg_timings* timings) {
  return qbxg::guarded([&] {
    if (!hp || !d_weights || !d_out_target_pot) throw qbxg::InvalidArgument("qbxg_apply_device: null argument");
    auto& H = hp->h;
    if (H.helm) throw qbxg::InvalidArgument("qbxg_apply_device: Helmholtz handle, use qbxg_apply_complex");
    QCK(cudaSetDevice(H.device));
    cudaStream_t s = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : H.stream;
    qbxg::full_apply(H, d_weights, d_dipoles, d_out_target_pot, d_out_center_coeffs, s);
    qbxg::fill_timings(H, timings, false, 0, 0);
    qbxg::check_domain(H, s);
  });
}

int qbxg_create_sharded(const qbxg_config* cfg, const qbxg_geometry* geom, const qbxg_plan* plan, int32_t device,
                        int32_t n_ranks, int32_t rank, qbxg_handle** out) {
  return qbxg::guarded([&] {
    if (!cfg || !geom || !plan || !out) throw qbxg::InvalidArgument("qbxg_create_sharded: null argument");
    auto* h = new qbxg_handle;
    try {
      qbxg::create(h->h, *cfg, *geom, plan, device, n_ranks, rank, true);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int qbxg_apply_phase(qbxg_handle* hp, int32_t phase, const double* d_weights, const double* d_dipoles,
                     double* d_out_target_pot, double* d_out_center_coeffs, void* cuda_stream) {
  return qbxg::guarded([&] {
    if (!hp || phase < 1 || phase > 2) throw qbxg::InvalidArgument("qbxg_apply_phase: bad argument");
    if (phase == 1 && !d_weights) throw qbxg::InvalidArgument("qbxg_apply_phase: null weights");
    if (phase == 2 && !d_out_target_pot) throw qbxg::InvalidArgument("qbxg_apply_phase: null output");
    auto& H = hp->h;
    QCK(cudaSetDevice(H.device));
    cudaStream_t s = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : H.stream;
    if (H.helm)  // complex interleaved device arrays (the layouts of qbxg_apply_complex)
      qbxg::run_helm(H, d_weights, d_dipoles, d_out_target_pot, d_out_center_coeffs, s, phase);
    else
      qbxg::run_device(H, d_weights, d_dipoles, d_out_target_pot, d_out_center_coeffs, s, phase);
    QCK(cudaStreamSynchronize(s));
    if (phase == 2) qbxg::check_domain(H, s);
  });
}

int qbxg_multipole_buffer(qbxg_handle* hp, double** d_multipoles, int64_t* row_doubles, int32_t* cuts) {
  return qbxg::guarded([&] {
    if (!hp || !d_multipoles || !row_doubles) throw qbxg::InvalidArgument("qbxg_multipole_buffer: null argument");
    auto& H = hp->h;
    *d_multipoles = qbxg::m_ptr(H);
    *row_doubles = int64_t(qbxg::m_row(H));
    if (cuts) std::copy(H.cuts.begin(), H.cuts.end(), cuts);
  });
}

int qbxg_exchange_local(qbxg_handle** hs, int32_t n) {
  return qbxg::guarded([&] {
    if (!hs || n < 1) throw qbxg::InvalidArgument("qbxg_exchange_local: bad argument");
    QCK(cudaDeviceSynchronize());  // phase 1 of every rank complete, whatever stream it ran on
    for (int r = 0; r < n; ++r) {
      auto& src = hs[r]->h;
      if (src.nranks != n || src.rank != r) throw qbxg::InvalidArgument("qbxg_exchange_local: handles not rank-ordered");
      const size_t row = qbxg::m_row(src);
      const size_t a = size_t(src.cuts[r]), b = size_t(src.cuts[r + 1]);
      for (int q = 0; q < n; ++q) {
        if (q == r || b <= a) continue;
        auto& dst = hs[q]->h;
        if (dst.helm != src.helm) throw qbxg::InvalidArgument("qbxg_exchange_local: mixed kernels");
        QCK(cudaMemcpy(qbxg::m_ptr(dst) + a * row, qbxg::m_ptr(src) + a * row, (b - a) * row * sizeof(double),
                       cudaMemcpyDefault));
      }
    }
    // device-to-device cudaMemcpy does not wait on the host, and the handles' streams do
    // not synchronise with the default stream: phase 2 must not start before the rows land
    QCK(cudaDeviceSynchronize());
  });
}

int qbxg_result_exchange_local(qbxg_handle** hs, int32_t n, double* const* d_pots, double* const* d_coeffs) {
  return qbxg::guarded([&] {
    if (!hs || n < 1 || !d_pots) throw qbxg::InvalidArgument("qbxg_result_exchange_local: bad argument");
    for (int r = 0; r < n; ++r)
      if (hs[r]->h.nranks != n || hs[r]->h.rank != r || hs[r]->h.helm != hs[0]->h.helm)
        throw qbxg::InvalidArgument("qbxg_result_exchange_local: handles not rank-ordered");
    for (int r = 0; r < n; ++r) QCK(cudaStreamSynchronize(hs[r]->h.stream));
    for (int r = 0; r < n; ++r) {  // each rank's packed segment into every other rank's buffers
      auto& src = hs[r]->h;
      const int w = qbxg::coef_w(src), pw = qbxg::pot_w(src);
      for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        auto& dst = hs[q]->h;
        const int64_t a = src.res_off[r], e = src.res_off[r + 1];
        if (e > a)
          QCK(cudaMemcpy(dst.d_res_buf + a * pw, src.d_res_buf + a * pw, size_t(e - a) * pw * sizeof(double),
                         cudaMemcpyDefault));
        const int64_t ca = src.cres_off[r], ce = src.cres_off[r + 1];
        if (d_coeffs && ce > ca)
          QCK(cudaMemcpy(dst.d_cres_buf + ca * w, src.d_cres_buf + ca * w, size_t(ce - ca) * w * sizeof(double),
                         cudaMemcpyDefault));
      }
    }
    QCK(cudaDeviceSynchronize());  // (device-to-device copies above: see qbxg_exchange_local)
    for (int r = 0; r < n; ++r) {
      auto& H = hs[r]->h;
      qbxg::dev::launch_pack(int(H.nt), H.d_res_idx, qbxg::pot_w(H), d_pots[r], H.d_res_buf, true, H.stream);
      if (d_coeffs && d_coeffs[r])
        qbxg::dev::launch_pack(int(H.nc), H.d_cres_idx, qbxg::coef_w(H), d_coeffs[r], H.d_cres_buf, true, H.stream);
      QCK(cudaStreamSynchronize(H.stream));
    }
  });
}

int qbxg_nccl_unique_id(uint8_t* out128) {
  return qbxg::guarded([&] {
    if (!out128) throw qbxg::InvalidArgument("qbxg_nccl_unique_id: null argument");
    ncclUniqueId id;
    qbxg::nck(qbxg::nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
  });
}

int qbxg_nccl_attach(qbxg_handle* hp, const uint8_t* id128) {
  return qbxg::guarded([&] {
    if (!hp || !id128) throw qbxg::InvalidArgument("qbxg_nccl_attach: null argument");
    auto& H = hp->h;
    QCK(cudaSetDevice(H.device));
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    ncclComm_t comm;
    qbxg::nck(qbxg::nccl().CommInitRank(&comm, H.nranks, id, H.rank), "ncclCommInitRank");
    H.nccl_comm = comm;
  });
}

int qbxg_apply(qbxg_handle* hp, const double* weights, const double* dipoles, double* out_target_pot,
               double* out_center_coeffs, qbxg_timings* timings) {
  return qbxg::guarded([&] {
    if (!hp || !weights || !out_target_pot) throw qbxg::InvalidArgument("qbxg_apply: null argument");
    auto& H = hp->h;
    if (H.helm) throw qbxg::InvalidArgument("qbxg_apply: Helmholtz handle, use qbxg_apply_complex");
    QCK(cudaSetDevice(H.device));
    cudaStream_t s = H.stream;
    const bool dip = H.D.dipole;
    if (dip && !dipoles) throw qbxg::InvalidArgument("qbxg_apply: Laplace SL+DL requires dipole moments");
    QCK(cudaEventRecord(H.ev[11], s));
    int64_t h2d = H.ns * 8, d2h = H.nt * 8;
    QCK(cudaMemcpyAsync(H.d_w, weights, H.ns * sizeof(double), cudaMemcpyHostToDevice, s));
    if (dip) {
      QCK(cudaMemcpyAsync(H.d_mu_in, dipoles, 3 * H.ns * sizeof(double), cudaMemcpyHostToDevice, s));
      h2d += 24 * H.ns;
    }
    qbxg::full_apply(H, H.d_w, dip ? H.d_mu_in : nullptr, H.d_pot, out_center_coeffs ? H.d_coeffs : nullptr, s);
    QCK(cudaMemcpyAsync(out_target_pot, H.d_pot, H.nt * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out_center_coeffs) {
      const size_t nbytes = size_t(H.nc) * 2 * H.D.kq * sizeof(double);
      QCK(cudaMemcpyAsync(out_center_coeffs, H.d_coeffs, nbytes, cudaMemcpyDeviceToHost, s));
      d2h += int64_t(nbytes);
    }
    QCK(cudaEventRecord(H.ev[12], s));
    qbxg::fill_timings(H, timings, true, h2d, d2h);
    QCK(cudaStreamSynchronize(s));
    qbxg::check_domain(H, s);
  });
}

int qbxg_apply_batch_device(qbxg_handle* hp, int32_t n_rhs, const double* d_weights, const double* d_dipoles,
                            double* d_out_target_pot, double* d_out_center_coeffs, void* cuda_stream,
                            qbxg_timings* timings) {
  return qbxg::guarded([&] {
    if (!hp || !d_weights || !d_out_target_pot) throw qbxg::InvalidArgument("qbxg_apply_batch_device: null argument");
    if (n_rhs < 1) throw qbxg::InvalidArgument("qbxg_apply_batch_device: n_rhs must be >= 1");
    auto& H = hp->h;
    if (H.helm) throw qbxg::InvalidArgument("qbxg_apply_batch_device: Helmholtz handle, use qbxg_apply_complex");
    QCK(cudaSetDevice(H.device));
    if (H.D.dipole && !d_dipoles) throw qbxg::InvalidArgument("qbxg_apply_batch: Laplace SL+DL requires dipole moments");
    cudaStream_t s = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : H.stream;
    QCK(cudaEventRecord(H.ev[11], s));
    qbxg::batch_apply(H, n_rhs, d_weights, d_dipoles, d_out_target_pot, d_out_center_coeffs, s);
    QCK(cudaEventRecord(H.ev[12], s));
    QCK(cudaEventSynchronize(H.ev[12]));
    if (timings) {
      std::memset(timings, 0, sizeof(*timings));
      float ms = 0;
      cudaEventElapsedTime(&ms, H.ev[11], H.ev[12]);
      timings->ms[QBXG_T_TOTAL] = ms;
      timings->kernel_launches = H.last_launches;
    }
    qbxg::check_domain(H, s);
  });
}

int qbxg_apply_batch(qbxg_handle* hp, int32_t n_rhs, const double* weights, const double* dipoles,
                     double* out_target_pot, double* out_center_coeffs, qbxg_timings* timings) {
  return qbxg::guarded([&] {
    if (!hp || !weights || !out_target_pot) throw qbxg::InvalidArgument("qbxg_apply_batch: null argument");
    if (n_rhs < 1) throw qbxg::InvalidArgument("qbxg_apply_batch: n_rhs must be >= 1");
    auto& H = hp->h;
    if (H.helm) throw qbxg::InvalidArgument("qbxg_apply_batch: Helmholtz handle, use qbxg_apply_complex");
    QCK(cudaSetDevice(H.device));
    const bool dip = H.D.dipole;
    if (dip && !dipoles) throw qbxg::InvalidArgument("qbxg_apply_batch: Laplace SL+DL requires dipole moments");
    cudaStream_t s = H.stream;
    // host-path staging grows to the largest batch seen; superseded buffers are freed
    auto regrow = [&](double*& buf, size_t n) {
      if (buf) {
        QCK(cudaStreamSynchronize(s));
        cudaFree(buf);
        H.owned.erase(std::find(H.owned.begin(), H.owned.end(), static_cast<void*>(buf)));
        buf = nullptr;
      }
      if (n) buf = qbxg::dalloc<double>(H.owned, n);
    };
    if (H.bhost_cap < n_rhs) {
      regrow(H.d_bw_in, size_t(n_rhs) * H.ns);
      regrow(H.d_bmu_in, dip ? size_t(n_rhs) * 3 * H.ns : 0);
      regrow(H.d_bpot, size_t(n_rhs) * std::max<int64_t>(H.nt, 1));
      H.bhost_cap = n_rhs;
    }
    const size_t cbytes = size_t(H.nc) * 2 * H.D.kq * sizeof(double);
    if (out_center_coeffs && H.bcoeff_cap < n_rhs) {
      regrow(H.d_bcoeffs, size_t(n_rhs) * std::max<int64_t>(H.nc, 1) * 2 * H.D.kq);
      H.bcoeff_cap = n_rhs;
    }
    double* d_coeffs = out_center_coeffs ? H.d_bcoeffs : nullptr;
    QCK(cudaEventRecord(H.ev[11], s));
    QCK(cudaMemcpyAsync(H.d_bw_in, weights, size_t(n_rhs) * H.ns * sizeof(double), cudaMemcpyHostToDevice, s));
    if (dip)
      QCK(cudaMemcpyAsync(H.d_bmu_in, dipoles, size_t(n_rhs) * 3 * H.ns * sizeof(double), cudaMemcpyHostToDevice, s));
    qbxg::batch_apply(H, n_rhs, H.d_bw_in, dip ? H.d_bmu_in : nullptr, H.d_bpot, d_coeffs, s);
    QCK(cudaMemcpyAsync(out_target_pot, H.d_bpot, size_t(n_rhs) * H.nt * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (d_coeffs) QCK(cudaMemcpyAsync(out_center_coeffs, d_coeffs, size_t(n_rhs) * cbytes, cudaMemcpyDeviceToHost, s));
    QCK(cudaEventRecord(H.ev[12], s));
    QCK(cudaStreamSynchronize(s));
    if (timings) {
      std::memset(timings, 0, sizeof(*timings));
      float ms = 0;
      cudaEventElapsedTime(&ms, H.ev[11], H.ev[12]);
      timings->ms[QBXG_T_TOTAL] = ms;
      timings->kernel_launches = H.last_launches;
      timings->h2d_bytes = int64_t(n_rhs) * H.ns * (dip ? 32 : 8);
      timings->d2h_bytes = int64_t(n_rhs) * H.nt * 8 + (d_coeffs ? int64_t(n_rhs) * int64_t(cbytes) : 0);
    }
    qbxg::check_domain(H, s);
  });
}

int qbxg_apply_complex(qbxg_handle* hp, const double* weights_c, const double* dipoles_c,
                       double* out_target_pot_c, double* out_center_coeffs_c, qbxg_timings* timings) {
  return qbxg::guarded([&] {
    if (!hp || !weights_c || !out_target_pot_c) throw qbxg::InvalidArgument("qbxg_apply_complex: null argument");
    auto& H = hp->h;
    if (!H.helm) throw qbxg::InvalidArgument("qbxg_apply_complex: handle was not created for the Helmholtz kernel");
    QCK(cudaSetDevice(H.device));
    cudaStream_t s = H.stream;
    for (int64_t i = 0; i < 2 * H.ns; ++i)
      if (!std::isfinite(weights_c[i])) throw qbxg::InvalidArgument("qbxg_apply_complex: non-finite weight");
    if (dipoles_c && !H.HD.hmu)
      throw qbxg::InvalidArgument("qbxg_apply_complex: dipoles given to a single-layer handle");
    if (!dipoles_c && H.HD.hmu) throw qbxg::InvalidArgument("qbxg_apply_complex: Helmholtz SL+DL requires dipole moments");
    if (dipoles_c)
      for (int64_t i = 0; i < 6 * H.ns; ++i)
        if (!std::isfinite(dipoles_c[i])) throw qbxg::InvalidArgument("qbxg_apply_complex: non-finite dipole");
    QCK(cudaEventRecord(H.ev[11], s));
    QCK(cudaMemcpyAsync(H.d_wc, weights_c, 2 * H.ns * sizeof(double), cudaMemcpyHostToDevice, s));
    if (dipoles_c) QCK(cudaMemcpyAsync(H.d_muc, dipoles_c, 6 * H.ns * sizeof(double), cudaMemcpyHostToDevice, s));
    // (sharded handles: owned upward pass, NCCL multipole exchange, downward pass, result all-gather)
    qbxg::full_apply(H, H.d_wc, dipoles_c ? H.d_muc : nullptr, H.d_potc, out_center_coeffs_c ? H.d_coeffc : nullptr, s);
    QCK(cudaMemcpyAsync(out_target_pot_c, H.d_potc, 2 * H.nt * sizeof(double), cudaMemcpyDeviceToHost, s));
    const size_t cbytes = size_t(H.nc) * 2 * H.HD.KQ * sizeof(double);
    if (out_center_coeffs_c) QCK(cudaMemcpyAsync(out_center_coeffs_c, H.d_coeffc, cbytes, cudaMemcpyDeviceToHost, s));
    QCK(cudaEventRecord(H.ev[12], s));
    qbxg::fill_timings(H, timings, true, (dipoles_c ? 64 : 16) * H.ns,
                       16 * H.nt + (out_center_coeffs_c ? int64_t(cbytes) : 0));
    QCK(cudaStreamSynchronize(s));
    qbxg::check_domain(H, s);
  });
}

int qbxg_set_overlap(qbxg_handle* hp, int32_t enable) {
  return qbxg::guarded([&] {
    if (!hp) throw qbxg::InvalidArgument("qbxg_set_overlap: null handle");
    hp->h.overlap = enable != 0;
  });
}

int qbxg_destroy(qbxg_handle* h) {
  delete h;
  return QBXG_OK;
}

int qbxg_direct_sum(int64_t n_sources, const double* source_pos, const double* weights, const double* dipoles_or_null,
                    int64_t n_targets, const double* target_pos, double* out_pot) {
  return qbxg::guarded([&] {
    if (n_sources < 0 || n_targets < 0) throw qbxg::InvalidArgument("direct_sum: negative size");
    if ((n_sources && (!source_pos || !weights)) || (n_targets && (!target_pos || !out_pot)))
      throw qbxg::InvalidArgument("direct_sum: null array");
    if (n_sources >= (int64_t(1) << 31) || n_targets >= (int64_t(1) << 31))
      throw qbxg::InvalidArgument("direct_sum: too many points");
    qbxg::validate_sources(n_sources, source_pos, weights, dipoles_or_null);
    if (n_targets == 0) return;
    qbxg::check_device();
    std::vector<void*> owned;
    struct Free {
      std::vector<void*>& o;
      ~Free() {
        for (void* p : o) cudaFree(p);
      }
    } fr{owned};
    std::vector<double4> src(n_sources), mu(dipoles_or_null ? n_sources : 0), tgt(n_targets);
    for (int64_t i = 0; i < n_sources; ++i) {
      src[i] = make_double4(source_pos[3 * i], source_pos[3 * i + 1], source_pos[3 * i + 2], weights[i]);
      if (dipoles_or_null)
        mu[i] = make_double4(dipoles_or_null[3 * i], dipoles_or_null[3 * i + 1], dipoles_or_null[3 * i + 2], 0);
    }
    for (int64_t i = 0; i < n_targets; ++i)
      tgt[i] = make_double4(target_pos[3 * i], target_pos[3 * i + 1], target_pos[3 * i + 2], 0);
    cudaStream_t s = nullptr;
    double4* ds = qbxg::dupload(owned, src, s);
    double4* dm = dipoles_or_null ? qbxg::dupload(owned, mu, s) : nullptr;
    double4* dt = qbxg::dupload(owned, tgt, s);
    double* dp = qbxg::dalloc<double>(owned, n_targets);
    unsigned long long* bad = qbxg::dalloc<unsigned long long>(owned, 1);
    QCK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    qbxg::dev::launch_direct_sum(int(n_sources), ds, dm, int(n_targets), dt, dp, bad, s);
    QCK(cudaGetLastError());
    unsigned long long hb = 0;
    QCK(cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost));
    QCK(cudaMemcpy(out_pot, dp, n_targets * sizeof(double), cudaMemcpyDeviceToHost));
    if (hb != ~0ull)
      throw qbxg::DomainError("direct_sum: target " + std::to_string(hb >> 32) + " coincides with source " +
                              std::to_string(hb & 0xffffffffull));
  });
}

int qbxg_helm_direct_sum(double k, int64_t n_sources, const double* source_pos, const double* weights_c,
                         const double* dipoles_c, int64_t n_targets, const double* target_pos, double* out_pot_c) {
  return qbxg::guarded([&] {
    using qbxg::InvalidArgument;
    if (n_sources < 0 || n_targets < 0) throw InvalidArgument("helm_direct_sum: negative size");
    if (n_sources >= (int64_t(1) << 31) || n_targets >= (int64_t(1) << 31))
      throw InvalidArgument("helm_direct_sum: too many points");
    if ((n_sources && (!source_pos || !weights_c)) || (n_targets && (!target_pos || !out_pot_c)))
      throw InvalidArgument("helm_direct_sum: null array");
    if (!(k > 0) || !std::isfinite(k)) throw InvalidArgument("helm_direct_sum: wavenumber must be positive");
    for (int64_t i = 0; i < 2 * n_sources; ++i)
      if (!std::isfinite(weights_c[i])) throw InvalidArgument("helm_direct_sum: non-finite weight");
    if (dipoles_c)
      for (int64_t i = 0; i < 6 * n_sources; ++i)
        if (!std::isfinite(dipoles_c[i])) throw InvalidArgument("helm_direct_sum: non-finite dipole");
    if (n_targets == 0) return;
    qbxg::check_device();
    std::vector<void*> owned;
    struct Free {
      std::vector<void*>& o;
      ~Free() {
        for (void* p : o) cudaFree(p);
      }
    } fr{owned};
    std::vector<double4> src(n_sources), tgt(n_targets);
    std::vector<double2> w(n_sources);
    for (int64_t i = 0; i < n_sources; ++i) {
      src[i] = make_double4(source_pos[3 * i], source_pos[3 * i + 1], source_pos[3 * i + 2], 0);
      w[i] = make_double2(weights_c[2 * i], weights_c[2 * i + 1]);
    }
    for (int64_t i = 0; i < n_targets; ++i)
      tgt[i] = make_double4(target_pos[3 * i], target_pos[3 * i + 1], target_pos[3 * i + 2], 0);
    cudaStream_t s = nullptr;
    double4* ds = qbxg::dupload(owned, src, s);
    double2* dw = qbxg::dupload(owned, w, s);
    double2* dm = dipoles_c ? qbxg::dupload(owned, std::vector<double2>(reinterpret_cast<const double2*>(dipoles_c),
                                                                         reinterpret_cast<const double2*>(dipoles_c) +
                                                                             3 * n_sources),
                                            s)
                            : nullptr;
    double4* dt = qbxg::dupload(owned, tgt, s);
    double2* dp = qbxg::dalloc<double2>(owned, n_targets);
    unsigned long long* bad = qbxg::dalloc<unsigned long long>(owned, 1);
    QCK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    qbxg::dev::launch_helm_direct_sum(k, int(n_sources), ds, dw, dm, int(n_targets), dt, dp, bad, s);
    QCK(cudaGetLastError());
    unsigned long long hb = 0;
    QCK(cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost));
    if (hb != ~0ull)
      throw qbxg::DomainError("helm_direct_sum: target " + std::to_string(hb >> 32) + " coincides with source " +
                              std::to_string(hb & 0xffffffffull));
    QCK(cudaMemcpy(out_pot_c, dp, n_targets * sizeof(double2), cudaMemcpyDeviceToHost));
  });
}

int qbxg_helm_direct_qbx(double k, int64_t n_sources, const double* source_pos, const double* weights_c,
                         const double* dipoles_c, int64_t n_centers, const double* center_pos, int64_t n_targets, const double* target_pos,
                         const int32_t* association, int32_t p_qbx, double* out_pot_c) {
  return qbxg::guarded([&] {
    using qbxg::InvalidArgument;
    if (n_sources < 0 || n_centers < 0 || n_targets < 0) throw InvalidArgument("helm_direct_qbx: negative size");
    if (n_sources >= (int64_t(1) << 31) || n_centers >= (int64_t(1) << 31) || n_targets >= (int64_t(1) << 31))
      throw InvalidArgument("helm_direct_qbx: too many points");
    if (p_qbx < 0 || p_qbx > 8) throw InvalidArgument("helm_direct_qbx: p_qbx must be in [0, 8]");
    if (!(k > 0) || !std::isfinite(k)) throw InvalidArgument("helm_direct_qbx: wavenumber must be positive");
    if ((n_sources && (!source_pos || !weights_c)) || (n_centers && !center_pos) ||
        (n_targets && (!target_pos || !association || !out_pot_c)))
      throw InvalidArgument("helm_direct_qbx: null array");
    std::vector<int> conv;
    for (int64_t i = 0; i < n_targets; ++i) {
      const int32_t a = association[i];
      if (a < -1 || a >= n_centers)
        throw InvalidArgument("helm_direct_qbx: target " + std::to_string(i) + " has association " +
                              std::to_string(a) + " outside [-1, n_centers)");
      if (a < 0) conv.push_back(int(i));
    }
    if (n_targets == 0) return;
    qbxg::check_device();
    std::vector<void*> owned;
    struct Free {
      std::vector<void*>& o;
      ~Free() {
        for (void* p : o) cudaFree(p);
      }
    } fr{owned};
    std::vector<double4> src(n_sources), ctr(n_centers), ctg(conv.size());
    std::vector<double2> w(n_sources);
    for (int64_t i = 0; i < n_sources; ++i) {
      src[i] = make_double4(source_pos[3 * i], source_pos[3 * i + 1], source_pos[3 * i + 2], 0);
      w[i] = make_double2(weights_c[2 * i], weights_c[2 * i + 1]);
    }
    for (int64_t c = 0; c < n_centers; ++c)
      ctr[c] = make_double4(center_pos[3 * c], center_pos[3 * c + 1], center_pos[3 * c + 2], 0);
    for (size_t j = 0; j < conv.size(); ++j)
      ctg[j] = make_double4(target_pos[3 * conv[j]], target_pos[3 * conv[j] + 1], target_pos[3 * conv[j] + 2], 0);
    cudaStream_t s = nullptr;
    double4* ds = qbxg::dupload(owned, src, s);
    double2* dw = qbxg::dupload(owned, w, s);
    if (dipoles_c)
      for (int64_t i = 0; i < 6 * n_sources; ++i)
        if (!std::isfinite(dipoles_c[i])) throw InvalidArgument("helm_direct_qbx: non-finite dipole");
    double2* dm = dipoles_c ? qbxg::dupload(owned, std::vector<double2>(reinterpret_cast<const double2*>(dipoles_c),
                                                                         reinterpret_cast<const double2*>(dipoles_c) +
                                                                             3 * n_sources),
                                            s)
                            : nullptr;
    double4* dc = qbxg::dupload(owned, ctr, s);
    double* dtp = qbxg::dupload(owned, std::vector<double>(target_pos, target_pos + 3 * n_targets), s);
    int* das = qbxg::dupload(owned, std::vector<int>(association, association + n_targets), s);
    double2* dl = qbxg::dalloc<double2>(owned, size_t(std::max<int64_t>(n_centers, 1)) * (p_qbx + 1) * (p_qbx + 1));
    double2* dp = qbxg::dalloc<double2>(owned, n_targets);
    QCK(cudaMemsetAsync(dp, 0, n_targets * sizeof(double2), s));
    qbxg::dev::launch_helm_direct_qbx(k, p_qbx, int(n_sources), ds, dw, dm, int(n_centers), dc, dl, int(n_targets),
                                      dtp, das, dp, s);
    QCK(cudaGetLastError());
    std::vector<double2> pot(n_targets);
    QCK(cudaMemcpy(pot.data(), dp, n_targets * sizeof(double2), cudaMemcpyDeviceToHost));
    if (!conv.empty()) {
      double4* dt = qbxg::dupload(owned, ctg, s);
      double2* dq = qbxg::dalloc<double2>(owned, conv.size());
      unsigned long long* bad = qbxg::dalloc<unsigned long long>(owned, 1);
      QCK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
      qbxg::dev::launch_helm_direct_sum(k, int(n_sources), ds, dw, dm, int(conv.size()), dt, dq, bad, s);
      QCK(cudaGetLastError());
      unsigned long long hb = 0;
      QCK(cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost));
      if (hb != ~0ull)
        throw qbxg::DomainError("helm_direct_qbx: target " + std::to_string(conv[hb >> 32]) +
                                " coincides with source " + std::to_string(hb & 0xffffffffull));
      std::vector<double2> pc(conv.size());
      QCK(cudaMemcpy(pc.data(), dq, conv.size() * sizeof(double2), cudaMemcpyDeviceToHost));
      for (size_t j = 0; j < conv.size(); ++j) pot[conv[j]] = pc[j];
    }
    std::memcpy(out_pot_c, pot.data(), n_targets * sizeof(double2));
  });
}

int qbxg_direct_qbx(int64_t n_sources, const double* source_pos, const double* weights, const double* dipoles_or_null,
                    int64_t n_centers, const double* center_pos, const double* center_radius, int64_t n_targets,
                    const double* target_pos, const int32_t* association, int32_t p_qbx, double* out_pot) {
  return qbxg::guarded([&] {
    using qbxg::InvalidArgument;
    if (n_sources < 0 || n_centers < 0 || n_targets < 0) throw InvalidArgument("direct_qbx: negative size");
    if (n_sources >= (int64_t(1) << 31) || n_centers >= (int64_t(1) << 31) || n_targets >= (int64_t(1) << 31))
      throw InvalidArgument("direct_qbx: too many points");
    if (p_qbx < 0 || p_qbx > 8) throw InvalidArgument("direct_qbx: p_qbx must be in [0, 8]");
    if ((n_sources && (!source_pos || !weights)) || (n_centers && (!center_pos || !center_radius)) ||
        (n_targets && (!target_pos || !association || !out_pot)))
      throw InvalidArgument("direct_qbx: null array");
    qbxg::validate_sources(n_sources, source_pos, weights, dipoles_or_null);
    for (int64_t c = 0; c < n_centers; ++c)
      if (!(center_radius[c] > 0) || !std::isfinite(center_radius[c]) || !std::isfinite(center_pos[3 * c]) ||
          !std::isfinite(center_pos[3 * c + 1]) || !std::isfinite(center_pos[3 * c + 2]))
        throw InvalidArgument("direct_qbx: centre " + std::to_string(c) + " has a bad position or radius");
    std::vector<int> conv;
    for (int64_t i = 0; i < n_targets; ++i) {
      const int32_t a = association[i];
      if (a < -1 || a >= n_centers)
        throw InvalidArgument("direct_qbx: target " + std::to_string(i) + " has association " + std::to_string(a) +
                              " outside [-1, n_centers)");
      if (a < 0) conv.push_back(int(i));
    }
    if (n_targets == 0) return;
    qbxg::check_device();
    std::vector<void*> owned;
    struct Free {
      std::vector<void*>& o;
      ~Free() {
        for (void* p : o) cudaFree(p);
      }
    } fr{owned};
    std::vector<double4> src(n_sources), mu(dipoles_or_null ? n_sources : 0), ctr(n_centers), ctg(conv.size());
    for (int64_t i = 0; i < n_sources; ++i) {
      src[i] = make_double4(source_pos[3 * i], source_pos[3 * i + 1], source_pos[3 * i + 2], weights[i]);
      if (dipoles_or_null)
        mu[i] = make_double4(dipoles_or_null[3 * i], dipoles_or_null[3 * i + 1], dipoles_or_null[3 * i + 2], 0);
    }
    for (int64_t c = 0; c < n_centers; ++c)
      ctr[c] = make_double4(center_pos[3 * c], center_pos[3 * c + 1], center_pos[3 * c + 2], center_radius[c]);
    for (size_t j = 0; j < conv.size(); ++j) {
      const int64_t i = conv[j];
      ctg[j] = make_double4(target_pos[3 * i], target_pos[3 * i + 1], target_pos[3 * i + 2], 0);
    }
    cudaStream_t s = nullptr;
    qbxg::dev::upload_constants();
    double4* ds = qbxg::dupload(owned, src, s);
    double4* dm = dipoles_or_null ? qbxg::dupload(owned, mu, s) : nullptr;
    double4* dc = qbxg::dupload(owned, ctr, s);
    std::vector<double> tp(target_pos, target_pos + 3 * n_targets);
    std::vector<int> as(association, association + n_targets);
    double* dtp = qbxg::dupload(owned, tp, s);
    int* das = qbxg::dupload(owned, as, s);
    double2* dl = qbxg::dalloc<double2>(owned, size_t(std::max<int64_t>(n_centers, 1)) * ((p_qbx + 1) * (p_qbx + 2) / 2));
    double* dp = qbxg::dalloc<double>(owned, n_targets);
    QCK(cudaMemsetAsync(dp, 0, n_targets * sizeof(double), s));
    qbxg::dev::launch_direct_qbx(p_qbx, int(n_sources), ds, dm, int(n_centers), dc, dl, s);
    QCK(cudaGetLastError());
    qbxg::dev::launch_direct_qbx_eval(p_qbx, int(n_targets), dtp, das, dc, dl, dp, s);
    QCK(cudaGetLastError());
    std::vector<double> pot(n_targets);
    QCK(cudaMemcpy(pot.data(), dp, n_targets * sizeof(double), cudaMemcpyDeviceToHost));
    if (!conv.empty()) {
      double4* dt = qbxg::dupload(owned, ctg, s);
      double* dq = qbxg::dalloc<double>(owned, conv.size());
      unsigned long long* bad = qbxg::dalloc<unsigned long long>(owned, 1);
      QCK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
      qbxg::dev::launch_direct_sum(int(n_sources), ds, dm, int(conv.size()), dt, dq, bad, s);
      QCK(cudaGetLastError());
      unsigned long long hb = 0;
      QCK(cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost));
      if (hb != ~0ull)
        throw qbxg::DomainError("direct_qbx: target " + std::to_string(conv[hb >> 32]) +
                                " coincides with source " + std::to_string(hb & 0xffffffffull));
      std::vector<double> pc(conv.size());
      QCK(cudaMemcpy(pc.data(), dq, conv.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (size_t j = 0; j < conv.size(); ++j) pot[conv[j]] = pc[j];
    }
    std::copy(pot.begin(), pot.end(), out_pot);
  });
}

}  // extern "C"
