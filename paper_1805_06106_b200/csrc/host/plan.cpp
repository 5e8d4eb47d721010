// Stage 1 of Algorithm 4 and the GIGAQBX interaction
// lists (Definitions 1-8), in host C++ as BASELINE.json's
// north_star requires.  Replaces the reference's declared src/tree.cpp and
// src/interaction_lists.cpp (proj/CMakeLists.txt:24-25).
//
// Tree: the target-confinement octree of PAPER.md:2050-2062 / SPEC.md:333-351.
//   - boxes with more than n_max owned particles (sources + centres +
//     conventional targets) subdivide while at least one particle moves down
//     (SPEC.md:395); empty children are pruned;
//   - a QBX centre moves into the spatially appropriate child only when its
//     ball fits that child's TCR B2(sqrt(3)|child|(1+t_f), centre),
//     otherwise it stays suspended in the parent;
//   - boxes are numbered in DFS preorder with children in octant (Morton)
//     order, so every subtree is a contiguous box range and every box's
//     particles (own first, then children's) are contiguous in each role's
//     box-sorted array.  Contiguous Morton ranges are the multi-GPU shards.
//
// Lists (rows sorted by box id): U, V, W_close, W_far, X_close,
// X_far, restricted to boxes whose subtree holds sources (the field of a box
// without sources is zero).  U, W_* are built for target boxes; V and X_* for
// target and target-ancestor boxes.
#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <numeric>
#include <unordered_map>

#include "plan.hpp"

namespace qbxg {

namespace {

struct BuildBox {
  double c[3];
  double h;
  int32_t level, parent;
  int64_t ic[3];
  int64_t start, end, own;
  int32_t child[8];
};

}  // namespace

void validate_inputs(const qbxg_config& cfg, const qbxg_geometry& g) {
  if (cfg.p_fmm < 0 || cfg.p_qbx < 0) throw InvalidArgument("FmmConfig: negative order");
  if (cfg.p_qbx > cfg.p_fmm) throw InvalidArgument("FmmConfig: p_qbx must not exceed p_fmm (SPEC.md:416)");
  if (cfg.p_fmm > 40) throw InvalidArgument("FmmConfig: p_fmm > 40 unsupported");
  if (!(cfg.t_f >= 0) || !(cfg.t_f < 2 * std::sqrt(3.0) - 2))
    throw InvalidArgument("FmmConfig: t_f must satisfy 0 <= t_f < 2 sqrt(3) - 2 (SPEC.md:416)");
  if (cfg.n_max < 1) throw InvalidArgument("FmmConfig: n_max must be positive");
  if (cfg.kernel != QBXG_KERNEL_LAPLACE_SL && cfg.kernel != QBXG_KERNEL_LAPLACE_SL_DL &&
      cfg.kernel != QBXG_KERNEL_HELMHOLTZ_SL && cfg.kernel != QBXG_KERNEL_HELMHOLTZ_SL_DL)
    throw InvalidArgument("FmmConfig: unknown kernel");
  if ((cfg.kernel == QBXG_KERNEL_HELMHOLTZ_SL || cfg.kernel == QBXG_KERNEL_HELMHOLTZ_SL_DL) && !(cfg.helmholtz_k > 0 && std::isfinite(cfg.helmholtz_k)))
    throw InvalidArgument("FmmConfig: Helmholtz needs a positive wavenumber helmholtz_k");
  if (cfg.level_restrict != 0 && cfg.level_restrict != 1)
    throw InvalidArgument("FmmConfig: level_restrict must be 0 or 1");
  if (g.n_sources < 0 || g.n_centers < 0 || g.n_targets < 0) throw InvalidArgument("geometry: negative size");
  if (g.n_sources + g.n_centers + g.n_targets >= std::numeric_limits<int32_t>::max())
    throw InvalidArgument("geometry: too many particles for int32 indexing");
  if ((g.n_sources && !g.source_pos) || (g.n_centers && (!g.center_pos || !g.center_radius)) ||
      (g.n_targets && (!g.target_pos || !g.association)))
    throw InvalidArgument("geometry: null array");
  for (int64_t i = 0; i < 3 * g.n_sources; ++i)
    if (!std::isfinite(g.source_pos[i])) throw InvalidArgument("geometry: non-finite source position at index " + std::to_string(i / 3));
  for (int64_t i = 0; i < g.n_centers; ++i) {
    if (!std::isfinite(g.center_pos[3 * i]) || !std::isfinite(g.center_pos[3 * i + 1]) ||
        !std::isfinite(g.center_pos[3 * i + 2]))
      throw InvalidArgument("geometry: non-finite centre position at index " + std::to_string(i));
    if (!(g.center_radius[i] > 0) || !std::isfinite(g.center_radius[i]))
      throw InvalidArgument("geometry: centre radius must be positive and finite (index " + std::to_string(i) + ")");
  }
  for (int64_t i = 0; i < g.n_targets; ++i) {
    if (!std::isfinite(g.target_pos[3 * i]) || !std::isfinite(g.target_pos[3 * i + 1]) ||
        !std::isfinite(g.target_pos[3 * i + 2]))
      throw InvalidArgument("geometry: non-finite target position at index " + std::to_string(i));
    if (g.association[i] < -1 || g.association[i] >= g.n_centers)
      throw InvalidArgument("target " + std::to_string(i) + " is neither associated to a valid centre nor conventional");
  }
}

void build_tree(Plan& P, const qbxg_geometry& g) {
  const double t0 = now_seconds();
  const qbxg_config& cfg = P.cfg;
  P.ns = g.n_sources;
  P.nc = g.n_centers;
  P.ntgt = g.n_targets;
  std::vector<int32_t> conv;
  for (int64_t t = 0; t < g.n_targets; ++t)
    if (g.association[t] < 0) conv.push_back(int32_t(t));
  P.nconv = int64_t(conv.size());
  const int64_t np = P.ns + P.nc + P.nconv;

  // particle table: [sources][centres][conventional targets]
  std::vector<double> pos(3 * np), rad(np, 0.0);
  std::vector<uint8_t> role(np);
  for (int64_t i = 0; i < P.ns; ++i) {
    for (int d = 0; d < 3; ++d) pos[3 * i + d] = g.source_pos[3 * i + d];
    role[i] = 0;
  }
  for (int64_t i = 0; i < P.nc; ++i) {
    const int64_t k = P.ns + i;
    for (int d = 0; d < 3; ++d) pos[3 * k + d] = g.center_pos[3 * i + d];
    rad[k] = g.center_radius[i];
    role[k] = 1;
  }
  for (int64_t i = 0; i < P.nconv; ++i) {
    const int64_t k = P.ns + P.nc + i;
    for (int d = 0; d < 3; ++d) pos[3 * k + d] = g.target_pos[3 * int64_t(conv[i]) + d];
    role[k] = 2;
  }

  // root: axis-aligned cube containing every particle and every expansion ball
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t k = 0; k < np; ++k)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], pos[3 * k + d] - rad[k]);
      hi[d] = std::max(hi[d], pos[3 * k + d] + rad[k]);
    }
  if (np == 0) {
    for (int d = 0; d < 3; ++d) lo[d] = -1, hi[d] = 1;
  }
  double hroot = 0;
  for (int d = 0; d < 3; ++d) {
    P.root_c[d] = 0.5 * (lo[d] + hi[d]);
    hroot = std::max(hroot, 0.5 * (hi[d] - lo[d]));
  }
  if (!(hroot > 0)) hroot = 1.0;
  hroot *= 1.0 + 1.0 / 1024.0;
  P.root_h = hroot;

  std::vector<BuildBox> bx;
  BuildBox root{};
  for (int d = 0; d < 3; ++d) root.c[d] = P.root_c[d], root.ic[d] = 0;
  root.h = hroot;
  root.level = 0;
  root.parent = -1;
  root.start = 0;
  root.end = np;
  root.own = np;
  std::fill(root.child, root.child + 8, -1);
  bx.push_back(root);

  std::vector<int32_t> perm(np);
  std::iota(perm.begin(), perm.end(), 0);
  std::vector<int32_t> cur{0};
  bool depth_exceeded = false;
  while (!cur.empty()) {
    const int64_t nq = int64_t(cur.size());
    std::vector<std::array<int64_t, 9>> counts(nq);
    std::vector<uint8_t> split(nq, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < nq; ++qi) {
      const BuildBox b = bx[cur[qi]];
      const int64_t n = b.end - b.start;
      if (n <= cfg.n_max) continue;
      const double hc = 0.5 * b.h;
      std::vector<uint8_t> dest(n);
      int64_t moving = 0;
      std::array<int64_t, 9> cnt{};
      for (int64_t i = 0; i < n; ++i) {
        const int32_t k = perm[b.start + i];
        const double* x = &pos[3 * int64_t(k)];
        int o = (x[0] >= b.c[0] ? 1 : 0) | (x[1] >= b.c[1] ? 2 : 0) | (x[2] >= b.c[2] ? 4 : 0);
        if (role[k] == 1) {
          double cc[3] = {b.c[0] + ((o & 1) ? hc : -hc), b.c[1] + ((o & 2) ? hc : -hc),
                          b.c[2] + ((o & 4) ? hc : -hc)};
          if (!ball_fits_tcr(x, rad[k], cc, hc, cfg.t_f)) o = 8;
        }
        dest[i] = uint8_t(o);
        cnt[o]++;
        if (o != 8) moving++;
      }
      if (moving == 0) continue;
      if (b.level + 1 > kMaxDepth) {
#pragma omp critical
        depth_exceeded = true;
        continue;
      }
      // stable bucket order: suspended (stay) first, then octants 0..7
      std::array<int64_t, 9> off{};
      int64_t acc = cnt[8];
      off[8] = 0;
      for (int o = 0; o < 8; ++o) {
        off[o] = acc;
        acc += cnt[o];
      }
      std::vector<int32_t> tmp(n);
      for (int64_t i = 0; i < n; ++i) tmp[off[dest[i]]++] = perm[b.start + i];
      std::copy(tmp.begin(), tmp.end(), perm.begin() + b.start);
      counts[qi] = cnt;
      split[qi] = 1;
    }
    if (depth_exceeded) throw InvalidArgument("build_tree: depth cap exceeded (SPEC.md:347)");
    std::vector<int32_t> next;
    for (int64_t qi = 0; qi < nq; ++qi) {
      if (!split[qi]) continue;
      const int32_t bid = cur[qi];
      BuildBox b = bx[bid];
      const auto& cnt = counts[qi];
      b.own = cnt[8];
      int64_t s = b.start + cnt[8];
      for (int o = 0; o < 8; ++o) {
        if (cnt[o] == 0) continue;
        BuildBox c{};
        const double hc = 0.5 * b.h;
        c.c[0] = b.c[0] + ((o & 1) ? hc : -hc);
        c.c[1] = b.c[1] + ((o & 2) ? hc : -hc);
        c.c[2] = b.c[2] + ((o & 4) ? hc : -hc);
        c.h = hc;
        c.level = b.level + 1;
        c.parent = bid;
        for (int d = 0; d < 3; ++d) c.ic[d] = 2 * b.ic[d] + ((o >> d) & 1);
        c.start = s;
        c.end = s + cnt[o];
        c.own = cnt[o];
        std::fill(c.child, c.child + 8, -1);
        s += cnt[o];
        b.child[o] = int32_t(bx.size());
        next.push_back(int32_t(bx.size()));
        bx.push_back(c);
      }
      bx[bid] = b;
    }
    cur.swap(next);
  }

  // Level restriction (Remark C.1 PAPER.md:3661-3687; off unless
  // cfg.level_restrict): subdivide larger leaves until adjacent leaves (closed boxes
  // that touch) differ by at most one level.  A leaf A of level a violates when some
  // leaf of level >= a + 2 touches it; such a leaf lies inside a level-(a+1) box that
  // touches A, so the level-(a+1) boxes around A are looked up by integer coordinates
  // and searched downwards through the children that still touch A.  Leaves split
  // like any box (centres move only when their ball fits the child's TCR; a leaf
  // whose particles cannot move stays); repeat until no leaf changes.
  if (cfg.level_restrict) {
    auto key = [](int level, int64_t x, int64_t y, int64_t z) {
      return (uint64_t(level) << 58) ^ (uint64_t(x) << 38) ^ (uint64_t(y) << 19) ^ uint64_t(z);
    };
    auto touches = [&](const BuildBox& a, const BuildBox& b) {
      const int L = std::max(a.level, b.level);
      for (int d = 0; d < 3; ++d) {
        const int64_t sa = int64_t(1) << (L - a.level), sb = int64_t(1) << (L - b.level);
        const int64_t a0 = a.ic[d] * sa, a1 = a0 + sa, b0 = b.ic[d] * sb, b1 = b0 + sb;
        if (a1 < b0 || b1 < a0) return false;
      }
      return true;
    };
    for (int round = 0;; ++round) {
      std::unordered_map<uint64_t, int32_t> at;
      at.reserve(bx.size() * 2);
      for (int32_t i = 0; i < int32_t(bx.size()); ++i) at[key(bx[i].level, bx[i].ic[0], bx[i].ic[1], bx[i].ic[2])] = i;
      auto is_leaf = [&](int32_t i) {
        for (int o = 0; o < 8; ++o)
          if (bx[i].child[o] >= 0) return false;
        return true;
      };
      std::vector<int32_t> viol;
      for (int32_t i = 0; i < int32_t(bx.size()); ++i) {
        if (!is_leaf(i)) continue;
        const BuildBox& A = bx[i];
        bool bad = false;
        for (int64_t dx = -1; dx <= 2 && !bad; ++dx)
          for (int64_t dy = -1; dy <= 2 && !bad; ++dy)
            for (int64_t dz = -1; dz <= 2 && !bad; ++dz) {
              const int64_t x = 2 * A.ic[0] + dx, y = 2 * A.ic[1] + dy, z = 2 * A.ic[2] + dz;
              if (x < 0 || y < 0 || z < 0) continue;
              auto it = at.find(key(A.level + 1, x, y, z));
              if (it == at.end()) continue;
              // a leaf of level >= a + 2 touching A below this level-(a+1) box?
              std::vector<int32_t> st;
              for (int o = 0; o < 8; ++o)
                if (bx[it->second].child[o] >= 0) st.push_back(bx[it->second].child[o]);
              while (!st.empty() && !bad) {
                const int32_t c = st.back();
                st.pop_back();
                if (!touches(A, bx[c])) continue;
                if (is_leaf(c)) {
                  bad = true;
                  break;
                }
                for (int o = 0; o < 8; ++o)
                  if (bx[c].child[o] >= 0) st.push_back(bx[c].child[o]);
              }
            }
        if (bad) viol.push_back(i);
      }
      int split_any = 0;
      for (int32_t bid : viol) {
        BuildBox b = bx[bid];
        const int64_t n = b.end - b.start;
        if (n == 0 || b.level + 1 > kMaxDepth) continue;
        const double hc = 0.5 * b.h;
        std::vector<uint8_t> dest(n);
        std::array<int64_t, 9> cnt{};
        int64_t moving = 0;
        for (int64_t i = 0; i < n; ++i) {
          const int32_t k = perm[b.start + i];
          const double* x = &pos[3 * int64_t(k)];
          int o = (x[0] >= b.c[0] ? 1 : 0) | (x[1] >= b.c[1] ? 2 : 0) | (x[2] >= b.c[2] ? 4 : 0);
          if (role[k] == 1) {
            double cc[3] = {b.c[0] + ((o & 1) ? hc : -hc), b.c[1] + ((o & 2) ? hc : -hc),
                            b.c[2] + ((o & 4) ? hc : -hc)};
            if (!ball_fits_tcr(x, rad[k], cc, hc, cfg.t_f)) o = 8;
          }
          dest[i] = uint8_t(o);
          cnt[o]++;
          if (o != 8) moving++;
        }
        if (moving == 0) continue;
        std::array<int64_t, 9> off{};
        int64_t acc = cnt[8];
        for (int o = 0; o < 8; ++o) {
          off[o] = acc;
          acc += cnt[o];
        }
        std::vector<int32_t> tmp(n);
        for (int64_t i = 0; i < n; ++i) tmp[off[dest[i]]++] = perm[b.start + i];
        std::copy(tmp.begin(), tmp.end(), perm.begin() + b.start);
        b.own = cnt[8];
        int64_t s = b.start + cnt[8];
        for (int o = 0; o < 8; ++o) {
          if (cnt[o] == 0) continue;
          BuildBox c{};
          c.c[0] = b.c[0] + ((o & 1) ? hc : -hc);
          c.c[1] = b.c[1] + ((o & 2) ? hc : -hc);
          c.c[2] = b.c[2] + ((o & 4) ? hc : -hc);
          c.h = hc;
          c.level = b.level + 1;
          c.parent = bid;
          for (int d = 0; d < 3; ++d) c.ic[d] = 2 * b.ic[d] + ((o >> d) & 1);
          c.start = s;
          c.end = s + cnt[o];
          c.own = cnt[o];
          std::fill(c.child, c.child + 8, -1);
          s += cnt[o];
          b.child[o] = int32_t(bx.size());
          bx.push_back(c);
        }
        bx[bid] = b;
        ++split_any;
      }
      if (!split_any) break;
    }
  }

  // DFS preorder renumbering (children in octant order)
  const int32_t nb = int32_t(bx.size());
  std::vector<int32_t> newid(nb, -1), order;
  order.reserve(nb);
  {
    std::vector<int32_t> stack{0};
    while (!stack.empty()) {
      int32_t b = stack.back();
      stack.pop_back();
      newid[b] = int32_t(order.size());
      order.push_back(b);
      for (int o = 7; o >= 0; --o)
        if (bx[b].child[o] >= 0) stack.push_back(bx[b].child[o]);
    }
  }
  P.nb = nb;
  P.center.resize(3 * nb);
  P.h.resize(nb);
  P.level.resize(nb);
  P.parent.resize(nb);
  P.ic.resize(3 * nb);
  P.child_starts.assign(nb + 1, 0);
  P.children.clear();
  std::vector<int64_t> bstart(nb), bend(nb), bown(nb);
  int32_t maxlev = 0;
  for (int32_t nbid = 0; nbid < nb; ++nbid) {
    const BuildBox& b = bx[order[nbid]];
    for (int d = 0; d < 3; ++d) {
      P.center[3 * nbid + d] = b.c[d];
      P.ic[3 * nbid + d] = b.ic[d];
    }
    P.h[nbid] = b.h;
    P.level[nbid] = b.level;
    P.parent[nbid] = b.parent >= 0 ? newid[b.parent] : -1;
    maxlev = std::max(maxlev, b.level);
    for (int o = 0; o < 8; ++o)
      if (b.child[o] >= 0) P.children.push_back(newid[b.child[o]]);
    P.child_starts[nbid + 1] = int32_t(P.children.size());
    bstart[nbid] = b.start;
    bend[nbid] = b.end;
    bown[nbid] = b.own;
  }
  P.nlev = maxlev + 1;
  P.subtree_end.resize(nb);
  for (int32_t b = nb - 1; b >= 0; --b) {
    int32_t e = b + 1;
    for (int32_t k = P.child_starts[b]; k < P.child_starts[b + 1]; ++k) e = std::max(e, P.subtree_end[P.children[k]]);
    P.subtree_end[b] = e;
  }
  P.level_starts.assign(P.nlev + 1, 0);
  for (int32_t b = 0; b < nb; ++b) P.level_starts[P.level[b] + 1]++;
  for (int l = 0; l < P.nlev; ++l) P.level_starts[l + 1] += P.level_starts[l];
  P.level_boxes.resize(nb);
  {
    std::vector<int32_t> fill(P.level_starts.begin(), P.level_starts.end() - 1);
    for (int32_t b = 0; b < nb; ++b) P.level_boxes[fill[P.level[b]]++] = b;
  }

  // per-role box-sorted arrays and ranges
  std::vector<int32_t> cs(np + 1, 0), cc(np + 1, 0), ct(np + 1, 0);
  P.src_perm.clear();
  P.ctr_perm.clear();
  P.tgt_perm.clear();
  P.src_perm.reserve(P.ns);
  P.ctr_perm.reserve(P.nc);
  P.tgt_perm.reserve(P.nconv);
  for (int64_t i = 0; i < np; ++i) {
    const int32_t k = perm[i];
    cs[i + 1] = cs[i];
    cc[i + 1] = cc[i];
    ct[i + 1] = ct[i];
    if (role[k] == 0) {
      P.src_perm.push_back(k);
      cs[i + 1]++;
    } else if (role[k] == 1) {
      P.ctr_perm.push_back(int32_t(k - P.ns));
      cc[i + 1]++;
    } else {
      P.tgt_perm.push_back(conv[k - P.ns - P.nc]);
      ct[i + 1]++;
    }
  }
  auto fill_role = [&](const std::vector<int32_t>& pre, std::vector<int32_t>& os, std::vector<int32_t>& oc,
                       std::vector<int32_t>& ss, std::vector<int32_t>& sc) {
    os.resize(nb);
    oc.resize(nb);
    ss.resize(nb);
    sc.resize(nb);
    for (int32_t b = 0; b < nb; ++b) {
      os[b] = pre[bstart[b]];
      oc[b] = pre[bstart[b] + bown[b]] - pre[bstart[b]];
      ss[b] = pre[bstart[b]];
      sc[b] = pre[bend[b]] - pre[bstart[b]];
    }
  };
  fill_role(cs, P.src_own_start, P.src_own_count, P.src_sub_start, P.src_sub_count);
  fill_role(cc, P.ctr_own_start, P.ctr_own_count, P.ctr_sub_start, P.ctr_sub_count);
  fill_role(ct, P.tgt_own_start, P.tgt_own_count, P.tgt_sub_start, P.tgt_sub_count);

  P.flags.assign(nb, 0);
  for (int32_t b = 0; b < nb; ++b) {
    uint8_t f = 0;
    if (P.ctr_own_count[b] + P.tgt_own_count[b] > 0) f |= QBXG_BOX_TARGET;
    if (P.ctr_sub_count[b] + P.tgt_sub_count[b] > P.ctr_own_count[b] + P.tgt_own_count[b]) f |= QBXG_BOX_TARGET_ANCESTOR;
    if (P.src_sub_count[b] > 0) f |= QBXG_BOX_HAS_SOURCES;
    if (P.leaf(b)) f |= QBXG_BOX_LEAF;
    P.flags[b] = f;
  }
  P.t_tree = now_seconds() - t0;
}

namespace {
void flatten(const std::vector<std::vector<int32_t>>& rows, std::vector<int64_t>& starts, std::vector<int32_t>& out) {
  starts.assign(rows.size() + 1, 0);
  for (size_t b = 0; b < rows.size(); ++b) starts[b + 1] = starts[b] + int64_t(rows[b].size());
  out.resize(size_t(starts.back()));
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < int64_t(rows.size()); ++b)
    std::copy(rows[b].begin(), rows[b].end(), out.begin() + starts[b]);
}
}  // namespace

void hash_lists(Plan& P) {
  // one list per thread: FNV-1a is serial within a list (~1 ns per byte)
#pragma omp parallel for schedule(dynamic, 1) num_threads(QBXG_NUM_LISTS)
  for (int k = 0; k < QBXG_NUM_LISTS; ++k) {
    const uint64_t hsh = fnv1a(P.lst_starts[k].data(), P.lst_starts[k].size() * sizeof(int64_t));
    P.hash[k] = fnv1a(P.lst[k].data(), P.lst[k].size() * sizeof(int32_t), hsh);
  }
}

void build_lists(Plan& P) {
  const double t0 = now_seconds();
  const int32_t nb = P.nb;
  const double tf = P.cfg.t_f;
  const int32_t demote = P.cfg.w_far_demote;

  // 2-colleagues (same level, within the 2-near neighbourhood B_inf(5|b|), incl. self)
  P.coll.assign(nb, {});
  P.coll[0] = {0};
  for (int l = 1; l < P.nlev; ++l) {
    const int32_t a = P.level_starts[l], e = P.level_starts[l + 1];
#pragma omp parallel for schedule(dynamic, 64)
    for (int32_t i = a; i < e; ++i) {
      const int32_t b = P.level_boxes[i];
      auto& row = P.coll[b];
      for (int32_t pc : P.coll[P.parent[b]])
        for (int32_t k = P.child_starts[pc]; k < P.child_starts[pc + 1]; ++k) {
          const int32_t d = P.children[k];
          if (P.cheb(d, b) <= 2) row.push_back(d);
        }
      std::sort(row.begin(), row.end());
    }
  }

  std::vector<std::vector<int32_t>> rows[QBXG_NUM_LISTS];
  for (auto& r : rows) r.assign(nb, {});
  auto is_tgt = [&](int32_t b) { return (P.flags[b] & QBXG_BOX_TARGET) != 0; };
  auto is_tgt_or_anc = [&](int32_t b) { return (P.flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR)) != 0; };

  // U, W_close, W_far (target boxes); V (target and target-ancestor boxes)
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t b = 0; b < nb; ++b) {
    if (is_tgt_or_anc(b) && b != 0) {
      auto& v = rows[QBXG_LIST_V][b];
      for (int32_t pc : P.coll[P.parent[b]])
        for (int32_t k = P.child_starts[pc]; k < P.child_starts[pc + 1]; ++k) {
          const int32_t d = P.children[k];
          if (P.has_src(d) && P.cheb(d, b) > 2) v.push_back(d);
        }
      std::sort(v.begin(), v.end());
    }
    if (!is_tgt(b)) continue;
    // List 1 (Definition 1): source leaves in Desc(b) u {b} and leaves adjacent to b
    auto& u = rows[QBXG_LIST_U][b];
    for (int32_t d = b; d < P.subtree_end[b]; ++d)
      if (P.leaf(d) && P.src_own_count[d] > 0) u.push_back(d);
    std::vector<int32_t> stack;
    for (int32_t e : P.coll[b]) {
      if (e == b || P.cheb(e, b) > 1) continue;
      stack.push_back(e);
      while (!stack.empty()) {
        const int32_t x = stack.back();
        stack.pop_back();
        if (!P.has_src(x) || !P.adjacent(x, b)) continue;
        if (P.leaf(x)) {
          u.push_back(x);
        } else {
          for (int32_t k = P.child_starts[x]; k < P.child_starts[x + 1]; ++k) stack.push_back(P.children[k]);
        }
      }
    }
    for (int32_t a = P.parent[b]; a >= 0; a = P.parent[a])
      for (int32_t e : P.coll[a])
        if (e != a && P.cheb(e, a) <= 1 && P.leaf(e) && P.src_own_count[e] > 0 && P.adjacent(e, b)) u.push_back(e);
    std::sort(u.begin(), u.end());

    // List 3 (Definition 3) split into close / far (Definitions 5, 6)
    auto& wc = rows[QBXG_LIST_W_CLOSE][b];
    auto& wf = rows[QBXG_LIST_W_FAR][b];
    std::vector<int32_t> l3;
    for (int32_t e : P.coll[b]) {
      if (e == b || P.leaf(e)) continue;
      for (int32_t k = P.child_starts[e]; k < P.child_starts[e + 1]; ++k) stack.push_back(P.children[k]);
      while (!stack.empty()) {
        const int32_t d = stack.back();
        stack.pop_back();
        if (!P.has_src(d)) continue;
        if (!P.adjacent(d, b)) {
          l3.push_back(d);
        } else if (!P.leaf(d)) {
          for (int32_t k = P.child_starts[d]; k < P.child_starts[d + 1]; ++k) stack.push_back(P.children[k]);
        }
      }
    }
    const double* cb = &P.center[3 * b];
    for (int32_t d0 : l3) {
      stack.push_back(d0);
      while (!stack.empty()) {
        const int32_t d = stack.back();
        stack.pop_back();
        if (!P.has_src(d)) continue;
        if (sep_box_tcr(&P.center[3 * d], P.h[d], cb, P.h[b], tf)) {
          if (demote > 0 && P.src_sub_count[d] < demote) {
            // Remark 1: replace by its source leaves in W_close
            for (int32_t x = d; x < P.subtree_end[d]; ++x)
              if (P.leaf(x) && P.src_own_count[x] > 0) wc.push_back(x);
          } else {
            wf.push_back(d);
          }
        } else if (P.leaf(d)) {
          wc.push_back(d);
        } else {
          for (int32_t k = P.child_starts[d]; k < P.child_starts[d + 1]; ++k) stack.push_back(P.children[k]);
        }
      }
    }
    std::sort(wc.begin(), wc.end());
    std::sort(wf.begin(), wf.end());
  }

  // List 4 (Definition 4), then close / far (Definitions 7, 8), top-down
  std::vector<std::vector<int32_t>> l4(nb);
  for (int l = 0; l < P.nlev; ++l) {
    const int32_t a = P.level_starts[l], e = P.level_starts[l + 1];
#pragma omp parallel for schedule(dynamic, 64)
    for (int32_t i = a; i < e; ++i) {
      const int32_t b = P.level_boxes[i];
      if (!is_tgt_or_anc(b)) continue;
      auto& x4 = l4[b];
      for (int32_t c : P.coll[b])
        if (c != b && P.leaf(c) && P.src_own_count[c] > 0 && !P.adjacent(c, b)) x4.push_back(c);
      const int32_t par = P.parent[b];
      if (par >= 0) {
        for (int32_t anc = par; anc >= 0; anc = P.parent[anc])
          for (int32_t c : P.coll[anc])
            if (P.leaf(c) && P.src_own_count[c] > 0 && P.adjacent(c, par) && !P.adjacent(c, b)) x4.push_back(c);
      }
      std::vector<int32_t> cand = x4;
      if (par >= 0) cand.insert(cand.end(), rows[QBXG_LIST_X_CLOSE][par].begin(), rows[QBXG_LIST_X_CLOSE][par].end());
      auto& xc = rows[QBXG_LIST_X_CLOSE][b];
      auto& xf = rows[QBXG_LIST_X_FAR][b];
      const double* cb = &P.center[3 * b];
      for (int32_t d : cand) {
        if (sep_tcr_box(cb, P.h[b], &P.center[3 * d], P.h[d], tf))
          xf.push_back(d);
        else
          xc.push_back(d);
      }
      std::sort(xc.begin(), xc.end());
      std::sort(xf.begin(), xf.end());
    }
  }

  for (int k = 0; k < QBXG_NUM_LISTS; ++k) flatten(rows[k], P.lst_starts[k], P.lst[k]);
  hash_lists(P);
  P.t_lists = now_seconds() - t0;
}

void compute_ledger(const Plan& P, qbxg_ledger& L) {
  std::memset(&L, 0, sizeof(L));
  const double p = P.cfg.p_fmm, q = P.cfg.p_qbx;
  for (int32_t b = 0; b < P.nb; ++b) {
    const double nt = P.ctr_own_count[b];  // Table 3: n_t = QBX centres in the target box
    const int64_t nctr = P.ctr_own_count[b], ntg = P.tgt_own_count[b];
    for (int k = 0; k < QBXG_NUM_LISTS; ++k) {
      for (int64_t i = P.lst_starts[k][b]; i < P.lst_starts[k][b + 1]; ++i) {
        const int32_t d = P.lst[k][i];
        const double ns = P.src_sub_count[d];
        L.entries[k]++;
        switch (k) {
          case QBXG_LIST_U:
          case QBXG_LIST_W_CLOSE:
          case QBXG_LIST_X_CLOSE:
            L.modeled[k] += q * q * ns * nt;
            L.pairs_qbx_near += int64_t(ns) * nctr;
            L.pairs_p2p_near += int64_t(ns) * ntg;
            break;
          case QBXG_LIST_V:
            L.modeled[k] += p * p * p;
            break;
          case QBXG_LIST_W_FAR:
            L.modeled[k] += p * p * p * nt;
            L.pairs_wfar_centre += nctr;
            L.pairs_wfar_target += ntg;
            break;
          case QBXG_LIST_X_FAR:
            L.modeled[k] += p * p * ns;
            L.pairs_xfar_source += int64_t(ns);
            break;
        }
      }
    }
    if (P.parent[b] >= 0 && P.has_src(b)) L.n_m2m++;
    if (P.parent[b] >= 0 && (P.flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR))) L.n_l2l++;
    if (P.leaf(b)) L.n_p2m_sources += P.src_own_count[b];
    L.n_l2qbxl_centres += nctr;
    L.n_l2p_targets += ntg;
  }
  for (int k = 0; k < QBXG_NUM_LISTS; ++k) L.modeled_total += L.modeled[k];
  L.n_qbxl2p_targets = P.ntgt - P.nconv;
}

// Contiguous DFS-preorder ranges balanced by a per-box cost estimate (fp64
// flops of the work attached to the box: near field, List 2, List 3 far,
// List 4 far, L2QBXL, upward/downward shifts; SURVEY.md §8d unit costs at
// p=15, q=5 scaled with the configured orders).
void compute_shard(const Plan& P, int nranks, int rank, std::vector<int32_t>& cuts, std::vector<uint8_t>& mask) {
  const int32_t nb = P.nb;
  const double p = P.cfg.p_fmm, q = P.cfg.p_qbx;
  const double kp = (p + 1) * (p + 2) / 2, kq = (q + 1) * (q + 2) / 2;
  const double c_near = 26 * kq + 40, c_dense = 2 * std::pow(p + 1, 4), c_wfar = 8 * kp * kq, c_p2 = 26 * kp + 40;
  std::vector<double> cost(nb, 0.0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int32_t b = 0; b < nb; ++b) {
    const double nc = P.ctr_own_count[b], nt = P.tgt_own_count[b];
    double c = c_dense;  // one shift up and one down
    for (int k : {int(QBXG_LIST_U), int(QBXG_LIST_W_CLOSE), int(QBXG_LIST_X_CLOSE)})
      for (int64_t i = P.lst_starts[k][b]; i < P.lst_starts[k][b + 1]; ++i)
        c += P.src_own_count[P.lst[k][i]] * (c_near * nc + 30 * nt);
    c += double(P.lst_starts[QBXG_LIST_V][b + 1] - P.lst_starts[QBXG_LIST_V][b]) * c_dense;
    c += double(P.lst_starts[QBXG_LIST_W_FAR][b + 1] - P.lst_starts[QBXG_LIST_W_FAR][b]) * (c_wfar * nc + c_p2 * nt);
    for (int64_t i = P.lst_starts[QBXG_LIST_X_FAR][b]; i < P.lst_starts[QBXG_LIST_X_FAR][b + 1]; ++i)
      c += P.src_own_count[P.lst[QBXG_LIST_X_FAR][i]] * c_p2;
    c += nc * c_wfar + P.src_own_count[b] * c_p2;
    cost[b] = c;
  }
  double total = 0;
  for (double c : cost) total += c;
  cuts.assign(nranks + 1, nb);
  cuts[0] = 0;
  double acc = 0;
  int k = 1;
  for (int32_t b = 0; b < nb && k < nranks; ++b) {
    while (k < nranks && acc >= total * k / nranks) cuts[k++] = b;
    acc += cost[b];
  }
  for (; k < nranks; ++k) cuts[k] = nb;
  mask.assign(nb, 0);
  const int32_t lo = cuts[rank], hi = cuts[rank + 1];
  // straddling: subtree [b, end) not inside one rank range
  std::vector<int32_t> owner(nb, 0);
  for (int r = 0; r < nranks; ++r)
    for (int32_t b = cuts[r]; b < cuts[r + 1]; ++b) owner[b] = r;
  for (int32_t b = 0; b < nb; ++b) {
    uint8_t m = 0;
    const int32_t e = P.subtree_end[b];
    if (b >= lo && b < hi) m |= QBXG_SHARD_OWN;
    if (b >= lo && e <= hi) m |= QBXG_SHARD_SUBTREE;
    if (e > cuts[owner[b] + 1]) m |= QBXG_SHARD_STRADDLE;
    if (b >= lo && b < hi) m |= QBXG_SHARD_DOWN;
    mask[b] = m;
  }
  if (lo < nb)
    for (int32_t a = P.parent[lo]; a >= 0; a = P.parent[a]) mask[a] |= QBXG_SHARD_DOWN;
}

}  // namespace qbxg


extern "C" int qbxg_plan_shard(const qbxg_plan* pl, int32_t n_ranks, int32_t rank, int32_t* cuts, uint8_t* mask) {
  return qbxg::guarded([&] {
    if (!pl || !cuts) throw qbxg::InvalidArgument("plan_shard: null argument");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) throw qbxg::InvalidArgument("plan_shard: bad rank");
    std::vector<int32_t> c;
    std::vector<uint8_t> m;
    qbxg::compute_shard(pl->p, n_ranks, rank, c, m);
    std::copy(c.begin(), c.end(), cuts);
    if (mask) std::copy(m.begin(), m.end(), mask);
  });
}

extern "C" {

int qbxg_plan_create(const qbxg_config* cfg, const qbxg_geometry* geom, qbxg_plan** out) {
  return qbxg::guarded([&] {
    if (!cfg || !geom || !out) throw qbxg::InvalidArgument("plan_create: null argument");
    qbxg::validate_inputs(*cfg, *geom);
    auto* pl = new qbxg_plan;
    try {
      pl->p.cfg = *cfg;
      qbxg::build_tree(pl->p, *geom);
      qbxg::build_lists(pl->p);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

int qbxg_plan_create_gpu(const qbxg_config* cfg, const qbxg_geometry* geom, int32_t gpu_lists, qbxg_plan** out) {
  return qbxg::guarded([&] {
    if (!cfg || !geom || !out) throw qbxg::InvalidArgument("plan_create_gpu: null argument");
    qbxg::validate_inputs(*cfg, *geom);
    if (cfg->level_restrict)
      throw qbxg::InvalidArgument("plan_create_gpu: level restriction is built by the host plan (qbxg_plan_create)");
    auto* pl = new qbxg_plan;
    try {
      pl->p.cfg = *cfg;
      qbxg::build_tree_gpu(pl->p, *geom);
      if (gpu_lists)
        qbxg::build_lists_gpu(pl->p);
      else
        qbxg::build_lists(pl->p);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

int qbxg_plan_view_get(const qbxg_plan* pl, qbxg_plan_view* v) {
  return qbxg::guarded([&] {
    if (!pl || !v) throw qbxg::InvalidArgument("plan_view: null argument");
    const auto& P = pl->p;
    std::memset(v, 0, sizeof(*v));
    v->n_boxes = P.nb;
    v->n_levels = P.nlev;
    for (int d = 0; d < 3; ++d) v->root_center[d] = P.root_c[d];
    v->root_radius = P.root_h;
    v->box_center = P.center.data();
    v->box_radius = P.h.data();
    v->box_level = P.level.data();
    v->box_parent = P.parent.data();
    v->child_starts = P.child_starts.data();
    v->children = P.children.data();
    v->level_starts = P.level_starts.data();
    v->level_boxes = P.level_boxes.data();
    v->src_own_start = P.src_own_start.data();
    v->src_own_count = P.src_own_count.data();
    v->src_sub_start = P.src_sub_start.data();
    v->src_sub_count = P.src_sub_count.data();
    v->ctr_own_start = P.ctr_own_start.data();
    v->ctr_own_count = P.ctr_own_count.data();
    v->ctr_sub_start = P.ctr_sub_start.data();
    v->ctr_sub_count = P.ctr_sub_count.data();
    v->tgt_own_start = P.tgt_own_start.data();
    v->tgt_own_count = P.tgt_own_count.data();
    v->tgt_sub_start = P.tgt_sub_start.data();
    v->tgt_sub_count = P.tgt_sub_count.data();
    v->n_sources = P.ns;
    v->n_centers = P.nc;
    v->n_conv_targets = P.nconv;
    v->n_targets = P.ntgt;
    v->src_perm = P.src_perm.data();
    v->ctr_perm = P.ctr_perm.data();
    v->tgt_perm = P.tgt_perm.data();
    v->box_flags = P.flags.data();
    for (int k = 0; k < QBXG_NUM_LISTS; ++k) {
      v->list_starts[k] = P.lst_starts[k].data();
      v->list_boxes[k] = P.lst[k].data();
      v->list_hash[k] = P.hash[k];
    }
    v->build_seconds_tree = P.t_tree;
    v->build_seconds_lists = P.t_lists;
  });
}

int qbxg_plan_ledger(const qbxg_plan* pl, qbxg_ledger* out) {
  return qbxg::guarded([&] {
    if (!pl || !out) throw qbxg::InvalidArgument("plan_ledger: null argument");
    qbxg::compute_ledger(pl->p, *out);
  });
}

void qbxg_plan_destroy(qbxg_plan* pl) { delete pl; }

}  // extern "C"
