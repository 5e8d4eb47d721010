// ORACLE -- test infrastructure only.
//
// Brute-force, definition-by-definition construction of the GIGAQBX
// interaction lists (Definitions 1-8) over all box pairs,
// O(N_B^2 * depth).  SPEC.md:386 and 398 require the production lists to equal
// this on small trees ("lists vs brute-force definitions on depth<=4 trees").
// It shares nothing with the production builder: the two separation relations
// are restated below from SPEC.md:370-378 (and checked against its worked examples
// and against the product's predicates in tests/test_predicates.py), and box
// integer coordinates are derived independently from box centres.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "qbxg.h"

namespace {

// SPEC.md:373 box_vs_tcr: the l2 distance from centre(a) to the boundary of
// TCR(b) -- the ball of radius sqrt(3)|b|(1 + t_f) about centre(b)
// -- is at least 3|a|.  A centre inside the ball has no such distance (false).
bool oracle_box_vs_tcr(const double* ca, double ha, const double* cb, double hb, double tf) {
  double d2 = 0.0;
  for (int k = 0; k < 3; ++k) d2 += (ca[k] - cb[k]) * (ca[k] - cb[k]);
  const double tcr_radius = std::sqrt(3.0) * hb * (1.0 + tf);
  return std::sqrt(d2) - tcr_radius >= 3.0 * ha;
}

// SPEC.md:373 tcr_vs_box: the l-inf distance from centre(a) to the boundary of box b
// is at least 3|a|(1 + t_f).
bool oracle_tcr_vs_box(const double* ca, double ha, const double* cb, double hb, double tf) {
  double dinf = 0.0;
  for (int k = 0; k < 3; ++k) dinf = std::max(dinf, std::fabs(ca[k] - cb[k]));
  return dinf - hb >= 3.0 * ha * (1.0 + tf);
}

struct Boxes {
  const qbxg_plan_view* V;
  int nb;
  std::vector<int64_t> ic;
  std::vector<std::vector<int>> anc;  // strict ancestors, nearest first

  explicit Boxes(const qbxg_plan_view* v) : V(v), nb(v->n_boxes), ic(3 * size_t(v->n_boxes)), anc(v->n_boxes) {
    for (int b = 0; b < nb; ++b) {
      const double w = 2.0 * V->box_radius[b];
      for (int d = 0; d < 3; ++d) {
        const double lo = V->root_center[d] - V->root_radius;
        ic[3 * b + d] = int64_t(std::llround((V->box_center[3 * b + d] - lo) / w - 0.5));
      }
      for (int a = V->box_parent[b]; a >= 0; a = V->box_parent[a]) anc[b].push_back(a);
    }
  }
  bool leaf(int b) const { return V->child_starts[b + 1] == V->child_starts[b]; }
  bool src_leaf(int b) const { return leaf(b) && V->src_own_count[b] > 0; }
  bool has_src(int b) const { return V->src_sub_count[b] > 0; }
  bool is_anc(int a, int b) const {  // a strict ancestor of b
    return std::find(anc[b].begin(), anc[b].end(), a) != anc[b].end();
  }
  // closed boxes touch or overlap: compare the integer extents on the finer level's grid
  bool adjacent(int a, int b) const {
    const int la = V->box_level[a], lb = V->box_level[b], L = std::max(la, lb);
    for (int k = 0; k < 3; ++k) {
      const int64_t sa = int64_t(1) << (L - la), sb = int64_t(1) << (L - lb);
      const int64_t a0 = ic[3 * a + k] * sa, a1 = a0 + sa, b0 = ic[3 * b + k] * sb, b1 = b0 + sb;
      if (a1 < b0 || b1 < a0) return false;
    }
    return true;
  }
  bool colleague2(int a, int b) const {  // same level, inside the 2-near neighbourhood
    if (V->box_level[a] != V->box_level[b]) return false;
    for (int d = 0; d < 3; ++d)
      if (std::llabs(ic[3 * a + d] - ic[3 * b + d]) > 2) return false;
    return true;
  }
  bool target(int b) const { return V->box_flags[b] & QBXG_BOX_TARGET; }
  bool target_or_anc(int b) const { return V->box_flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR); }
};

}  // namespace

extern "C" {

// Fills six CSR lists (starts: n_boxes+1 int64 each, boxes: caller-provided
// capacity `cap` each); returns the number of entries of each list in counts.
// Returns 0 on success, 1 if a capacity is exceeded.
int qbxo_lists_brute(const qbxg_plan_view* V, double tf, int32_t demote, int64_t cap, int64_t* starts[6],
                     int32_t* boxes[6], int64_t counts[6]) {
  Boxes B(V);
  const int nb = B.nb;
  std::vector<std::vector<int>> rows[6];
  for (auto& r : rows) r.assign(nb, {});
  std::vector<std::vector<int>> L4(nb);
  auto ctr = [&](int b) { return &V->box_center[3 * b]; };
  auto h = [&](int b) { return V->box_radius[b]; };

  for (int b = 0; b < nb; ++b) {
    // Definition 2 (List 2)
    if (B.target_or_anc(b) && V->box_parent[b] >= 0) {
      const int pb = V->box_parent[b];
      for (int d = 0; d < nb; ++d) {
        if (V->box_level[d] != V->box_level[b] || !B.has_src(d)) continue;
        const int pd = V->box_parent[d];
        if (pd >= 0 && B.colleague2(pd, pb) && !B.colleague2(d, b)) rows[QBXG_LIST_V][b].push_back(d);
      }
    }
    if (B.target_or_anc(b)) {
      // Definition 4 (List 4)
      for (int d = 0; d < nb; ++d) {
        if (!B.src_leaf(d)) continue;
        bool in = false;
        if (B.colleague2(d, b) && !B.adjacent(d, b)) in = true;
        if (V->box_parent[b] >= 0) {
          bool coll_anc = false;
          for (int a : B.anc[b])
            if (B.colleague2(d, a)) coll_anc = true;
          if (coll_anc && B.adjacent(d, V->box_parent[b]) && !B.adjacent(d, b)) in = true;
        }
        if (in) L4[b].push_back(d);
      }
    }
    if (!B.target(b)) continue;
    // Definition 1 (List 1)
    for (int d = 0; d < nb; ++d)
      if (B.src_leaf(d) && (d == b || B.is_anc(b, d) || B.adjacent(d, b))) rows[QBXG_LIST_U][b].push_back(d);
    // Definition 3 (List 3): d in Desc(T_b), not adjacent, all ancestors inside Desc(T_b) adjacent
    auto in_desc_T = [&](int d) {
      for (int a : B.anc[d])
        if (B.colleague2(a, b)) return true;
      return false;
    };
    std::vector<char> l3(nb, 0);
    for (int d = 0; d < nb; ++d) {
      if (!B.has_src(d) || !in_desc_T(d) || B.adjacent(d, b)) continue;
      bool ok = true;
      for (int w : B.anc[d])
        if (in_desc_T(w) && !B.adjacent(w, b)) ok = false;
      if (ok) l3[d] = 1;
    }
    // Definitions 5, 6 over D = L3 u Desc(L3)
    auto in_D = [&](int d) {
      if (l3[d]) return true;
      for (int a : B.anc[d])
        if (l3[a]) return true;
      return false;
    };
    std::vector<int> far, close;
    for (int d = 0; d < nb; ++d) {
      if (!B.has_src(d) || !in_D(d)) continue;
      const bool sep = oracle_box_vs_tcr(ctr(d), h(d), ctr(b), h(b), tf);
      if (!sep) {
        if (B.src_leaf(d)) close.push_back(d);
        continue;
      }
      bool ok = true;
      for (int w : B.anc[d])
        if (in_D(w) && oracle_box_vs_tcr(ctr(w), h(w), ctr(b), h(b), tf)) ok = false;
      if (ok) far.push_back(d);
    }
    // Remark 1 demotion, applied identically to the production builder's rule
    for (int d : far) {
      if (demote > 0 && V->src_sub_count[d] < demote) {
        for (int x = 0; x < nb; ++x)
          if (B.src_leaf(x) && (x == d || B.is_anc(d, x))) close.push_back(x);
      } else {
        rows[QBXG_LIST_W_FAR][b].push_back(d);
      }
    }
    rows[QBXG_LIST_W_CLOSE][b] = close;
  }
  // Definitions 7, 8
  for (int b = 0; b < nb; ++b) {
    if (!B.target_or_anc(b)) continue;
    std::vector<int> xc;
    for (int w = 0; w < nb; ++w) {
      if (!(w == b || B.is_anc(w, b))) continue;
      for (int d : L4[w])
        if (!oracle_tcr_vs_box(ctr(b), h(b), ctr(d), h(d), tf)) xc.push_back(d);
    }
    rows[QBXG_LIST_X_CLOSE][b] = xc;
  }
  for (int b = 0; b < nb; ++b) {
    if (!B.target_or_anc(b)) continue;
    std::vector<int> xf;
    for (int d : L4[b])
      if (oracle_tcr_vs_box(ctr(b), h(b), ctr(d), h(d), tf)) xf.push_back(d);
    const int pb = V->box_parent[b];
    if (pb >= 0)
      for (int d : rows[QBXG_LIST_X_CLOSE][pb])
        if (oracle_tcr_vs_box(ctr(b), h(b), ctr(d), h(d), tf)) xf.push_back(d);
    rows[QBXG_LIST_X_FAR][b] = xf;
  }
  for (int k = 0; k < 6; ++k) {
    int64_t n = 0;
    starts[k][0] = 0;
    for (int b = 0; b < nb; ++b) {
      auto& r = rows[k][b];
      std::sort(r.begin(), r.end());
      for (int d : r) {
        if (n >= cap) return 1;
        boxes[k][n++] = d;
      }
      starts[k][b + 1] = n;
    }
    counts[k] = n;
  }
  return 0;
}

}  // extern "C"

extern "C" int qbxo_adequately_separated(int kind, const double* ca, double ha, const double* cb, double hb,
                                         double tf) {
  return kind == 0 ? oracle_box_vs_tcr(ca, ha, cb, hb, tf) : oracle_tcr_vs_box(ca, ha, cb, hb, tf);
}
