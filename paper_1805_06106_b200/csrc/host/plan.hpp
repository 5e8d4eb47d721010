// The host plan: target-confinement octree + interaction lists (plan.cpp
// builds it on the host, plan_gpu.cu on the device; both fill this struct).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <vector>

#include "common.hpp"
#include "predicates.hpp"

namespace qbxg {

constexpr int kMaxDepth = 60;

struct Plan {
  qbxg_config cfg{};
  int32_t nb = 0, nlev = 0;
  double root_c[3] = {0, 0, 0}, root_h = 1;
  std::vector<double> center, h;
  std::vector<int32_t> level, parent, child_starts, children, level_starts, level_boxes, subtree_end;
  std::vector<int64_t> ic;  // 3*nb integer coordinates at the box's level
  std::vector<int32_t> src_own_start, src_own_count, src_sub_start, src_sub_count;
  std::vector<int32_t> ctr_own_start, ctr_own_count, ctr_sub_start, ctr_sub_count;
  std::vector<int32_t> tgt_own_start, tgt_own_count, tgt_sub_start, tgt_sub_count;
  std::vector<int32_t> src_perm, ctr_perm, tgt_perm;
  std::vector<uint8_t> flags;
  std::vector<std::vector<int32_t>> coll;  // 2-colleagues incl. self, sorted
  std::vector<int64_t> lst_starts[QBXG_NUM_LISTS];
  std::vector<int32_t> lst[QBXG_NUM_LISTS];
  uint64_t hash[QBXG_NUM_LISTS] = {};
  int64_t ns = 0, nc = 0, nconv = 0, ntgt = 0;
  double t_tree = 0, t_lists = 0;

  bool leaf(int32_t b) const { return child_starts[b + 1] == child_starts[b]; }
  bool has_src(int32_t b) const { return src_sub_count[b] > 0; }
  bool adjacent(int32_t a, int32_t b) const {
    return boxes_adjacent(&ic[3 * a], level[a], &ic[3 * b], level[b]);
  }
  int64_t cheb(int32_t a, int32_t b) const {  // same-level offset (l-inf, in boxes)
    int64_t m = 0;
    for (int d = 0; d < 3; ++d) m = std::max<int64_t>(m, std::llabs(ic[3 * a + d] - ic[3 * b + d]));
    return m;
  }
};

void validate_inputs(const qbxg_config& cfg, const qbxg_geometry& g);
void build_tree(Plan& P, const qbxg_geometry& g);     // host (plan.cpp)
void build_lists(Plan& P);                            // host (plan.cpp)
void build_tree_gpu(Plan& P, const qbxg_geometry& g); // device (plan_gpu.cu)
void build_lists_gpu(Plan& P);                        // device (plan_gpu.cu)
void hash_lists(Plan& P);

}  // namespace qbxg

struct qbxg_plan {
  qbxg::Plan p;
};
