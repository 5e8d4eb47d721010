// Reference-side drop-in for the B200 path: keeps the reference's
// qbx:: signatures (/root/reference/proj/include/qbx3d/kernels.hpp) and forwards to the
// C ABI of include/qbxg.h, rethrowing the reference's exception types:
//   QBXG_ERR_INVALID_ARGUMENT -> std::invalid_argument (kernels.cpp:28-36)
//   QBXG_ERR_DOMAIN           -> std::domain_error     (kernels.cpp:15, 22, 69-71)
//   anything else             -> std::runtime_error    (no device, CUDA / NCCL failure)
// Vec3 is three doubles (vec3.hpp), so positions and moments pass zero-copy.
// Compiled against the reference header and exercised by integration/test_b200_wrapper.cpp
// (tests/test_integration.py).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qbx3d/kernels.hpp"
#include "qbxg.h"

namespace qbx {

inline void qbxg_throw(int st) {
  if (st == QBXG_OK) return;
  const std::string msg = qbxg_last_error();
  if (st == QBXG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == QBXG_ERR_DOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

// Same contract as direct_sum (kernels.cpp:46-73): validates, throws domain_error on a
// coincident target / source pair naming both.
inline std::vector<double> direct_sum_b200(const SourceEnsemble& s, const TargetSet& t) {
  s.validate();
  std::vector<double> pot(t.size());
  qbxg_throw(qbxg_direct_sum(int64_t(s.size()), s.size() ? &s.positions[0].x : nullptr, s.weights.data(),
                             s.has_dipoles() ? &s.dipole_moments[0].x : nullptr, int64_t(t.size()),
                             t.size() ? &t.positions[0].x : nullptr, pot.data()));
  return pot;
}

// execute(bundle, density, FmmConfig): the host plan (tree + lists) is
// built once per geometry, then apply() runs Stages 2-9 on the GPU per density.
class FmmB200 {
 public:
  FmmB200(const qbxg_config& cfg, const qbxg_geometry& g, int device = 0) {
    qbxg_throw(qbxg_plan_create(&cfg, &g, &plan_));
    const int st = qbxg_create(&cfg, &g, plan_, device, &h_);
    if (st != QBXG_OK) {
      qbxg_plan_destroy(plan_);
      qbxg_throw(st);
    }
    n_targets_ = size_t(g.n_targets);
  }
  ~FmmB200() {
    if (h_) qbxg_destroy(h_);
    if (plan_) qbxg_plan_destroy(plan_);
  }
  FmmB200(const FmmB200&) = delete;
  FmmB200& operator=(const FmmB200&) = delete;

  // densities as the reference's SourceEnsemble carries them: weights premultiplied,
  // dipole moments (SL+DL) = weight x density x normal; positions must be the geometry's
  std::vector<double> apply(const SourceEnsemble& s) {
    s.validate();
    std::vector<double> pot(n_targets_);
    qbxg_throw(qbxg_apply(h_, s.weights.data(), s.has_dipoles() ? &s.dipole_moments[0].x : nullptr, pot.data(),
                          nullptr, nullptr));
    return pot;
  }

 private:
  qbxg_plan* plan_ = nullptr;
  qbxg_handle* h_ = nullptr;
  size_t n_targets_ = 0;
};

}  // namespace qbx
