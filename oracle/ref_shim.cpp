// ORACLE -- test infrastructure only.
// extern "C" shim over the reference's own qbx::direct_sum / laplace_green /
// laplace_dipole (/root/reference/proj/src/kernels.cpp:13-73), compiled from the
// reference sources where they lie by oracle/Makefile into oracle/_ref/.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qbx3d/kernels.hpp"

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* qbxref_last_error(void) { return g_err.c_str(); }

int qbxref_laplace_green(const double* x, const double* y, double* out) {
  try {
    *out = qbx::laplace_green({x[0], x[1], x[2]}, {y[0], y[1], y[2]});
    return 0;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  }
}

int qbxref_laplace_dipole(const double* x, const double* y, const double* m, double* out) {
  try {
    *out = qbx::laplace_dipole({x[0], x[1], x[2]}, {y[0], y[1], y[2]}, {m[0], m[1], m[2]});
    return 0;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  }
}

// Returns 0 ok, 1 invalid_argument, 2 domain_error (message in qbxref_last_error).
int qbxref_direct_sum(int64_t ns, const double* pos, const double* w, const double* mu, int64_t nt,
                      const double* tpos, double* out) {
  try {
    qbx::SourceEnsemble S;
    S.positions.resize(ns);
    S.weights.assign(w, w + ns);
    for (int64_t i = 0; i < ns; ++i) S.positions[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    if (mu) {
      S.dipole_moments.resize(ns);
      for (int64_t i = 0; i < ns; ++i) S.dipole_moments[i] = {mu[3 * i], mu[3 * i + 1], mu[3 * i + 2]};
    }
    qbx::TargetSet T;
    T.positions.resize(nt);
    for (int64_t i = 0; i < nt; ++i) T.positions[i] = {tpos[3 * i], tpos[3 * i + 1], tpos[3 * i + 2]};
    T.association.assign(nt, -1);
    std::vector<double> r = qbx::direct_sum(S, T);
    for (int64_t i = 0; i < nt; ++i) out[i] = r[i];
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"
