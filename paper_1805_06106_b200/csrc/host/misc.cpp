// Thread-local last-error storage and version string for the C ABI.
#include <string>

#include "common.hpp"
#include "predicates.hpp"

namespace qbxg {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* get_last_error() { return g_last_error.c_str(); }

}  // namespace qbxg

extern "C" {

const char* qbxg_last_error(void) { return qbxg::get_last_error(); }

const char* qbxg_version(void) {
  return "qbxg 0.2 (sm_100a; fp64 Laplace SL / SL+DL, complex128 Helmholtz SL / SL+DL)";
}

int qbxg_adequately_separated(int32_t kind, const double* ca, double ha, const double* cb, double hb, double t_f,
                              int32_t* out) {
  return qbxg::guarded([&] {
    if (!ca || !cb || !out || (kind != 0 && kind != 1))
      throw qbxg::InvalidArgument("qbxg_adequately_separated: bad argument");
    *out = kind == 0 ? qbxg::sep_box_tcr(ca, ha, cb, hb, t_f) : qbxg::sep_tcr_box(ca, ha, cb, hb, t_f);
  });
}

}  // extern "C"
