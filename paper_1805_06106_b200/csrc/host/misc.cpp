// Thread-local last-error storage and version string for the C ABI.
#include <string>

#include "common.hpp"

namespace qbxg {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* get_last_error() { return g_last_error.c_str(); }

}  // namespace qbxg

extern "C" {

const char* qbxg_last_error(void) { return qbxg::get_last_error(); }

const char* qbxg_version(void) { return "qbxg 0.1 (sm_100a, fp64 Laplace SL/SL+DL)"; }

}  // extern "C"
