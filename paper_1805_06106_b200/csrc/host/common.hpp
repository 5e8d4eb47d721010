// Shared host-side utilities: status/exception mapping across the C ABI,
// deterministic RNG, timers and hashing.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qbxg.h"

namespace qbxg {

// Exceptions used inside the library; mapped to status codes at the ABI edge.
// They mirror std::invalid_argument / std::domain_error thrown by the reference
// (/root/reference/proj/src/kernels.cpp:15, 22, 28-36, 69-71).
struct InvalidArgument : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NcclError : std::runtime_error { using std::runtime_error::runtime_error; };

void set_last_error(const std::string& msg);
// Helmholtz translation Gaunt table (helm_tables.cpp): (P+1)^4 x (P+1) doubles
std::vector<double> helm_gaunt_table(int P);
const char* get_last_error();

// Run f, translating exceptions to status codes; never lets one escape.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return QBXG_OK;
  } catch (const InvalidArgument& e) {
    set_last_error(e.what());
    return QBXG_ERR_INVALID_ARGUMENT;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return QBXG_ERR_INVALID_ARGUMENT;
  } catch (const DomainError& e) {
    set_last_error(e.what());
    return QBXG_ERR_DOMAIN;
  } catch (const std::domain_error& e) {
    set_last_error(e.what());
    return QBXG_ERR_DOMAIN;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return QBXG_ERR_CUDA;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return QBXG_ERR_NCCL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return QBXG_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return QBXG_ERR_INTERNAL;
  }
}

// SplitMix-seeded xoshiro is not needed: the survey pins std::mt19937_64 draw
// order.  We implement mt19937_64 via <random> and derive
// doubles with a fixed 53-bit mapping so every platform sees the same stream.
struct Rng {
  explicit Rng(uint64_t seed);
  uint64_t next();
  double uniform01();                 // [0,1)
  double uniform(double a, double b); // [a,b)
  int64_t uniform_int(int64_t lo, int64_t hi);  // inclusive
  void* state;
  ~Rng();
  Rng(const Rng&) = delete;
  Rng& operator=(const Rng&) = delete;
};

inline double now_seconds() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

inline uint64_t fnv1a(const void* data, size_t n, uint64_t h = 1469598103934665603ull) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace qbxg
