// Geometric predicates shared by the production list builder (plan.cpp) and
// the brute-force definitional list oracle (oracle/lists_brute.cpp).  Both
// sides must evaluate the adequate-separation relation with the same
// floating-point expression for list contents to match bit-exactly.
#pragma once

#include <cmath>
#include <cstdint>

namespace qbxg {

// a < TCR(b): l2 distance from centre(a) to the boundary of
// TCR(b) = B2(sqrt(3)|b|(1+t_f), centre(b)) is at least 3|a|.
// A box centre inside the TCR is never separated.
inline bool sep_box_tcr(const double* ca, double ha, const double* cb, double hb, double tf) {
  const double dx = ca[0] - cb[0], dy = ca[1] - cb[1], dz = ca[2] - cb[2];
  const double d = std::sqrt(dx * dx + dy * dy + dz * dz);
  return d - std::sqrt(3.0) * hb * (1.0 + tf) >= 3.0 * ha;
}

// TCR(a) < b: l-inf distance from centre(a) to the boundary of b is at least
// 3|a|(1+t_f).
inline bool sep_tcr_box(const double* ca, double ha, const double* cb, double hb, double tf) {
  const double dx = std::fabs(ca[0] - cb[0]), dy = std::fabs(ca[1] - cb[1]), dz = std::fabs(ca[2] - cb[2]);
  const double d = dx > dy ? (dx > dz ? dx : dz) : (dy > dz ? dy : dz);
  return d - hb >= 3.0 * ha * (1.0 + tf);
}

// Closed boxes a, b (integer coordinates at their levels) touch or overlap.
inline bool boxes_adjacent(const int64_t* ia, int la, const int64_t* ib, int lb) {
  const int L = la > lb ? la : lb;
  for (int d = 0; d < 3; ++d) {
    const int64_t alo = ia[d] << (L - la), ahi = (ia[d] + 1) << (L - la);
    const int64_t blo = ib[d] << (L - lb), bhi = (ib[d] + 1) << (L - lb);
    if (alo > bhi || blo > ahi) return false;
  }
  return true;
}

// Does a centre ball (c, r) fit the TCR of a box (cb, hb)?
inline bool ball_fits_tcr(const double* c, double r, const double* cb, double hb, double tf) {
  const double dx = c[0] - cb[0], dy = c[1] - cb[1], dz = c[2] - cb[2];
  return std::sqrt(dx * dx + dy * dy + dz * dz) + r <= std::sqrt(3.0) * hb * (1.0 + tf);
}

}  // namespace qbxg
