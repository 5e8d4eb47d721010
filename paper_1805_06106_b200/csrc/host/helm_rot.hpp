// Host tables of the Helmholtz point-and-shoot M2L (see helm_rot.cpp).
#pragma once

#include <cstddef>
#include <vector>

namespace qbxg {

// padded DMMA fragment storage of a real s x s block (rows to 8, columns to 4)
size_t hpas_frag_size(int s);
// row-major s x s block -> fragment order (ks, mt), 32 doubles each
void hpas_to_frags(int s, const double* B, double* out);

struct HpasLayout {
  // per theta class: [W even n=0..P | W odd n=1..P | V even | V odd], offsets in doubles
  std::vector<size_t> wv_off[2][2];  // [phase W=0 / V=1][parity][block]
  size_t wv_stride = 0;
  // per operator: Z_m (m = 0..P), real embedding [[Re, -Im], [Im, Re]] of size 2 (P + 1 - m)
  std::vector<size_t> z_off;
  size_t z_stride = 0;
};
HpasLayout hpas_layout(int P);

// W / V blocks for each polar angle (fragment order, hpas_layout strides)
void hpas_build_wv(int P, const std::vector<double>& thetas, std::vector<double>& out);

}  // namespace qbxg
