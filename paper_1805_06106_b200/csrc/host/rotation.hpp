// Rotation blocks for the point-and-shoot M2L:
// M2L along offset v = rotate the multipole so v lies on +z, translate along z
// (coefficients (-1)^{n+m} (j+n)!/|v|^{j+n+1}, diagonal in m), rotate the local
// back.  Blocks act on the real degrees of freedom of one degree n
// (index 0 = Re X_n^0, 2m-1+part = Re/Im X_n^m), row-major [out][in].
// Derivation and check against the dense operator: tests/test_rotation_math.py.
#pragma once

#include <cstddef>

namespace qbxg {

// sum_{j<=p} (2j+1)^2 and the offset of degree j's block
inline size_t rot_blocks_size(int p) { return size_t(p + 1) * (2 * p + 1) * (2 * p + 3) / 3; }
inline size_t rot_block_offset(int j) { return size_t(j) * (4 * size_t(j) * j - 1) / 3; }

// Rf: multipole rotation (v -> +z); Rb: local back-rotation; both rot_blocks_size(p) doubles.
void m2l_rotation_blocks(int p, const double v[3], double* Rf, double* Rb);

}  // namespace qbxg
