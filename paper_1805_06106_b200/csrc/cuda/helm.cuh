// Helmholtz single- and double-layer FMM (helm_fmm.cu): device data and launchers.
#pragma once

#include <vector>

#include <cstdint>

#include <cuda_runtime.h>

namespace qbxg {
namespace dev {

struct HelmData {
  double k;
  int P, Q, KP, KQ, GL;  // orders, full table sizes (P+1)^2 / (Q+1)^2, Gaunt l-slots (P+1)
  // tree and particles (shared with the Laplace uploads)
  const double4* box;
  const int* child_starts;
  const int* children;
  const int* parent;
  const int* src_own_start;
  const int* src_own_count;
  const int* ctr_own_start;
  const int* ctr_own_count;
  const int* tgt_own_start;
  const int* tgt_own_count;
  const double4* src;  // positions (w unused)
  const double4* ctr;  // (x, y, z, r)
  const double4* tgt;
  double2* hw;         // sorted complex weights
  double2* hmu;        // sorted complex dipole moments (3 per source), null for the single layer
  // expansions: full complex tables, index n^2 + n + m
  double2* M;          // nb x KP
  double2* L;          // nb x KP
  double2* Lc;         // nc x KQ (sorted centre order)
  double2* phi;        // conventional targets (sorted)
  // lists
  const int64_t* near_starts;
  const int2* near_seg;
  const int64_t* xfar_starts;
  const int2* xfar_seg;
  const int64_t* v_starts;
  const int64_t* wfar_starts;
  const int* wfar_box;
  const double* gaunt;  // KP x KP x GL
  // the same coefficients in the order the centre translations read them:
  // [|mu|][sign][l][term k][row i'] (n = n_lo + 2k), consecutive rows i' contiguous
  const double* gaunt_ctr;
  unsigned int* bad;    // Stage 9 non-finite flag (shared with the Laplace DevData)
};

// one centre-translation CTA: box, first entry in the item list, count (<= kHCtrMax)
constexpr int kHCtrMax = 32;

void helm_upload_constants();  // solid-harmonic recurrence tables (this TU's __constant__)
int helm_gather(const HelmData& H, int64_t ns, const int* perm, const double* w, const double* mu, cudaStream_t s);
int helm_p2m(const HelmData& H, const int* leaves, int n, cudaStream_t s);
int helm_build_ops(const HelmData& H, int n_ops, const double4* shifts, double2* ops, cudaStream_t s);
// M2M (mode 0: M[dst] += T M[src]) / L2L (mode 1: L[dst] += T L[src]) over (src, dst)
// pairs that share one (level, octant) operator, 8 pairs per CTA
int helm_shift_pairs(const HelmData& H, int mode, const int2* pairs, int n, const double2* ops, cudaStream_t s);
int helm_m2l_split_cols();
// point-and-shoot M2L (even / odd split frame): Z blocks + e^{i m alpha} per operator,
// block tables, apply (pas kernel + the split reduce)
bool helm_pas_supported(int P);
int helm_build_zpas(const HelmData& H, int n_ops, const double4* shifts, const int* z_off, int zstride, double* zops,
                    double2* cs, cudaStream_t s);
void helm_pas_tables(int P, const size_t* wv_off_w0, const size_t* wv_off_w1, const size_t* wv_off_v0,
                     const size_t* wv_off_v1, const size_t* z_off, std::vector<int>& tab, int (&base)[2][3]);
int helm_m2l_pas(const HelmData& H, int n_tiles, const int4* tiles, const int* col_src, const int* col_pos,
                 const int* tab, int tab_n, const int (&base)[2][3], const double* zops, int zstride,
                 const double* wvops, int wvstride, const int* op_cls, const double2* cs, double2* temp, int n_boxes,
                 const int* boxes, int64_t vbase, const int* ent_op, cudaStream_t s);
int helm_near(const HelmData& H, const int* boxes, int n, cudaStream_t s);
int helm_p2p(const HelmData& H, const int* boxes, int n, cudaStream_t s);
int helm_p2l(const HelmData& H, const int* boxes, int n, cudaStream_t s);
// centre translations: ctas (box, first, count) over item lists ctr_of (sorted centre)
// and out_row (row of `out`, KQ complex each); accumulate = add into out rows
size_t helm_gaunt_ctr_size(int P, int Q);
int helm_build_gaunt_ctr(const HelmData& H, double* out, cudaStream_t s);
int helm_ctr(const HelmData& H, int singular, const double2* X, int n_ctas, const int4* ctas, const int* ctr_of,
             const int* out_row, double2* out, int accumulate, cudaStream_t s);
int helm_pair_reduce(const HelmData& H, const int* centres, const int* starts, int n, const double2* rows,
                     cudaStream_t s);
int helm_m2p(const HelmData& H, const int* boxes, int n, cudaStream_t s);
int helm_eval(const HelmData& H, int n_assoc, const int* assoc_items, const double* tpos, const int* assoc,
              const int* ctr_sorted, int n_tboxes, const int* tboxes, const int* tgt_perm, double* pot,
              cudaStream_t s);
int helm_centre_out(const HelmData& H, int nc, const int* ctr_perm, double* out, cudaStream_t s);

}  // namespace dev
}  // namespace qbxg
