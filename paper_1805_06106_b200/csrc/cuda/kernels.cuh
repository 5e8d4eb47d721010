// Kernel interface shared by the stage kernels (kernels.cu) and the device
// handle (handle.cu).  One struct of device pointers, passed by value.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace qbxg {
namespace dev {

struct DevData {
  int p, q;          // FMM / QBX order
  int kp, kq;        // half-table sizes hsize(p), hsize(q)
  int ktab_m2l;      // hsize(2p): M2L offset table row length
  int dipole;        // 1 for Laplace SL+DL
  // tree (DFS-preorder boxes)
  const double4* box;  // (cx, cy, cz, |b|)
  const int* child_starts;
  const int* children;
  const int* parent;
  const int* src_own_start;
  const int* src_own_count;
  const int* ctr_own_start;
  const int* ctr_own_count;
  const int* tgt_own_start;
  const int* tgt_own_count;
  // box-sorted particles
  double4* src;        // (x, y, z, w)
  double4* mu;         // (mx, my, mz, 0) or null
  const double4* ctr;  // (x, y, z, r)
  const double4* tgt;  // conventional targets (x, y, z, 0)
  // expansions
  double2* M;   // nb x kp   box multipoles (box-scaled)
  double2* L;   // nb x kp   box locals (box-scaled)
  double2* Lc;  // nc x kq   QBX locals (radius-scaled), sorted centre order
  double* phi;  // nconv     near + W-far point potential (no 1/4pi)
  // lists (device CSR)
  const int64_t* near_starts;  // per box -> segments (src_start, src_count) of U u W_close u X_close
  const int2* near_seg;
  const int64_t* xfar_starts;  // per box -> segments of X_far
  const int2* xfar_seg;
  const int64_t* v_starts;     // per box -> (source box, offset index)
  const int2* v_ent;
  const int64_t* wfar_starts;  // per box -> source box
  const int* wfar_box;
  // operator tables
  const double2* m2l_tab;  // 1331 x ktab_m2l: I(2*delta) for box offsets delta in [-5,5]^3
  const double2* oct_m2m;  // 8 x kp: R((child-parent)/|child|)
  const double2* oct_l2l;  // 8 x kp: R((child-parent)/|parent|)
};

// launchers (return number of kernels launched)
int launch_gather(const DevData& D, int ns, const int* perm, const double* w, const double* mu, cudaStream_t s);
int launch_p2m(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_m2m(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_near_qbx(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_near_p2p(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_m2l(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_wfar(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_p2l(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_l2l(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_l2qbxl(const DevData& D, const int* boxes, int n, cudaStream_t s);
int launch_eval(const DevData& D, int nt, const double* tpos, const int* assoc, const int* ctr_sorted,
                int nconv, const int* tgt_perm, const int* tgt_box, double* pot, cudaStream_t s);
int launch_centre_out(const DevData& D, int nc, const int* ctr_perm, double* out, cudaStream_t s);
int launch_tables(const DevData& D, double2* m2l_tab, double2* oct_m2m, double2* oct_l2l, cudaStream_t s);
int launch_direct_sum(int ns, const double4* src, const double4* mu, int nt, const double4* tgt, double* pot,
                      unsigned long long* bad, cudaStream_t s);
void upload_constants();
void set_smem_limits();

}  // namespace dev
}  // namespace qbxg
