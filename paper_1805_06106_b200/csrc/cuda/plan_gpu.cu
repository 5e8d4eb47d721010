// Stage 1 on the GPU: the target-confinement octree of
// csrc/host/plan.cpp built on the
// device, bit-identical to the host build -- same boxes, same DFS numbering, same
// particle permutations -- so every list, operator and result downstream is
// unchanged.  (The host build is what BASELINE.json's north star names; this is
// the "host setup dominates once the apply is fast" follow-up.)
//
// Host algorithm: level by level, every box with more than n_max particles
// computes each particle's octant (a QBX centre whose ball does not fit the
// child's TCR stays, "suspended") and, if anything moves, stably partitions its
// range as [suspended | octant 0 | ... | octant 7] and creates the non-empty
// children.  Device formulation, one pass per level:
//   - k_dest: one thread per particle position finds its box among the level's
//     boxes (binary search on the range starts), computes the destination and
//     counts (box, destination) with integer atomics, and writes the sort key
//     (box start << 4 | digit), digit 0 = suspended, 1 + octant otherwise.
//     Positions outside splitting boxes get key (position << 4), so one stable
//     radix sort of the whole permutation performs every box's partition at
//     once and leaves everything else in place;
//   - k_split / scan / k_children: the split decision and the children, in the
//     host's creation order.
// DFS preorder: a box's particles are [own | child 0 | ... | child 7] and every
// box holds at least one particle, so preorder is the order of (range start,
// level) -- one radix sort.  Subtree ends are binary searches on range starts.
// Per-role arrays and ranges are three prefix sums over the final permutation.
//
// The only floating-point decision, the TCR fit test, is evaluated operation
// by operation (__dmul_rn / __dadd_rn / __dsqrt_rn) in the order plan.cpp
// writes it, and plan.cpp is compiled with -ffp-contract=off: bit-identical.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../host/plan.hpp"

namespace qbxg {
namespace {

#define PCK(call)                                                                                    \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      throw ::qbxg::CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call); \
  } while (0)

constexpr double kSqrt3 = 1.7320508075688772;  // std::sqrt(3.0), correctly rounded

struct DBox {
  double c[3];
  double h;
  long long ic[3];
  int level, parent;
  int start, end, own;
  int child[8];
};

// owned device allocations, freed on scope exit
struct Arena {
  std::vector<void*> p;
  template <class T>
  T* alloc(size_t n) {
    void* q = nullptr;
    PCK(cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)));
    p.push_back(q);
    return static_cast<T*>(q);
  }
  ~Arena() {
    for (void* q : p) cudaFree(q);
  }
};

// QBXG_PLAN_TIMING=1: per-phase wall times (device-synchronised) on stderr
struct PhaseClock {
  bool on = std::getenv("QBXG_PLAN_TIMING") != nullptr;
  double t = now_seconds();
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const double n = now_seconds();
    std::fprintf(stderr, "[plan_gpu] %-24s %8.2f ms\n", what, (n - t) * 1e3);
    t = n;
  }
};

int bits_for(long long v) {
  int b = 1;
  while ((1ll << b) <= v) ++b;
  return b;
}

// ---------------------------------------------------------------- kernels
__global__ void k_particles(long long ns, long long nc, long long nconv, const double* __restrict__ spos,
                            const double* __restrict__ cpos, const double* __restrict__ crad,
                            const double* __restrict__ tpos, const int* __restrict__ conv,
                            double4* __restrict__ P4, unsigned char* __restrict__ role, int* __restrict__ perm) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long np = ns + nc + nconv;
  if (k >= np) return;
  double4 v;
  unsigned char r;
  if (k < ns) {
    v = make_double4(spos[3 * k], spos[3 * k + 1], spos[3 * k + 2], 0.0);
    r = 0;
  } else if (k < ns + nc) {
    const long long i = k - ns;
    v = make_double4(cpos[3 * i], cpos[3 * i + 1], cpos[3 * i + 2], crad[i]);
    r = 1;
  } else {
    const long long i = conv[k - ns - nc];
    v = make_double4(tpos[3 * i], tpos[3 * i + 1], tpos[3 * i + 2], 0.0);
    r = 2;
  }
  P4[k] = v;
  role[k] = r;
  perm[k] = int(k);
}

// per-block (min(pos - rad), max(pos + rad)) per axis
__global__ void __launch_bounds__(256) k_bounds(long long np, const double4* __restrict__ P4,
                                               double* __restrict__ part) {
  __shared__ double s[6][8];
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < np; k += (long long)gridDim.x * blockDim.x) {
    const double4 v = P4[k];
    lo[0] = fmin(lo[0], v.x - v.w), hi[0] = fmax(hi[0], v.x + v.w);
    lo[1] = fmin(lo[1], v.y - v.w), hi[1] = fmax(hi[1], v.y + v.w);
    lo[2] = fmin(lo[2], v.z - v.w), hi[2] = fmax(hi[2], v.z + v.w);
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int d = 0; d < 3; ++d) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int d = 0; d < 3; ++d) s[d][w] = lo[d], s[3 + d][w] = hi[d];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 8; ++k)
      for (int d = 0; d < 3; ++d) lo[d] = fmin(lo[d], s[d][k]), hi[d] = fmax(hi[d], s[3 + d][k]);
    for (int d = 0; d < 3; ++d) part[6 * blockIdx.x + d] = lo[d], part[6 * blockIdx.x + 3 + d] = hi[d];
  }
}

__device__ __forceinline__ bool fits_tcr(double4 x, double cx, double cy, double cz, double hc, double tf) {
  const double dx = x.x - cx, dy = x.y - cy, dz = x.z - cz;
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return __dadd_rn(__dsqrt_rn(d2), x.w) <= __dmul_rn(__dmul_rn(kSqrt3, hc), __dadd_rn(1.0, tf));
}

__global__ void k_dest(long long np, const int* __restrict__ perm, const double4* __restrict__ P4,
                       const unsigned char* __restrict__ role, const DBox* __restrict__ box, int lo, int ncur,
                       int n_max, double tf, int* __restrict__ cnt, unsigned long long* __restrict__ key) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= np) return;
  // last level box with start <= i (starts ascend with the box index within a level)
  int a = 0, b = ncur - 1, q = -1;
  while (a <= b) {
    const int m = (a + b) >> 1;
    if (box[lo + m].start <= i) q = m, a = m + 1;
    else b = m - 1;
  }
  unsigned long long k = (unsigned long long)i << 4;
  if (q >= 0) {
    const DBox& B = box[lo + q];
    if (i < B.end && B.end - B.start > n_max) {
      const int p = perm[i];
      const double4 x = P4[p];
      int o = (x.x >= B.c[0] ? 1 : 0) | (x.y >= B.c[1] ? 2 : 0) | (x.z >= B.c[2] ? 4 : 0);
      if (role[p] == 1) {
        const double hc = 0.5 * B.h;
        const double cx = B.c[0] + ((o & 1) ? hc : -hc), cy = B.c[1] + ((o & 2) ? hc : -hc),
                     cz = B.c[2] + ((o & 4) ? hc : -hc);
        if (!fits_tcr(x, cx, cy, cz, hc, tf)) o = 8;
      }
      atomicAdd(&cnt[9 * q + o], 1);
      k = ((unsigned long long)B.start << 4) | (unsigned long long)(o == 8 ? 0 : o + 1);
    }
  }
  key[i] = k;
}

__global__ void k_split(int lo, int ncur, int n_max, DBox* __restrict__ box, const int* __restrict__ cnt,
                        int* __restrict__ nchild, int* __restrict__ depth_flag) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ncur) return;
  DBox& B = box[lo + q];
  const int n = B.end - B.start;
  int nc = 0;
  if (n > n_max && n - cnt[9 * q + 8] > 0) {
    if (B.level + 1 > kMaxDepth) {
      atomicExch(depth_flag, 1);
    } else {
      B.own = cnt[9 * q + 8];
      for (int o = 0; o < 8; ++o) nc += cnt[9 * q + o] > 0;
    }
  }
  nchild[q] = nc;
}

__global__ void k_children(int lo, int ncur, int nb, DBox* __restrict__ box, const int* __restrict__ cnt,
                           const int* __restrict__ nchild, const int* __restrict__ coff) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ncur || nchild[q] == 0) return;
  DBox& B = box[lo + q];
  const double hc = 0.5 * B.h;
  int s = B.start + cnt[9 * q + 8], id = nb + coff[q];
  for (int o = 0; o < 8; ++o) {
    const int c = cnt[9 * q + o];
    if (c == 0) continue;
    DBox C;
    C.c[0] = B.c[0] + ((o & 1) ? hc : -hc);
    C.c[1] = B.c[1] + ((o & 2) ? hc : -hc);
    C.c[2] = B.c[2] + ((o & 4) ? hc : -hc);
    C.h = hc;
    C.level = B.level + 1;
    C.parent = lo + q;
    for (int d = 0; d < 3; ++d) C.ic[d] = 2 * B.ic[d] + ((o >> d) & 1);
    C.start = s;
    C.end = s + c;
    C.own = c;
    for (int k = 0; k < 8; ++k) C.child[k] = -1;
    s += c;
    B.child[o] = id;
    box[id++] = C;
  }
}

__global__ void k_dfs_keys(int nb, int lev_bits, const DBox* __restrict__ box, unsigned long long* __restrict__ key,
                           int* __restrict__ val) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  key[b] = ((unsigned long long)box[b].start << lev_bits) | (unsigned long long)box[b].level;
  val[b] = b;
}

__global__ void k_newid(int nb, const int* __restrict__ order, int* __restrict__ newid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) newid[order[i]] = i;
}

__global__ void k_emit(int nb, const DBox* __restrict__ box, const int* __restrict__ order,
                       const int* __restrict__ newid, double* __restrict__ center, double* __restrict__ h,
                       int* __restrict__ level, int* __restrict__ parent, long long* __restrict__ ic,
                       int* __restrict__ bstart, int* __restrict__ bend, int* __restrict__ bown,
                       int* __restrict__ nchild) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const DBox& B = box[order[i]];
  for (int d = 0; d < 3; ++d) center[3 * i + d] = B.c[d], ic[3 * i + d] = B.ic[d];
  h[i] = B.h;
  level[i] = B.level;
  parent[i] = B.parent >= 0 ? newid[B.parent] : -1;
  bstart[i] = B.start;
  bend[i] = B.end;
  bown[i] = B.own;
  int n = 0;
  for (int o = 0; o < 8; ++o) n += B.child[o] >= 0;
  nchild[i] = n;
}

__global__ void k_emit_children(int nb, const DBox* __restrict__ box, const int* __restrict__ order,
                                const int* __restrict__ newid, const int* __restrict__ cstart,
                                int* __restrict__ children, const int* __restrict__ bstart,
                                const int* __restrict__ bend, int* __restrict__ sub_end) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const DBox& B = box[order[i]];
  int k = cstart[i];
  for (int o = 0; o < 8; ++o)
    if (B.child[o] >= 0) children[k++] = newid[B.child[o]];
  // first box (in preorder) whose range starts at or after this box's end
  const int e = bend[i];
  int a = i + 1, z = nb;
  while (a < z) {
    const int m = (a + z) >> 1;
    if (bstart[m] >= e) z = m;
    else a = m + 1;
  }
  sub_end[i] = a;
}

__global__ void k_role_flags(long long np, const int* __restrict__ perm, const unsigned char* __restrict__ role,
                             int* __restrict__ fs, int* __restrict__ fc, int* __restrict__ ft) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > np) return;
  const int r = i < np ? role[perm[i]] : 3;
  fs[i] = r == 0;
  fc[i] = r == 1;
  ft[i] = r == 2;
}

__global__ void k_role_perms(long long np, long long ns, long long nc, const int* __restrict__ perm,
                             const unsigned char* __restrict__ role, const int* __restrict__ conv,
                             const int* __restrict__ cs, const int* __restrict__ cc, const int* __restrict__ ct,
                             int* __restrict__ sp, int* __restrict__ cp, int* __restrict__ tp) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= np) return;
  const int k = perm[i];
  const int r = role[k];
  if (r == 0) sp[cs[i]] = k;
  else if (r == 1) cp[cc[i]] = int(k - ns);
  else tp[ct[i]] = conv[k - ns - nc];
}

struct RoleOut {
  int *os, *oc, *ss, *sc;
};

__global__ void k_box_roles(int nb, const int* __restrict__ bstart, const int* __restrict__ bend,
                            const int* __restrict__ bown, const int* __restrict__ cs, const int* __restrict__ cc,
                            const int* __restrict__ ct, RoleOut S, RoleOut C, RoleOut T,
                            const int* __restrict__ nchild, unsigned char* __restrict__ flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int s0 = bstart[b], s1 = bstart[b] + bown[b], s2 = bend[b];
  const int* pre[3] = {cs, cc, ct};
  RoleOut* out[3] = {&S, &C, &T};
  int own[3], sub[3];
  for (int r = 0; r < 3; ++r) {
    const int* p = pre[r];
    out[r]->os[b] = p[s0];
    out[r]->oc[b] = own[r] = p[s1] - p[s0];
    out[r]->ss[b] = p[s0];
    out[r]->sc[b] = sub[r] = p[s2] - p[s0];
  }
  unsigned char f = 0;
  if (own[1] + own[2] > 0) f |= QBXG_BOX_TARGET;
  if (sub[1] + sub[2] > own[1] + own[2]) f |= QBXG_BOX_TARGET_ANCESTOR;
  if (sub[0] > 0) f |= QBXG_BOX_HAS_SOURCES;
  if (nchild[b] == 0) f |= QBXG_BOX_LEAF;
  flags[b] = f;
}

template <class T>
void to_host(std::vector<T>& v, const T* d, size_t n) {
  v.resize(n);
  if (n) PCK(cudaMemcpy(v.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

template <class T>
T* upload(Arena& A, const T* h, size_t n) {
  T* d = A.alloc<T>(n);
  if (n) PCK(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

// exclusive prefix sum of n ints (in may equal out)
void exclusive_sum(Arena& A, const int* in, int* out, long long n) {
  size_t tb = 0;
  PCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n));
  void* t = A.alloc<char>(tb);
  PCK(cub::DeviceScan::ExclusiveSum(t, tb, in, out, n));
}

template <class K, class V>
void sort_pairs(Arena& A, const K* kin, K* kout, const V* vin, V* vout, long long n, int end_bit) {
  size_t tb = 0;
  PCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit));
  void* t = A.alloc<char>(tb);
  PCK(cub::DeviceRadixSort::SortPairs(t, tb, kin, kout, vin, vout, n, 0, end_bit));
}

}  // namespace

void build_tree_gpu(Plan& P, const qbxg_geometry& g) {
  const double t0 = now_seconds();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device available (the GPU plan builder has no CPU fallback)");
  }
  const qbxg_config& cfg = P.cfg;
  P.ns = g.n_sources;
  P.nc = g.n_centers;
  P.ntgt = g.n_targets;
  std::vector<int32_t> conv;
  for (int64_t t = 0; t < g.n_targets; ++t)
    if (g.association[t] < 0) conv.push_back(int32_t(t));
  P.nconv = int64_t(conv.size());
  const long long np = P.ns + P.nc + P.nconv;
  if (np == 0) throw InvalidArgument("plan_create_device: no particles");
  Arena A;
  PhaseClock clk;
  const double* dsp = upload(A, g.source_pos, 3 * size_t(P.ns));
  const double* dcp = upload(A, g.center_pos, 3 * size_t(P.nc));
  const double* dcr = upload(A, g.center_radius, size_t(P.nc));
  const double* dtp = upload(A, g.target_pos, 3 * size_t(g.n_targets));
  const int* dconv = upload(A, conv.data(), conv.size());
  double4* P4 = A.alloc<double4>(np);
  unsigned char* role = A.alloc<unsigned char>(np);
  int* perm = A.alloc<int>(np);
  int* perm2 = A.alloc<int>(np);
  const int tb = 256;
  const unsigned gp = unsigned((np + tb - 1) / tb);
  k_particles<<<gp, tb>>>(P.ns, P.nc, P.nconv, dsp, dcp, dcr, dtp, dconv, P4, role, perm);
  PCK(cudaGetLastError());

  // root cube (plan.cpp): bounds of every particle and expansion ball
  const int nbk = int(std::min<long long>(1024, (np + tb - 1) / tb));
  double* part = A.alloc<double>(6 * size_t(nbk));
  k_bounds<<<nbk, tb>>>(np, P4, part);
  std::vector<double> hp;
  to_host(hp, part, 6 * size_t(nbk));
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int k = 0; k < nbk; ++k)
    for (int d = 0; d < 3; ++d) lo[d] = std::min(lo[d], hp[6 * k + d]), hi[d] = std::max(hi[d], hp[6 * k + 3 + d]);
  double hroot = 0;
  for (int d = 0; d < 3; ++d) {
    P.root_c[d] = 0.5 * (lo[d] + hi[d]);
    hroot = std::max(hroot, 0.5 * (hi[d] - lo[d]));
  }
  if (!(hroot > 0)) hroot = 1.0;
  hroot *= 1.0 + 1.0 / 1024.0;
  P.root_h = hroot;
  clk.mark("upload + root");

  // box table (creation order), grown on demand
  size_t cap = std::max<size_t>(1024, size_t(4 * np / std::max(1, cfg.n_max)) + 64);
  DBox* box = A.alloc<DBox>(cap);
  {
    DBox R{};
    for (int d = 0; d < 3; ++d) R.c[d] = P.root_c[d], R.ic[d] = 0;
    R.h = hroot;
    R.level = 0;
    R.parent = -1;
    R.start = 0;
    R.end = int(np);
    R.own = int(np);
    for (int k = 0; k < 8; ++k) R.child[k] = -1;
    PCK(cudaMemcpy(box, &R, sizeof(R), cudaMemcpyHostToDevice));
  }
  unsigned long long* key = A.alloc<unsigned long long>(np);
  unsigned long long* key2 = A.alloc<unsigned long long>(np);
  int* dflag = A.alloc<int>(1);
  PCK(cudaMemset(dflag, 0, sizeof(int)));
  const int kbits = bits_for(np) + 4;
  int nb = 1, lo_b = 0, ncur = 1;
  Arena L;  // per-level scratch sized for the widest level
  int* cnt = nullptr;
  int* nch = nullptr;
  int* coff = nullptr;
  int lvl_cap = 0;
  void* sort_tmp = nullptr;
  size_t sort_tb = 0;
  PCK(cub::DeviceRadixSort::SortPairs(nullptr, sort_tb, key, key2, perm, perm2, np, 0, kbits));
  sort_tmp = A.alloc<char>(sort_tb);
  while (ncur > 0) {
    if (ncur > lvl_cap) {
      lvl_cap = std::max(ncur, 2 * lvl_cap);
      cnt = L.alloc<int>(9 * size_t(lvl_cap));
      nch = L.alloc<int>(size_t(lvl_cap) + 1);
      coff = L.alloc<int>(size_t(lvl_cap) + 1);
    }
    PCK(cudaMemsetAsync(cnt, 0, 9 * sizeof(int) * size_t(ncur)));
    k_dest<<<gp, tb>>>(np, perm, P4, role, box, lo_b, ncur, cfg.n_max, cfg.t_f, cnt, key);
    k_split<<<(ncur + tb - 1) / tb, tb>>>(lo_b, ncur, cfg.n_max, box, cnt, nch, dflag);
    PCK(cudaMemsetAsync(nch + ncur, 0, sizeof(int)));
    exclusive_sum(L, nch, coff, ncur + 1);
    int tot = 0, flag = 0;
    PCK(cudaMemcpy(&tot, coff + ncur, sizeof(int), cudaMemcpyDeviceToHost));
    PCK(cudaMemcpy(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) throw InvalidArgument("build_tree: depth cap exceeded (SPEC.md:347)");
    if (tot == 0) break;
    if (size_t(nb) + size_t(tot) > cap) {
      const size_t ncap = std::max(cap * 2, size_t(nb) + size_t(tot));
      DBox* nbx = A.alloc<DBox>(ncap);
      PCK(cudaMemcpy(nbx, box, sizeof(DBox) * size_t(nb), cudaMemcpyDeviceToDevice));
      box = nbx;  // the old table is released with the arena
      cap = ncap;
    }
    k_children<<<(ncur + tb - 1) / tb, tb>>>(lo_b, ncur, nb, box, cnt, nch, coff);
    PCK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_tb, key, key2, perm, perm2, np, 0, kbits));
    std::swap(perm, perm2);
    lo_b = nb;
    nb += tot;
    ncur = tot;
  }
  PCK(cudaGetLastError());
  clk.mark("levels");

  // DFS preorder = order of (range start, level)
  const int lev_bits = 6;
  unsigned long long* bk = A.alloc<unsigned long long>(nb);
  unsigned long long* bk2 = A.alloc<unsigned long long>(nb);
  int* bv = A.alloc<int>(nb);
  int* order = A.alloc<int>(nb);
  int* newid = A.alloc<int>(nb);
  const unsigned gb = unsigned((nb + tb - 1) / tb);
  k_dfs_keys<<<gb, tb>>>(nb, lev_bits, box, bk, bv);
  sort_pairs(A, bk, bk2, bv, order, nb, bits_for(np) + lev_bits);
  k_newid<<<gb, tb>>>(nb, order, newid);
  double* dcen = A.alloc<double>(3 * size_t(nb));
  double* dh = A.alloc<double>(nb);
  int* dlev = A.alloc<int>(nb);
  int* dpar = A.alloc<int>(nb);
  long long* dic = A.alloc<long long>(3 * size_t(nb));
  int* bstart = A.alloc<int>(nb);
  int* bend = A.alloc<int>(nb);
  int* bown = A.alloc<int>(nb);
  int* nchild = A.alloc<int>(size_t(nb) + 1);
  int* cstart = A.alloc<int>(size_t(nb) + 1);
  k_emit<<<gb, tb>>>(nb, box, order, newid, dcen, dh, dlev, dpar, dic, bstart, bend, bown, nchild);
  PCK(cudaMemset(nchild + nb, 0, sizeof(int)));
  exclusive_sum(A, nchild, cstart, nb + 1);
  int nkids = 0;
  PCK(cudaMemcpy(&nkids, cstart + nb, sizeof(int), cudaMemcpyDeviceToHost));
  int* kids = A.alloc<int>(nkids);
  int* sub_end = A.alloc<int>(nb);
  k_emit_children<<<gb, tb>>>(nb, box, order, newid, cstart, kids, bstart, bend, sub_end);

  // per-role permutations and ranges
  int* gs = A.alloc<int>(np + 1);
  int* gc = A.alloc<int>(np + 1);
  int* gt = A.alloc<int>(np + 1);
  int* fs = A.alloc<int>(np + 1);
  int* fc = A.alloc<int>(np + 1);
  int* ft = A.alloc<int>(np + 1);
  const unsigned gp1 = unsigned((np + 1 + tb - 1) / tb);
  k_role_flags<<<gp1, tb>>>(np, perm, role, gs, gc, gt);
  exclusive_sum(A, gs, fs, np + 1);
  exclusive_sum(A, gc, fc, np + 1);
  exclusive_sum(A, gt, ft, np + 1);
  int* sp = A.alloc<int>(P.ns);
  int* cp = A.alloc<int>(P.nc);
  int* tp = A.alloc<int>(P.nconv);
  k_role_perms<<<gp, tb>>>(np, P.ns, P.nc, perm, role, dconv, fs, fc, ft, sp, cp, tp);
  RoleOut R[3];
  for (auto& r : R) r = RoleOut{A.alloc<int>(nb), A.alloc<int>(nb), A.alloc<int>(nb), A.alloc<int>(nb)};
  unsigned char* dflags = A.alloc<unsigned char>(nb);
  k_box_roles<<<gb, tb>>>(nb, bstart, bend, bown, fs, fc, ft, R[0], R[1], R[2], nchild, dflags);
  PCK(cudaGetLastError());

  clk.mark("dfs + roles");
  // download into the host plan
  P.nb = nb;
  to_host(P.center, dcen, 3 * size_t(nb));
  to_host(P.h, dh, nb);
  to_host(P.level, dlev, nb);
  to_host(P.parent, dpar, nb);
  std::vector<long long> icll;
  to_host(icll, dic, 3 * size_t(nb));
  P.ic.assign(icll.begin(), icll.end());
  to_host(P.child_starts, cstart, size_t(nb) + 1);
  to_host(P.children, kids, nkids);
  to_host(P.subtree_end, sub_end, nb);
  to_host(P.src_perm, sp, P.ns);
  to_host(P.ctr_perm, cp, P.nc);
  to_host(P.tgt_perm, tp, P.nconv);
  std::vector<int32_t>* dst[3][4] = {{&P.src_own_start, &P.src_own_count, &P.src_sub_start, &P.src_sub_count},
                                     {&P.ctr_own_start, &P.ctr_own_count, &P.ctr_sub_start, &P.ctr_sub_count},
                                     {&P.tgt_own_start, &P.tgt_own_count, &P.tgt_sub_start, &P.tgt_sub_count}};
  for (int r = 0; r < 3; ++r) {
    to_host(*dst[r][0], R[r].os, nb);
    to_host(*dst[r][1], R[r].oc, nb);
    to_host(*dst[r][2], R[r].ss, nb);
    to_host(*dst[r][3], R[r].sc, nb);
  }
  to_host(P.flags, dflags, nb);
  int maxlev = 0;
  for (int32_t l : P.level) maxlev = std::max(maxlev, int(l));
  P.nlev = maxlev + 1;
  P.level_starts.assign(P.nlev + 1, 0);
  for (int32_t b = 0; b < nb; ++b) P.level_starts[P.level[b] + 1]++;
  for (int l = 0; l < P.nlev; ++l) P.level_starts[l + 1] += P.level_starts[l];
  P.level_boxes.resize(nb);
  {
    std::vector<int32_t> fill(P.level_starts.begin(), P.level_starts.end() - 1);
    for (int32_t b = 0; b < nb; ++b) P.level_boxes[fill[P.level[b]]++] = b;
  }
  clk.mark("download");
  P.t_tree = now_seconds() - t0;
}

}  // namespace qbxg

// ============================================================================
// Interaction lists on the GPU (Definitions 1-8; plan.cpp
// build_lists): the same rows, sorted by box id, hence the same CSR arrays and
// hashes.  One thread per box; the host's explicit-stack descents become
// stackless preorder walks (descend = b + 1, prune = b = sub_end[b]), which
// visit the same boxes in a different order -- rows are sorted at the end
// (segmented sort), so order is immaterial.  Two passes (count, fill) per list.
// Colleague rows and the List-2 rows come out sorted by construction (children
// of sorted colleagues in DFS order).  List 4 is top-down by level because a
// box inherits its parent's List-4-close candidates.
// ============================================================================
namespace qbxg {
namespace {

constexpr int kColl = 125;  // 2-colleagues: at most 5^3

struct DTree {
  int nb;
  const double* center;
  const double* h;
  const int* level;
  const int* parent;
  const long long* ic;
  const int* cstart;
  const int* kids;
  const int* sub_end;
  const int* src_own;
  const int* src_sub;
  const unsigned char* flags;
  const int* coll;
  const int* ncoll;
};

__device__ __forceinline__ bool t_leaf(const DTree& T, int b) { return T.cstart[b + 1] == T.cstart[b]; }
__device__ __forceinline__ bool t_src(const DTree& T, int b) { return T.src_sub[b] > 0; }
__device__ __forceinline__ long long t_cheb(const DTree& T, int a, int b) {
  long long m = 0;
  for (int d = 0; d < 3; ++d) m = max(m, llabs(T.ic[3 * a + d] - T.ic[3 * b + d]));
  return m;
}
__device__ __forceinline__ bool t_adj(const DTree& T, int a, int b) {  // predicates.hpp boxes_adjacent
  const int la = T.level[a], lb = T.level[b], L = max(la, lb);
  for (int d = 0; d < 3; ++d) {
    const long long alo = T.ic[3 * a + d] << (L - la), ahi = (T.ic[3 * a + d] + 1) << (L - la);
    const long long blo = T.ic[3 * b + d] << (L - lb), bhi = (T.ic[3 * b + d] + 1) << (L - lb);
    if (alo > bhi || blo > ahi) return false;
  }
  return true;
}
// predicates.hpp sep_box_tcr(centre(a), |a|, centre(b), |b|): a < TCR(b)
__device__ __forceinline__ bool t_sep_box_tcr(const DTree& T, int a, int b, double tf) {
  const double dx = T.center[3 * a] - T.center[3 * b], dy = T.center[3 * a + 1] - T.center[3 * b + 1],
               dz = T.center[3 * a + 2] - T.center[3 * b + 2];
  const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  return __dsub_rn(d, __dmul_rn(__dmul_rn(kSqrt3, T.h[b]), __dadd_rn(1.0, tf))) >= __dmul_rn(3.0, T.h[a]);
}
// predicates.hpp sep_tcr_box(centre(a), |a|, centre(b), |b|): TCR(a) < b
__device__ __forceinline__ bool t_sep_tcr_box(const DTree& T, int a, int b, double tf) {
  const double dx = fabs(T.center[3 * a] - T.center[3 * b]), dy = fabs(T.center[3 * a + 1] - T.center[3 * b + 1]),
               dz = fabs(T.center[3 * a + 2] - T.center[3 * b + 2]);
  const double d = dx > dy ? (dx > dz ? dx : dz) : (dy > dz ? dy : dz);
  return __dsub_rn(d, T.h[b]) >= __dmul_rn(__dmul_rn(3.0, T.h[a]), __dadd_rn(1.0, tf));
}

__global__ void k_coll(DTree T, const int* __restrict__ lboxes, int n, int* __restrict__ coll,
                       int* __restrict__ ncoll) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = lboxes[i], p = T.parent[b];
  int c = 0;
  for (int j = 0; j < T.ncoll[p]; ++j) {
    const int pc = T.coll[kColl * p + j];
    for (int k = T.cstart[pc]; k < T.cstart[pc + 1]; ++k) {
      const int d = T.kids[k];
      if (t_cheb(T, d, b) <= 2) coll[kColl * size_t(b) + c++] = d;
    }
  }
  ncoll[b] = c;
}

enum { LU = 0, LV = 1, LWC = 2, LWF = 3 };

// Lists 1, 2, 3 close / far for every box: pass 0 counts into cnt[k][b], pass 1
// writes at start[k][b]
struct Rows {
  long long* cnt[4];
  const long long* start[4];
  int* out[4];
};

template <bool FILL>
__global__ void k_uvw(DTree T, double tf, int demote, Rows R) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= T.nb) return;
  long long n[4] = {0, 0, 0, 0};
  auto emit = [&](int k, int x) {
    if (FILL) R.out[k][R.start[k][b] + n[k]] = x;
    ++n[k];
  };
  const unsigned char f = T.flags[b];
  const bool tgt = f & QBXG_BOX_TARGET, tgt_anc = f & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR);
  if (tgt_anc && b != 0) {  // List 2: children of the parent's colleagues, well separated, with sources
    const int p = T.parent[b];
    for (int j = 0; j < T.ncoll[p]; ++j) {
      const int pc = T.coll[kColl * p + j];
      for (int k = T.cstart[pc]; k < T.cstart[pc + 1]; ++k) {
        const int d = T.kids[k];
        if (t_src(T, d) && t_cheb(T, d, b) > 2) emit(LV, d);
      }
    }
  }
  if (tgt) {
    // List 1 (Definition 1): source leaves of the subtree ...
    for (int d = b; d < T.sub_end[b];) {
      if (!t_src(T, d)) {
        d = T.sub_end[d];
        continue;
      }
      if (t_leaf(T, d) && T.src_own[d] > 0) emit(LU, d);
      ++d;
    }
    const int* cb = T.coll + kColl * size_t(b);
    const int ncb = T.ncoll[b];
    // ... source leaves adjacent to b below its adjacent colleagues ...
    for (int j = 0; j < ncb; ++j) {
      const int e = cb[j];
      if (e == b || t_cheb(T, e, b) > 1) continue;
      for (int x = e; x < T.sub_end[e];) {
        if (!t_src(T, x) || !t_adj(T, x, b)) {
          x = T.sub_end[x];
        } else {
          if (t_leaf(T, x)) emit(LU, x);
          ++x;
        }
      }
    }
    // ... and coarser source leaves adjacent to b among the ancestors' near colleagues
    for (int a = T.parent[b]; a >= 0; a = T.parent[a])
      for (int j = 0; j < T.ncoll[a]; ++j) {
        const int e = T.coll[kColl * size_t(a) + j];
        if (e != a && t_cheb(T, e, a) <= 1 && t_leaf(T, e) && T.src_own[e] > 0 && t_adj(T, e, b)) emit(LU, e);
      }
    // List 3 (Definition 3), split close / far (Definitions 5, 6; Remark 1 demotion)
    for (int j = 0; j < ncb; ++j) {
      const int e = cb[j];
      if (e == b || t_leaf(T, e)) continue;
      for (int d = e + 1; d < T.sub_end[e];) {
        if (!t_src(T, d)) {
          d = T.sub_end[d];
          continue;
        }
        if (t_adj(T, d, b)) {
          ++d;  // adjacent: descend (a leaf's subtree is itself)
          continue;
        }
        for (int y = d; y < T.sub_end[d];) {  // d is in List 3: classify its subtree
          if (!t_src(T, y)) {
            y = T.sub_end[y];
          } else if (t_sep_box_tcr(T, y, b, tf)) {
            if (demote > 0 && T.src_sub[y] < demote) {
              for (int x = y; x < T.sub_end[y]; ++x)
                if (t_leaf(T, x) && T.src_own[x] > 0) emit(LWC, x);
            } else {
              emit(LWF, y);
            }
            y = T.sub_end[y];
          } else {
            if (t_leaf(T, y)) emit(LWC, y);
            ++y;
          }
        }
        d = T.sub_end[d];
      }
    }
  }
  if (!FILL)
    for (int k = 0; k < 4; ++k) R.cnt[k][b] = n[k];
}

// List 4 (Definition 4) close / far (Definitions 7, 8) for the boxes of one level;
// the parent's close row is read from (xc_off, xc_len) in the pool
template <bool FILL>
__global__ void k_x(DTree T, double tf, const int* __restrict__ lboxes, int n, long long* __restrict__ cxc,
                    long long* __restrict__ cxf, const long long* __restrict__ oxc, const long long* __restrict__ oxf,
                    long long* __restrict__ xc_off, int* __restrict__ xc_len, long long* __restrict__ xf_off,
                    int* __restrict__ xf_len, int* __restrict__ pool) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = lboxes[i];
  long long nc = 0, nf = 0;
  auto put = [&](int d) {
    if (t_sep_tcr_box(T, b, d, tf)) {
      if (FILL) pool[oxf[i] + nf] = d;
      ++nf;
    } else {
      if (FILL) pool[oxc[i] + nc] = d;
      ++nc;
    }
  };
  if (T.flags[b] & (QBXG_BOX_TARGET | QBXG_BOX_TARGET_ANCESTOR)) {
    for (int j = 0; j < T.ncoll[b]; ++j) {
      const int c = T.coll[kColl * size_t(b) + j];
      if (c != b && t_leaf(T, c) && T.src_own[c] > 0 && !t_adj(T, c, b)) put(c);
    }
    const int par = T.parent[b];
    if (par >= 0) {
      for (int anc = par; anc >= 0; anc = T.parent[anc])
        for (int j = 0; j < T.ncoll[anc]; ++j) {
          const int c = T.coll[kColl * size_t(anc) + j];
          if (t_leaf(T, c) && T.src_own[c] > 0 && t_adj(T, c, par) && !t_adj(T, c, b)) put(c);
        }
      for (int j = 0; j < xc_len[par]; ++j) put(pool[xc_off[par] + j]);
    }
  }
  if (FILL) {
    xc_off[b] = oxc[i];
    xc_len[b] = int(nc);
    xf_off[b] = oxf[i];
    xf_len[b] = int(nf);
  } else {
    cxc[i] = nc;
    cxf[i] = nf;
  }
}

__global__ void k_gather(int nb, const long long* __restrict__ off, const int* __restrict__ len,
                         const long long* __restrict__ start, const int* __restrict__ pool, int* __restrict__ out) {
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < len[b]; j += blockDim.x) out[start[b] + j] = pool[off[b] + j];
}

__global__ void k_len64(int nb, const int* __restrict__ len, long long* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b <= nb) out[b] = b < nb ? len[b] : 0;
}

void exclusive_sum64(Arena& A, const long long* in, long long* out, long long n) {
  size_t tb = 0;
  PCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n));
  void* t = A.alloc<char>(tb);
  PCK(cub::DeviceScan::ExclusiveSum(t, tb, in, out, n));
}

// sort each row of a CSR list in place (rows begin at start[b], end at start[b+1])
void sort_rows(Arena& A, int* keys, long long total, int nb, const long long* start) {
  if (total == 0) return;
  int* tmp = A.alloc<int>(total);
  size_t tb = 0;
  PCK(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys, tmp, total, nb, start, start + 1));
  void* t = A.alloc<char>(tb);
  PCK(cub::DeviceSegmentedSort::SortKeys(t, tb, keys, tmp, total, nb, start, start + 1));
  PCK(cudaMemcpy(keys, tmp, sizeof(int) * size_t(total), cudaMemcpyDeviceToDevice));
}

__global__ void k_add(long long* __restrict__ v, int n, long long c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] += c;
}

void add_offset(long long* v, int n, long long c) {
  if (c != 0 && n > 0) k_add<<<(n + 255) / 256, 256>>>(v, n, c);
}

template <class T>
T* up(Arena& A, const std::vector<T>& v) {
  return upload(A, v.data(), v.size());
}

}  // namespace

void build_lists_gpu(Plan& P) {
  const double t0 = now_seconds();
  const int nb = P.nb;
  const double tf = P.cfg.t_f;
  const int demote = P.cfg.w_far_demote;
  Arena A;
  PhaseClock clk;
  std::vector<long long> icll(P.ic.begin(), P.ic.end());
  DTree T{};
  T.nb = nb;
  T.center = up(A, P.center);
  T.h = up(A, P.h);
  T.level = up(A, P.level);
  T.parent = up(A, P.parent);
  T.ic = up(A, icll);
  T.cstart = up(A, P.child_starts);
  T.kids = up(A, P.children);
  T.sub_end = up(A, P.subtree_end);
  T.src_own = up(A, P.src_own_count);
  T.src_sub = up(A, P.src_sub_count);
  T.flags = up(A, P.flags);
  int* coll = A.alloc<int>(size_t(kColl) * nb);
  int* ncoll = A.alloc<int>(nb);
  T.coll = coll;
  T.ncoll = ncoll;
  const int* lboxes = up(A, P.level_boxes);
  const int tb = 128;
  // 2-colleagues, level by level (root: itself)
  {
    const int zero = 0, one = 1;
    PCK(cudaMemcpy(coll, &zero, sizeof(int), cudaMemcpyHostToDevice));
    PCK(cudaMemcpy(ncoll, &one, sizeof(int), cudaMemcpyHostToDevice));
    for (int l = 1; l < P.nlev; ++l) {
      const int a = P.level_starts[l], n = P.level_starts[l + 1] - a;
      if (n) k_coll<<<(n + tb - 1) / tb, tb>>>(T, lboxes + a, n, coll, ncoll);
    }
  }
  clk.mark("upload + colleagues");
  // Lists 1, 2, 3
  Rows R{};
  long long* st[4];
  for (int k = 0; k < 4; ++k) {
    R.cnt[k] = A.alloc<long long>(size_t(nb) + 1);
    st[k] = A.alloc<long long>(size_t(nb) + 1);
    R.start[k] = st[k];
    PCK(cudaMemset(R.cnt[k] + nb, 0, sizeof(long long)));
  }
  const unsigned gb = unsigned((nb + tb - 1) / tb);
  k_uvw<false><<<gb, tb>>>(T, tf, demote, R);
  PCK(cudaGetLastError());
  long long tot[4];
  for (int k = 0; k < 4; ++k) {
    exclusive_sum64(A, R.cnt[k], st[k], nb + 1);
    PCK(cudaMemcpy(&tot[k], st[k] + nb, sizeof(long long), cudaMemcpyDeviceToHost));
    R.out[k] = A.alloc<int>(size_t(tot[k]));
  }
  k_uvw<true><<<gb, tb>>>(T, tf, demote, R);
  PCK(cudaGetLastError());
  sort_rows(A, R.out[LU], tot[LU], nb, st[LU]);  // List 2 rows are sorted by construction
  sort_rows(A, R.out[LWC], tot[LWC], nb, st[LWC]);
  sort_rows(A, R.out[LWF], tot[LWF], nb, st[LWF]);
  clk.mark("lists 1-3");

  // List 4, top-down by level; rows live in a growing pool until the final gather
  long long* xc_off = A.alloc<long long>(nb);
  long long* xf_off = A.alloc<long long>(nb);
  int* xc_len = A.alloc<int>(nb);
  int* xf_len = A.alloc<int>(nb);
  PCK(cudaMemset(xc_len, 0, sizeof(int) * size_t(nb)));
  PCK(cudaMemset(xf_len, 0, sizeof(int) * size_t(nb)));
  int maxw = 0;
  for (int l = 0; l < P.nlev; ++l) maxw = std::max(maxw, P.level_starts[l + 1] - P.level_starts[l]);
  long long* cxc = A.alloc<long long>(size_t(maxw) + 1);
  long long* cxf = A.alloc<long long>(size_t(maxw) + 1);
  long long* oxc = A.alloc<long long>(size_t(maxw) + 1);
  long long* oxf = A.alloc<long long>(size_t(maxw) + 1);
  size_t pool_cap = std::max<size_t>(1 << 20, size_t(nb) * 16);
  int* pool = A.alloc<int>(pool_cap);
  long long pool_used = 0;
  for (int l = 0; l < P.nlev; ++l) {
    const int a = P.level_starts[l], n = P.level_starts[l + 1] - a;
    if (n == 0) continue;
    const unsigned g = unsigned((n + tb - 1) / tb);
    k_x<false><<<g, tb>>>(T, tf, lboxes + a, n, cxc, cxf, nullptr, nullptr, xc_off, xc_len, xf_off, xf_len, pool);
    PCK(cudaMemset(cxc + n, 0, sizeof(long long)));
    PCK(cudaMemset(cxf + n, 0, sizeof(long long)));
    exclusive_sum64(A, cxc, oxc, n + 1);
    exclusive_sum64(A, cxf, oxf, n + 1);
    long long nc = 0, nf = 0;
    PCK(cudaMemcpy(&nc, oxc + n, sizeof(long long), cudaMemcpyDeviceToHost));
    PCK(cudaMemcpy(&nf, oxf + n, sizeof(long long), cudaMemcpyDeviceToHost));
    if (size_t(pool_used + nc + nf) > pool_cap) {
      const size_t ncap = std::max(2 * pool_cap, size_t(pool_used + nc + nf));
      int* np2 = A.alloc<int>(ncap);
      PCK(cudaMemcpy(np2, pool, sizeof(int) * size_t(pool_used), cudaMemcpyDeviceToDevice));
      pool = np2;
      pool_cap = ncap;
    }
    // close rows at [pool_used, +nc), far rows after them
    add_offset(oxc, n, pool_used);
    add_offset(oxf, n, pool_used + nc);
    k_x<true><<<g, tb>>>(T, tf, lboxes + a, n, nullptr, nullptr, oxc, oxf, xc_off, xc_len, xf_off, xf_len, pool);
    PCK(cudaGetLastError());
    pool_used += nc + nf;
  }
  long long* xst[2];
  int* xout[2];
  long long xtot[2];
  {
    const long long* offs[2] = {xc_off, xf_off};
    const int* lens[2] = {xc_len, xf_len};
    for (int k = 0; k < 2; ++k) {
      long long* l64 = A.alloc<long long>(size_t(nb) + 1);
      k_len64<<<(nb + 1 + tb - 1) / tb, tb>>>(nb, lens[k], l64);
      xst[k] = A.alloc<long long>(size_t(nb) + 1);
      exclusive_sum64(A, l64, xst[k], nb + 1);
      PCK(cudaMemcpy(&xtot[k], xst[k] + nb, sizeof(long long), cudaMemcpyDeviceToHost));
      xout[k] = A.alloc<int>(size_t(xtot[k]));
      k_gather<<<nb, 64>>>(nb, offs[k], lens[k], xst[k], pool, xout[k]);
      sort_rows(A, xout[k], xtot[k], nb, xst[k]);
    }
  }
  PCK(cudaGetLastError());
  clk.mark("list 4");

  // download in the host layout and hash
  const int map[QBXG_NUM_LISTS] = {LU, LV, LWC, LWF, -1, -2};
  for (int k = 0; k < QBXG_NUM_LISTS; ++k) {
    const long long* s = map[k] >= 0 ? st[map[k]] : xst[-1 - map[k]];
    const int* o = map[k] >= 0 ? R.out[map[k]] : xout[-1 - map[k]];
    const long long t = map[k] >= 0 ? tot[map[k]] : xtot[-1 - map[k]];
    std::vector<long long> s64;
    to_host(s64, s, size_t(nb) + 1);
    P.lst_starts[k].assign(s64.begin(), s64.end());
    to_host(P.lst[k], o, size_t(t));
  }
  clk.mark("download");
  hash_lists(P);
  clk.mark("hash");
  P.t_lists = now_seconds() - t0;
}

}  // namespace qbxg
