// Target association (Algorithm 3; spec associate_targets,
// SPEC.md:296-304) and area queries (Algorithm 5; spec
// area_query) on the GPU -- SURVEY.md §8(f) rank 2, the step
// before the evaluation path once targets are arbitrary.
//
// Algorithm 3 scatters: every source runs an area query of radius r_danger(s)
// and marks the targets it finds, every centre one of radius r_c(1+eps) and
// claims the closest endangered targets.  The output is a pure function of the
// point sets (PAPER.md:1385-1388 says as much), so the GPU gathers instead: one
// thread per target walks the plan's octree once, pruning with per-box bounds
// (largest danger radius of the subtree's sources, largest centre radius of its
// centres), and keeps both answers -- "some source within its danger radius" and
// "nearest admissible centre, ties to the lowest id".  No atomics on results,
// no scatter conflicts, one pass.
//
// The walk is stackless: boxes are in DFS preorder (csrc/host/plan.cpp), so a
// subtree is the id range [b, sub_end[b]); "descend" is b + 1 and "skip" is
// b = sub_end[b].  Targets are visited in Morton order (63-bit keys on the root
// cube, one radix sort) so a warp's 32 walks share their paths.
//
// Distances are compared squared as (dx*dx + dy*dy) + dz*dz with every
// operation rounded on its own (__dmul_rn / __dadd_rn: no FMA contraction), the
// arithmetic oracle/assoc_brute.cpp uses, so the answers are bit-identical --
// including the tie between a node's two centres x +- r n.  Box pruning uses a
// relative slack of 1e-9 so rounding never drops a qualifying particle.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../host/common.hpp"

struct qbxg_locator {
  int device = 0;
  cudaStream_t stream = nullptr;
  int32_t nb = 0;
  int64_t ns = 0, nc = 0;
  double root[4] = {0, 0, 0, 1};  // root centre, |root|
  std::vector<void*> owned;
  double4* box = nullptr;     // (cx, cy, cz, |b|)
  int* sub_end = nullptr;     // DFS subtree end
  int2* src_own = nullptr;    // (start, count) in the sorted source array
  int2* ctr_own = nullptr;
  double2* bnd = nullptr;     // (max danger radius, max centre radius) over the subtree; -1 if none
  double4* src = nullptr;     // sorted (x, y, z, r_danger)
  double4* ctr = nullptr;     // sorted (x, y, z, r_c)
  int* ctr_id = nullptr;      // sorted -> original centre id
  int8_t* ctr_side = nullptr; // sorted side tags, or null
  // per-call scratch (grown on demand)
  void* work = nullptr;
  size_t work_bytes = 0;
  void* io = nullptr;
  size_t io_bytes = 0;
  ~qbxg_locator() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : owned) cudaFree(p);
    if (work) cudaFree(work);
    if (io) cudaFree(io);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace qbxg {
namespace {

#define ACK(call)                                                                                    \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      throw ::qbxg::CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call); \
  } while (0)

constexpr double kSlack = 1.0 + 1e-9;
constexpr int kAssocThreads = 128;

template <class T>
T* upload(qbxg_locator& L, const std::vector<T>& v) {
  void* p = nullptr;
  ACK(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)));
  L.owned.push_back(p);
  if (!v.empty()) ACK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, L.stream));
  return static_cast<T*>(p);
}

void grow(void*& p, size_t& have, size_t need) {
  if (need <= have) return;
  if (p) ACK(cudaFree(p));
  p = nullptr;
  have = 0;
  ACK(cudaMalloc(&p, need));
  have = need;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__device__ __forceinline__ double dist2_rn(double ax, double ay, double az, double bx, double by, double bz) {
  const double dx = ax - bx, dy = ay - by, dz = az - bz;
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// squared l2 distance from t to the closed cube of box b (rounding-tolerant use only)
__device__ __forceinline__ double box_d2(double tx, double ty, double tz, double4 b) {
  const double ex = fmax(fabs(tx - b.x) - b.w, 0.0), ey = fmax(fabs(ty - b.y) - b.w, 0.0),
               ez = fmax(fabs(tz - b.z) - b.w, 0.0);
  return ex * ex + ey * ey + ez * ez;
}

// per-box bounds over the subtree's sorted ranges: one CTA per box
__global__ void __launch_bounds__(128) k_box_bounds(int nb, const int2* __restrict__ src_sub,
                                                   const int2* __restrict__ ctr_sub,
                                                   const double4* __restrict__ src,
                                                   const double4* __restrict__ ctr, double2* __restrict__ bnd) {
  __shared__ double s_red[2][4];
  const int b = blockIdx.x;
  const int2 rs = src_sub[b], rc = ctr_sub[b];
  double md = -1.0, mr = -1.0;
  for (int i = threadIdx.x; i < rs.y; i += blockDim.x) md = fmax(md, src[rs.x + i].w);
  for (int i = threadIdx.x; i < rc.y; i += blockDim.x) mr = fmax(mr, ctr[rc.x + i].w);
  for (int o = 16; o > 0; o >>= 1) {
    md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) s_red[0][w] = md, s_red[1][w] = mr;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < int(blockDim.x >> 5); ++k) md = fmax(md, s_red[0][k]), mr = fmax(mr, s_red[1][k]);
    bnd[b] = make_double2(md, mr);
  }
}

__device__ __forceinline__ unsigned long long spread21(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

__global__ void k_morton(int n, const double* __restrict__ t, double4 root, unsigned long long* __restrict__ key,
                         int* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = double(1 << 21) / (2.0 * root.w);
  unsigned long long q[3];
  const double c[3] = {root.x, root.y, root.z};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double u = (t[3 * size_t(i) + d] - (c[d] - root.w)) * s;
    u = fmin(fmax(u, 0.0), double((1 << 21) - 1));  // also maps NaN to 0
    q[d] = static_cast<unsigned long long>(u);
  }
  key[i] = spread21(q[0]) | spread21(q[1]) << 1 | spread21(q[2]) << 2;
  idx[i] = i;
}

// one thread per target (Morton order): endangered flag + nearest admissible centre
__global__ void __launch_bounds__(kAssocThreads) k_associate(
    int n, const int* __restrict__ order, const double* __restrict__ tpos, const int8_t* __restrict__ side_pref,
    double onep, int nb, const double4* __restrict__ box, const int* __restrict__ sub_end,
    const int2* __restrict__ src_own, const int2* __restrict__ ctr_own, const double2* __restrict__ bnd,
    const double4* __restrict__ src, const double4* __restrict__ ctr, const int* __restrict__ ctr_id,
    const int8_t* __restrict__ ctr_side, int* __restrict__ out, unsigned long long* __restrict__ n_flagged) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ti = order ? order[i] : i;
  const double tx = tpos[3 * size_t(ti)], ty = tpos[3 * size_t(ti) + 1], tz = tpos[3 * size_t(ti) + 2];
  const int side = (side_pref && ctr_side) ? int(side_pref[ti]) : 0;
  bool endangered = false;
  double best = INFINITY;
  int best_id = -1;
  int b = 0;
  while (b < nb) {
    const double4 bx = box[b];
    const double2 bd = __ldg(&bnd[b]);
    const double d2b = box_d2(tx, ty, tz, bx);
    const bool s_ok = !endangered && bd.x >= 0.0 && d2b <= bd.x * bd.x * kSlack;
    const double rm = bd.y * onep;
    const bool c_ok = bd.y >= 0.0 && d2b <= rm * rm * kSlack && d2b <= best * kSlack;
    if (!s_ok && !c_ok) {
      b = __ldg(&sub_end[b]);
      continue;
    }
    if (s_ok) {
      const int2 r = __ldg(&src_own[b]);
      for (int k = 0; k < r.y; ++k) {
        const double4 s = src[r.x + k];
        if (dist2_rn(tx, ty, tz, s.x, s.y, s.z) <= __dmul_rn(s.w, s.w)) {
          endangered = true;
          break;
        }
      }
    }
    if (c_ok) {
      const int2 r = __ldg(&ctr_own[b]);
      for (int k = 0; k < r.y; ++k) {
        if (side != 0 && int(ctr_side[r.x + k]) != side) continue;
        const double4 c = ctr[r.x + k];
        const double d2 = dist2_rn(tx, ty, tz, c.x, c.y, c.z);
        const double rr = __dmul_rn(c.w, onep);
        if (d2 <= __dmul_rn(rr, rr)) {
          const int id = __ldg(&ctr_id[r.x + k]);
          if (d2 < best || (d2 == best && id < best_id)) best = d2, best_id = id;
        }
      }
    }
    ++b;
  }
  int a = -1;
  if (endangered) {
    a = best_id >= 0 ? best_id : -2;
    if (best_id < 0) atomicAdd(n_flagged, 1ull);
  }
  out[ti] = a;
}

// area query: leaves whose closed cube meets the closed l-inf ball (c, r)
__device__ __forceinline__ bool cube_meets(double cx, double cy, double cz, double lim, double4 b) {
  return fabs(cx - b.x) <= lim && fabs(cy - b.y) <= lim && fabs(cz - b.z) <= lim;
}

__global__ void k_area_query(int nq, const double* __restrict__ qc, const double* __restrict__ qr, int nb,
                             const double4* __restrict__ box, const int* __restrict__ sub_end,
                             long long* __restrict__ counts, const long long* __restrict__ starts,
                             int* __restrict__ leaves) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double cx = qc[3 * size_t(q)], cy = qc[3 * size_t(q) + 1], cz = qc[3 * size_t(q) + 2], r = qr[q];
  long long cnt = 0, pos = starts ? starts[q] : 0;
  int b = 0;
  while (b < nb) {
    const double4 bx = box[b];
    const int e = __ldg(&sub_end[b]);
    const double lim = r + bx.w;
    if (e == b + 1) {  // leaf: the exact test
      if (cube_meets(cx, cy, cz, lim, bx)) {
        if (leaves) leaves[pos] = b;
        ++pos, ++cnt;
      }
      b = e;
    } else {
      b = cube_meets(cx, cy, cz, lim * kSlack, bx) ? b + 1 : e;
    }
  }
  if (counts) counts[q] = cnt;
}

void associate_core(qbxg_locator& L, int n, const double* d_t, double onep, const int8_t* d_side, int* d_out,
                    unsigned long long* d_cnt, cudaStream_t s) {
  ACK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s));
  if (n == 0) return;
  // scratch: keys[2n] | idx[2n] | cub temp
  size_t temp = 0;
  ACK(cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<unsigned long long*>(nullptr),
                                      static_cast<unsigned long long*>(nullptr), static_cast<int*>(nullptr),
                                      static_cast<int*>(nullptr), n, 0, 63, s));
  const size_t kb = align256(sizeof(unsigned long long) * size_t(n)), ib = align256(sizeof(int) * size_t(n));
  grow(L.work, L.work_bytes, 2 * kb + 2 * ib + align256(temp));
  char* w = static_cast<char*>(L.work);
  auto* k0 = reinterpret_cast<unsigned long long*>(w);
  auto* k1 = reinterpret_cast<unsigned long long*>(w + kb);
  int* i0 = reinterpret_cast<int*>(w + 2 * kb);
  int* i1 = reinterpret_cast<int*>(w + 2 * kb + ib);
  void* tp = w + 2 * kb + 2 * ib;
  const double4 root = make_double4(L.root[0], L.root[1], L.root[2], L.root[3]);
  k_morton<<<(n + 255) / 256, 256, 0, s>>>(n, d_t, root, k0, i0);
  ACK(cub::DeviceRadixSort::SortPairs(tp, temp, k0, k1, i0, i1, n, 0, 63, s));
  k_associate<<<(n + kAssocThreads - 1) / kAssocThreads, kAssocThreads, 0, s>>>(
      n, i1, d_t, d_side, onep, L.nb, L.box, L.sub_end, L.src_own, L.ctr_own, L.bnd, L.src, L.ctr, L.ctr_id,
      L.ctr_side, d_out, d_cnt);
  ACK(cudaGetLastError());
}

void check_eps(double eps) {
  if (!(eps >= 0.0) || !std::isfinite(eps)) throw InvalidArgument("associate_targets: eps_ta must be finite and >= 0");
}

}  // namespace
}  // namespace qbxg

extern "C" {

int qbxg_locator_create(const qbxg_plan* plan, const qbxg_geometry* geom, const double* danger,
                        const int8_t* center_side, qbxg_locator** out) {
  using namespace qbxg;
  return guarded([&] {
    if (!plan || !geom || !out) throw InvalidArgument("locator_create: null argument");
    *out = nullptr;
    qbxg_plan_view v;
    if (qbxg_plan_view_get(plan, &v) != QBXG_OK) throw InvalidArgument(get_last_error());
    if (geom->n_sources != v.n_sources || geom->n_centers != v.n_centers)
      throw InvalidArgument("locator_create: geometry does not match the plan's sources / centres");
    if ((v.n_sources && (!geom->source_pos || !danger)) ||
        (v.n_centers && (!geom->center_pos || !geom->center_radius)))
      throw InvalidArgument("locator_create: null array");
    for (int64_t i = 0; i < v.n_sources; ++i)
      if (!(danger[i] >= 0.0) || !std::isfinite(danger[i]))
        throw InvalidArgument("locator_create: danger radius must be finite and >= 0 (source " + std::to_string(i) +
                              ")");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device available (the qbxg GPU path has no CPU fallback)");
    }
    auto L = std::make_unique<qbxg_locator>();
    ACK(cudaGetDevice(&L->device));
    ACK(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking));
    const int32_t nb = v.n_boxes;
    L->nb = nb;
    L->ns = v.n_sources;
    L->nc = v.n_centers;
    for (int d = 0; d < 3; ++d) L->root[d] = v.root_center[d];
    L->root[3] = v.root_radius;
    std::vector<double4> box(nb);
    std::vector<int> sub_end(nb);
    std::vector<int2> so(nb), co(nb), ss(nb), cs(nb);
    for (int32_t b = 0; b < nb; ++b) {
      box[b] = make_double4(v.box_center[3 * b], v.box_center[3 * b + 1], v.box_center[3 * b + 2], v.box_radius[b]);
      so[b] = make_int2(v.src_own_start[b], v.src_own_count[b]);
      co[b] = make_int2(v.ctr_own_start[b], v.ctr_own_count[b]);
      ss[b] = make_int2(v.src_sub_start[b], v.src_sub_count[b]);
      cs[b] = make_int2(v.ctr_sub_start[b], v.ctr_sub_count[b]);
    }
    for (int32_t b = nb - 1; b >= 0; --b) {  // DFS preorder: subtree = [b, sub_end)
      int e = b + 1;
      for (int32_t k = v.child_starts[b]; k < v.child_starts[b + 1]; ++k) e = std::max(e, sub_end[v.children[k]]);
      sub_end[b] = e;
    }
    std::vector<double4> src(v.n_sources), ctr(v.n_centers);
    std::vector<int> cid(v.n_centers);
    std::vector<int8_t> cside(center_side ? v.n_centers : 0);
    for (int64_t i = 0; i < v.n_sources; ++i) {
      const int64_t o = v.src_perm[i];
      src[i] = make_double4(geom->source_pos[3 * o], geom->source_pos[3 * o + 1], geom->source_pos[3 * o + 2],
                            danger[o]);
    }
    for (int64_t i = 0; i < v.n_centers; ++i) {
      const int64_t o = v.ctr_perm[i];
      ctr[i] = make_double4(geom->center_pos[3 * o], geom->center_pos[3 * o + 1], geom->center_pos[3 * o + 2],
                            geom->center_radius[o]);
      cid[i] = int(o);
      if (center_side) cside[i] = center_side[o];
    }
    L->box = upload(*L, box);
    L->sub_end = upload(*L, sub_end);
    L->src_own = upload(*L, so);
    L->ctr_own = upload(*L, co);
    L->src = upload(*L, src);
    L->ctr = upload(*L, ctr);
    L->ctr_id = upload(*L, cid);
    if (center_side) L->ctr_side = upload(*L, cside);
    int2* dss = upload(*L, ss);
    int2* dcs = upload(*L, cs);
    void* pb = nullptr;
    ACK(cudaMalloc(&pb, std::max<size_t>(1, size_t(nb)) * sizeof(double2)));
    L->owned.push_back(pb);
    L->bnd = static_cast<double2*>(pb);
    if (nb > 0) k_box_bounds<<<nb, 128, 0, L->stream>>>(nb, dss, dcs, L->src, L->ctr, L->bnd);
    ACK(cudaGetLastError());
    ACK(cudaStreamSynchronize(L->stream));
    *out = L.release();
  });
}

void qbxg_locator_destroy(qbxg_locator* loc) { delete loc; }

int qbxg_associate_targets_device(qbxg_locator* loc, int64_t n, const double* d_t, double eps,
                                  const int8_t* d_side, int32_t* d_out, unsigned long long* d_cnt, void* stream) {
  using namespace qbxg;
  return guarded([&] {
    if (!loc || !d_cnt || (n > 0 && (!d_t || !d_out))) throw InvalidArgument("associate_targets: null argument");
    if (n < 0 || n >= (int64_t(1) << 31)) throw InvalidArgument("associate_targets: bad target count");
    check_eps(eps);
    if (d_side && !loc->ctr_side) throw InvalidArgument("associate_targets: side_pref needs centre sides at locator_create");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : loc->stream;
    associate_core(*loc, int(n), d_t, 1.0 + eps, d_side, reinterpret_cast<int*>(d_out), d_cnt, s);
  });
}

int qbxg_associate_targets(qbxg_locator* loc, int64_t n, const double* tpos, double eps, const int8_t* side_pref,
                           int32_t* out, int64_t* n_flagged) {
  using namespace qbxg;
  return guarded([&] {
    if (!loc || (n > 0 && (!tpos || !out))) throw InvalidArgument("associate_targets: null argument");
    if (n < 0 || n >= (int64_t(1) << 31)) throw InvalidArgument("associate_targets: bad target count");
    check_eps(eps);
    if (side_pref && !loc->ctr_side) throw InvalidArgument("associate_targets: side_pref needs centre sides at locator_create");
    for (int64_t i = 0; i < 3 * n; ++i)
      if (!std::isfinite(tpos[i]))
        throw InvalidArgument("associate_targets: non-finite target position at index " + std::to_string(i / 3));
    cudaStream_t s = loc->stream;
    // io: targets[3n] | side[n] | out[n] | count
    const size_t tb = align256(sizeof(double) * 3 * size_t(n)), sb = align256(size_t(n)),
                 ob = align256(sizeof(int) * size_t(n));
    grow(loc->io, loc->io_bytes, tb + sb + ob + 256);
    char* w = static_cast<char*>(loc->io);
    double* dt = reinterpret_cast<double*>(w);
    int8_t* ds = side_pref ? reinterpret_cast<int8_t*>(w + tb) : nullptr;
    int* dout = reinterpret_cast<int*>(w + tb + sb);
    auto* dc = reinterpret_cast<unsigned long long*>(w + tb + sb + ob);
    if (n) ACK(cudaMemcpyAsync(dt, tpos, sizeof(double) * 3 * size_t(n), cudaMemcpyHostToDevice, s));
    if (n && side_pref) ACK(cudaMemcpyAsync(ds, side_pref, size_t(n), cudaMemcpyHostToDevice, s));
    associate_core(*loc, int(n), dt, 1.0 + eps, ds, dout, dc, s);
    unsigned long long cnt = 0;
    if (n) ACK(cudaMemcpyAsync(out, dout, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost, s));
    ACK(cudaMemcpyAsync(&cnt, dc, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    ACK(cudaStreamSynchronize(s));
    if (n_flagged) *n_flagged = int64_t(cnt);
  });
}

int qbxg_area_query(qbxg_locator* loc, int64_t nq, const double* centers, const double* radii, int64_t* starts,
                    int32_t* leaves, int64_t capacity) {
  using namespace qbxg;
  return guarded([&] {
    if (!loc || !starts || (nq > 0 && (!centers || !radii))) throw InvalidArgument("area_query: null argument");
    if (nq < 0 || nq >= (int64_t(1) << 31)) throw InvalidArgument("area_query: bad query count");
    for (int64_t i = 0; i < nq; ++i) {
      if (!(radii[i] >= 0.0) || !std::isfinite(radii[i]))
        throw InvalidArgument("area_query: radius must be finite and >= 0 (query " + std::to_string(i) + ")");
      for (int d = 0; d < 3; ++d)
        if (!std::isfinite(centers[3 * i + d]))
          throw InvalidArgument("area_query: non-finite centre (query " + std::to_string(i) + ")");
    }
    starts[0] = 0;
    if (nq == 0) return;
    cudaStream_t s = loc->stream;
    const size_t cb = align256(sizeof(double) * 3 * size_t(nq)), rb = align256(sizeof(double) * size_t(nq)),
                 nb8 = align256(sizeof(long long) * size_t(nq));
    grow(loc->io, loc->io_bytes, cb + rb + 2 * nb8);
    char* w = static_cast<char*>(loc->io);
    double* dc = reinterpret_cast<double*>(w);
    double* dr = reinterpret_cast<double*>(w + cb);
    auto* dcnt = reinterpret_cast<long long*>(w + cb + rb);
    auto* dst = reinterpret_cast<long long*>(w + cb + rb + nb8);
    ACK(cudaMemcpyAsync(dc, centers, sizeof(double) * 3 * size_t(nq), cudaMemcpyHostToDevice, s));
    ACK(cudaMemcpyAsync(dr, radii, sizeof(double) * size_t(nq), cudaMemcpyHostToDevice, s));
    const int g = int((nq + 127) / 128);
    k_area_query<<<g, 128, 0, s>>>(int(nq), dc, dr, loc->nb, loc->box, loc->sub_end, dcnt, nullptr, nullptr);
    ACK(cudaGetLastError());
    std::vector<long long> cnt(nq);
    ACK(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(long long) * size_t(nq), cudaMemcpyDeviceToHost, s));
    ACK(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < nq; ++i) starts[i + 1] = starts[i] + cnt[i];
    const int64_t total = starts[nq];
    if (!leaves) return;  // counts only
    if (capacity < total)
      throw InvalidArgument("area_query: leaves_capacity " + std::to_string(capacity) + " < " + std::to_string(total) +
                            " leaves found (out_starts holds the counts)");
    if (total == 0) return;
    std::vector<long long> st(starts, starts + nq);
    ACK(cudaMemcpyAsync(dst, st.data(), sizeof(long long) * size_t(nq), cudaMemcpyHostToDevice, s));
    void* pl = nullptr;
    ACK(cudaMallocAsync(&pl, sizeof(int) * size_t(total), s));
    k_area_query<<<g, 128, 0, s>>>(int(nq), dc, dr, loc->nb, loc->box, loc->sub_end, nullptr, dst,
                                   static_cast<int*>(pl));
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(leaves, pl, sizeof(int) * size_t(total), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(pl, s);
    ACK(e);
    ACK(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
