/*
 * qbxg.h -- C ABI of the B200-native GIGAQBX-FMM evaluation path.
 *
 * Drop-in boundary for the reference's in-process C++ API (namespace qbx):
 *   - qbxg_direct_sum   replaces qbx::direct_sum
 *                       (/root/reference/proj/include/qbx3d/kernels.hpp:39-40,
 *                        /root/reference/proj/src/kernels.cpp:46-73)
 *   - qbxg_plan_create  replaces build_tree + build_lists
 *                       (declared in
 *                        proj/CMakeLists.txt:24-25 as src/tree.cpp, src/interaction_lists.cpp)
 *   - qbxg_create/qbxg_apply replace execute(bundle, density, FmmConfig)
 *                       (Algorithm 4 Stages 2-9 at PAPER.md:2343-2430;
 *                        declared as src/fmm.cpp in proj/CMakeLists.txt:27)
 *   - qbxg_plan_ledger  replaces modeled_flops / CostLedger
 *   - qbxg_geometry_*   procedural inputs of BASELINE.json configs 0-4;
 *                       stands in for gen_sphere / gen_urchin
 *
 * Conventions
 *   - Plain pointers and sizes only; all arrays are host memory unless the
 *     function name ends in _device.
 *   - Positions are AoS double[3*N], byte-compatible with std::vector<qbx::Vec3>
 *     (/root/reference/proj/include/qbx3d/vec3.hpp:9-10: three doubles, 24 B).
 *   - Source weights are premultiplied (quadrature weight x density) and dipole
 *     moments are weight x density x normal, exactly as qbx::SourceEnsemble
 *     (/root/reference/proj/include/qbx3d/kernels.hpp:16-22).
 *   - Target association follows qbx::TargetSet::association
 *     (/root/reference/proj/include/qbx3d/kernels.hpp:31-35): >=0 centre id, -1 conventional.
 *   - Potentials include the 1/(4 pi) of G, as direct_sum does
 *     (/root/reference/proj/src/kernels.cpp:67).
 *   - Centre coefficients are returned in the paper's normalisation, Eq. (5)/(8)
 *     (PAPER.md:287-289, 326-330): local coefficient (L_c)_n^m for 0<=m<=n<=p_qbx,
 *     packed n-major at index n(n+1)/2+m, interleaved (re,im); (L_c)_n^{-m} is the
 *     complex conjugate for real densities.
 *   - Every function returns a status code; no C++ exception crosses the ABI.
 *     qbxg_last_error() returns the message of the last failure on this thread.
 */
#ifndef QBXG_H_
#define QBXG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror the reference's exception classes) ---------- */
enum {
  QBXG_OK = 0,
  QBXG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (kernels.cpp:28-36)   */
  QBXG_ERR_DOMAIN = 2,           /* std::domain_error     (kernels.cpp:15,22,69) */
  QBXG_ERR_CUDA = 3,
  QBXG_ERR_NCCL = 4,
  QBXG_ERR_INTERNAL = 5,
  QBXG_ERR_NO_DEVICE = 6
};

enum {
  QBXG_KERNEL_LAPLACE_SL = 0,    /* single layer: sum w G                     */
  QBXG_KERNEL_LAPLACE_SL_DL = 1, /* single + double layer: sum w G + m.grad_y G */
  QBXG_KERNEL_HELMHOLTZ_SL = 2,  /* e^{ikr}/(4 pi r), complex density: qbxg_apply_complex */
  QBXG_KERNEL_HELMHOLTZ_SL_DL = 3 /* single + double layer: sum w G_k + m.grad_y G_k (complex w, m) */
};

/* Interaction-list kinds (Definitions 1-8). */
enum {
  QBXG_LIST_U = 0,       /* List 1                 */
  QBXG_LIST_V = 1,       /* List 2                 */
  QBXG_LIST_W_CLOSE = 2, /* List 3 close           */
  QBXG_LIST_W_FAR = 3,   /* List 3 far             */
  QBXG_LIST_X_CLOSE = 4, /* List 4 close           */
  QBXG_LIST_X_FAR = 5,   /* List 4 far             */
  QBXG_NUM_LISTS = 6
};

/* Stages timed by qbxg_apply (CUDA events). */
enum {
  QBXG_T_H2D = 0,      /* density upload + permutation                 */
  QBXG_T_P2M = 1,      /* Stage 2 leaf formation                        */
  QBXG_T_M2M = 2,      /* Stage 2 postorder shifts                      */
  QBXG_T_NEAR = 3,     /* Stages 3, 5a, 6a: P2QBXL + P2P over U, W_close, X_close */
  QBXG_T_M2L = 4,      /* Stage 4                                       */
  QBXG_T_WFAR = 5,     /* Stage 5b: M2QBXL + M2P                        */
  QBXG_T_P2L = 6,      /* Stage 6b                                      */
  QBXG_T_L2L = 7,      /* Stage 7                                       */
  QBXG_T_L2QBXL = 8,   /* Stage 8                                       */
  QBXG_T_EVAL = 9,     /* Stage 9: QBXL2P + L2P + sum                   */
  QBXG_T_D2H = 10,     /* result download + un-permutation              */
  QBXG_T_TOTAL = 11,
  QBXG_NUM_TIMERS = 12
};

typedef struct {
  int32_t p_fmm;        /* FMM order (p)                                  */
  int32_t p_qbx;        /* QBX order (q), q <= p            */
  double t_f;           /* target confinement factor, < 2 sqrt(3) - 2     */
  int32_t n_max;        /* max particles (sources+centres+targets) per box */
  int32_t kernel;       /* QBXG_KERNEL_*                                  */
  double helmholtz_k;   /* wavenumber k of the Helmholtz kernels           */
  int32_t w_far_demote; /* Remark 1: a List-3-far box whose
                           subtree holds fewer than this many sources is replaced by
                           its source leaves in List 3 close; 0 disables.  */
  int32_t level_restrict; /* 1: level-restricted tree (Remark C.1,
                           PAPER.md:3661-3687): leaves are subdivided until
                           adjacent leaves differ by at most one level; 0: off
                           (default).  Host plan only (qbxg_plan_create).  */
} qbxg_config;

typedef struct {
  int64_t n_sources;
  const double* source_pos;    /* 3*n_sources                             */
  int64_t n_centers;
  const double* center_pos;    /* 3*n_centers                             */
  const double* center_radius; /* n_centers                               */
  int64_t n_targets;
  const double* target_pos;    /* 3*n_targets                             */
  const int32_t* association;  /* n_targets: centre id or -1              */
} qbxg_geometry;

/* ---- procedural inputs (BASELINE.json configs) ---------- */
enum { QBXG_SURF_ICOSPHERE = 0, QBXG_SURF_TORUS = 1, QBXG_SURF_URCHIN = 2, QBXG_SURF_URCHIN_ARRAY = 3 };
enum { QBXG_DENS_UNIFORM = 0, QBXG_DENS_ONES = 1, QBXG_DENS_FOURIER8 = 2, QBXG_DENS_COMPLEX_UNIFORM = 3 };

typedef struct {
  int32_t surface;        /* QBXG_SURF_*                                   */
  int32_t level;          /* icosphere subdivision level                   */
  int32_t nu, nv;         /* torus grid                                    */
  int32_t nx, ny, nz;     /* urchin array dimensions                       */
  double spacing;         /* urchin array spacing                          */
  int32_t density;        /* QBXG_DENS_*                                   */
  int32_t reserved;
  int64_t n_volume_targets; /* uniform volume targets drawn before filtering */
  double volume_halfwidth;  /* cube [-hw, hw]^3                            */
  uint64_t seed;
} qbxg_geometry_spec;

typedef struct qbxg_generated qbxg_generated;

typedef struct {
  int64_t n_triangles;
  int64_t n_sources;
  const double* source_pos;    /* 3*n_sources                               */
  const double* source_normal; /* 3*n_sources, unit normals                 */
  const double* quad_weight;   /* n_sources (area-scaled Duffy weights)     */
  const double* density;       /* n_sources (real) or 2*n_sources (complex) */
  int32_t density_is_complex;
  int64_t n_centers;
  const double* center_pos;
  const double* center_radius;
  int64_t n_targets;           /* 2*n_sources on-surface + retained volume  */
  const double* target_pos;
  const int32_t* association;
  int64_t n_volume_drawn;      /* volume targets drawn (before filtering)   */
} qbxg_generated_view;

int qbxg_geometry_spec_for_config(int32_t config_id, int32_t variant, uint64_t seed,
                                  qbxg_geometry_spec* out);
int qbxg_geometry_generate(const qbxg_geometry_spec* spec, qbxg_generated** out);
int qbxg_geometry_view(const qbxg_generated* g, qbxg_generated_view* out);
void qbxg_geometry_destroy(qbxg_generated* g);

/* ---- host tree + interaction lists (Stage 1, stays in host C++) --------- */
typedef struct qbxg_plan qbxg_plan;

typedef struct {
  int32_t n_boxes;
  int32_t n_levels;
  double root_center[3];
  double root_radius;             /* l-inf half width |root|              */
  const double* box_center;       /* 3*n_boxes                            */
  const double* box_radius;       /* n_boxes (|b|)                        */
  const int32_t* box_level;       /* n_boxes                              */
  const int32_t* box_parent;      /* n_boxes (-1 for root)                */
  const int32_t* child_starts;    /* n_boxes+1 (CSR into children)        */
  const int32_t* children;
  const int32_t* level_starts;    /* n_levels+1 (CSR into level_boxes)    */
  const int32_t* level_boxes;
  /* per-role ranges in the box-sorted particle arrays (DFS preorder)     */
  const int32_t* src_own_start; const int32_t* src_own_count;
  const int32_t* src_sub_start; const int32_t* src_sub_count;
  const int32_t* ctr_own_start; const int32_t* ctr_own_count;
  const int32_t* ctr_sub_start; const int32_t* ctr_sub_count;
  const int32_t* tgt_own_start; const int32_t* tgt_own_count;  /* conventional targets */
  const int32_t* tgt_sub_start; const int32_t* tgt_sub_count;
  int64_t n_sources, n_centers, n_conv_targets, n_targets;
  const int32_t* src_perm;        /* sorted pos -> original source index   */
  const int32_t* ctr_perm;        /* sorted pos -> original centre index   */
  const int32_t* tgt_perm;        /* sorted pos -> original target index (conventional only) */
  const uint8_t* box_flags;       /* bit0 target box, bit1 target-ancestor, bit2 has sources in subtree, bit3 leaf */
  const int64_t* list_starts[QBXG_NUM_LISTS]; /* n_boxes+1 each           */
  const int32_t* list_boxes[QBXG_NUM_LISTS];
  uint64_t list_hash[QBXG_NUM_LISTS];         /* FNV-1a over (starts, boxes) */
  double build_seconds_tree, build_seconds_lists;
} qbxg_plan_view;

enum { QBXG_BOX_TARGET = 1, QBXG_BOX_TARGET_ANCESTOR = 2, QBXG_BOX_HAS_SOURCES = 4, QBXG_BOX_LEAF = 8 };

/* Modeled operation counts, Table 3, plus pair counts. */
typedef struct {
  double modeled[QBXG_NUM_LISTS]; /* per list kind                         */
  double modeled_total;
  int64_t entries[QBXG_NUM_LISTS];/* list entries over evaluated boxes     */
  int64_t pairs_qbx_near;         /* (source, centre) pairs, lists 1, 3c, 4c */
  int64_t pairs_p2p_near;         /* (source, conventional target) pairs   */
  int64_t pairs_wfar_centre;      /* (W_far box, centre) pairs             */
  int64_t pairs_wfar_target;      /* (W_far box, conventional target) pairs */
  int64_t pairs_xfar_source;      /* (source, X_far target box) pairs      */
  int64_t n_m2m, n_l2l;           /* child->parent shifts                  */
  int64_t n_p2m_sources;
  int64_t n_l2qbxl_centres;
  int64_t n_l2p_targets;
  int64_t n_qbxl2p_targets;
} qbxg_ledger;

/* ---- multi-GPU sharding ---------------------------------
 * Rank r owns the contiguous DFS-preorder (Morton) box range [cuts[r], cuts[r+1]),
 * cut by a per-box cost model.  Per-box role bits for one rank: */
enum {
  QBXG_SHARD_OWN = 1,        /* box in the rank's range: its centres/targets are evaluated here */
  QBXG_SHARD_SUBTREE = 2,    /* whole subtree in the range: upward pass done here              */
  QBXG_SHARD_STRADDLE = 4,   /* subtree spans ranks: M2M recomputed by every rank after exchange */
  QBXG_SHARD_DOWN = 8        /* in the range or an ancestor of it: M2L / P2L / L2L done here     */
};
/* cuts: n_ranks+1 ints; mask: n_boxes bytes (may be NULL). */
int qbxg_plan_shard(const qbxg_plan* plan, int32_t n_ranks, int32_t rank, int32_t* cuts, uint8_t* mask);

int qbxg_plan_create(const qbxg_config* cfg, const qbxg_geometry* geom, qbxg_plan** out);
int qbxg_plan_view_get(const qbxg_plan* plan, qbxg_plan_view* out);
/* Stage 1 on the GPU: the same plan as qbxg_plan_create,
 * bit for bit (boxes, DFS numbering, permutations, lists and their hashes), with
 * the octree built on the device and the lists built on the device when
 * gpu_lists != 0 (on the host otherwise).  QBXG_ERR_CUDA without a device. */
int qbxg_plan_create_gpu(const qbxg_config* cfg, const qbxg_geometry* geom, int32_t gpu_lists, qbxg_plan** out);
int qbxg_plan_ledger(const qbxg_plan* plan, qbxg_ledger* out);
void qbxg_plan_destroy(qbxg_plan* plan);
/* SPEC.md:370-378 adequately_separated(kind, a, b, t_f), the relation the list
 * builder uses: kind 0 = box_vs_tcr (a < TCR(b): l2 distance from centre(a) to the
 * boundary of the ball of radius sqrt(3)|b|(1+t_f) about centre(b) >= 3|a|),
 * kind 1 = tcr_vs_box (TCR(a) < b: l-inf distance from centre(a) to the boundary
 * of b >= 3|a|(1+t_f)).  ca/cb: box centres (3 doubles), ha/hb: half widths |a|, |b|.
 * *out = 1 when separated.  Pure host function, no device needed. */
int qbxg_adequately_separated(int32_t kind, const double* ca, double ha, const double* cb, double hb, double t_f,
                              int32_t* out);

/* ---- device evaluation (Stages 2-9 on one B200) ------------------------ */
typedef struct qbxg_handle qbxg_handle;

typedef struct {
  double ms[QBXG_NUM_TIMERS];     /* CUDA-event times of the last apply    */
  int32_t kernel_launches;        /* kernels launched by the last apply    */
  int64_t h2d_bytes, d2h_bytes;
} qbxg_timings;

/* Upload geometry, box-sorted particle data, tree and lists; build operator
 * tables.  The plan must have been created from the same cfg and geometry. */
int qbxg_create(const qbxg_config* cfg, const qbxg_geometry* geom, const qbxg_plan* plan,
                int32_t device, qbxg_handle** out);

/* Host-buffer apply (e2e).  weights: n_sources; dipoles: 3*n_sources or NULL
 * (required for QBXG_KERNEL_LAPLACE_SL_DL); out_target_pot: n_targets;
 * out_center_coeffs: NULL or n_centers*2*K_q (K_q=(q+1)(q+2)/2) doubles. */
int qbxg_apply(qbxg_handle* h, const double* weights, const double* dipoles,
               double* out_target_pot, double* out_center_coeffs, qbxg_timings* timings);

/* Device-buffer apply: same layout, pointers in device memory of the handle's
 * GPU, original (caller) ordering; stream may be NULL (handle stream). */
int qbxg_apply_device(qbxg_handle* h, const double* d_weights, const double* d_dipoles,
                      double* d_out_target_pot, double* d_out_center_coeffs,
                      void* cuda_stream, qbxg_timings* timings);

int qbxg_destroy(qbxg_handle* h);

/* Sharded handle for rank `rank` of `n_ranks` (one process per GPU).  Work
 * lists are restricted to the rank's boxes (qbxg_plan_shard); qbxg_apply /
 * qbxg_apply_device then need an NCCL communicator (qbxg_nccl_attach) and
 * return complete results on every rank.  Without NCCL, drive the phases and
 * the multipole exchange yourself: */
/* (n_ranks = 1 is allowed: the handle then runs the same protocol -- packed results,
 * NCCL broadcasts -- on a communicator of one rank; tests use it to exercise NCCL.) */
int qbxg_create_sharded(const qbxg_config* cfg, const qbxg_geometry* geom, const qbxg_plan* plan,
                        int32_t device, int32_t n_ranks, int32_t rank, qbxg_handle** out);
/* phase 1: gather density, P2M, M2M of owned subtrees.
 * phase 2: M2M of straddling boxes, Stages 3-9 for owned boxes; potentials and
 *          centre coefficients of other ranks' targets are written as 0.
 * Helmholtz handles take the complex interleaved DEVICE arrays of qbxg_apply_complex
 * (weights [n_sources][2], dipoles [n_sources][3][2], potentials [n_targets][2],
 * centre locals [n_centers][(p_qbx+1)^2][2]); the exchanged multipole rows are full
 * complex tables, 2 (p_fmm+1)^2 doubles per box. */
int qbxg_apply_phase(qbxg_handle* h, int32_t phase, const double* d_weights, const double* d_dipoles,
                     double* d_out_target_pot, double* d_out_center_coeffs, void* cuda_stream);
/* Device multipole buffer (n_boxes rows of row_doubles, DFS order) and cuts
 * (n_ranks+1): after phase 1, rows [cuts[r], cuts[r+1]) of rank r are final. */
int qbxg_multipole_buffer(qbxg_handle* h, double** d_multipoles, int64_t* row_doubles, int32_t* cuts);
/* Exchange between handles of one process (device copies), e.g. ranks emulated on one GPU. */
int qbxg_exchange_local(qbxg_handle** handles, int32_t n_ranks);
/* NCCL (libnccl.so.2 loaded at run time): rank 0 creates the id, all ranks attach. */
/* Result all-gather of a sharded apply emulated with device copies (ranks driven by
 * qbxg_apply_phase in one process; tests): after phase 2, every rank's packed
 * potentials (and centre coefficients when d_coeffs is given) are copied to all
 * ranks and scattered, so d_pots[r] (n_targets doubles per rank) holds the whole
 * result.  qbxg_apply_device on an NCCL-attached sharded handle does the same with
 * one grouped broadcast per rank (qbxg_nccl_attach). */
int qbxg_result_exchange_local(qbxg_handle** hs, int32_t n, double* const* d_pots, double* const* d_coeffs);
int qbxg_nccl_unique_id(uint8_t* out128);
int qbxg_nccl_attach(qbxg_handle* h, const uint8_t* id128);

/* Stream overlap (default off; QBXG_OVERLAP=1 or 2 in the environment turns the
 * default on): the near field runs on a second stream beside the far-field chain (M2L,
 * P2L, L2L) and is joined before the first stage that adds into the centre
 * locals.  Results are bitwise identical either way; per-stage timings of an
 * overlapped apply include the contention between the two streams. */
int qbxg_set_overlap(qbxg_handle* h, int32_t enable);

/* ---- batched densities (repeated applies in iterative
 * solves) ---------------------------------------------------
 * n_rhs densities on one handle, arrays rhs-major with a leading batch dimension:
 * weights [n_rhs][n_sources], dipoles [n_rhs][n_sources][3] (SL+DL), potentials
 * [n_rhs][n_targets], centre coefficients [n_rhs][n_centers][K_q][2] (or null).
 * Each density's result equals qbxg_apply on that density up to rounding; the
 * near field shares one harmonic table per (centre, source) pair between two
 * densities.  The timings report only QBXG_T_TOTAL and the launch count. */
int qbxg_apply_batch(qbxg_handle* h, int32_t n_rhs, const double* weights, const double* dipoles,
                     double* out_target_pot, double* out_center_coeffs_or_null, qbxg_timings* timings);
int qbxg_apply_batch_device(qbxg_handle* h, int32_t n_rhs, const double* d_weights, const double* d_dipoles,
                            double* d_out_target_pot, double* d_out_center_coeffs_or_null, void* cuda_stream,
                            qbxg_timings* timings);

/* ---- near-field P2P, the GPU counterpart of qbx::direct_sum ------------ */
/* pot[i] = (1/4pi) sum_j [w_j/|x_i-y_j| + m_j.(x_i-y_j)/|x_i-y_j|^3].
 * Returns QBXG_ERR_DOMAIN when a target coincides with a source (message names
 * the pair, as kernels.cpp:69-71) and QBXG_ERR_INVALID_ARGUMENT on non-finite
 * source data (kernels.cpp:27-38). */
int qbxg_direct_sum(int64_t n_sources, const double* source_pos, const double* weights,
                    const double* dipoles_or_null, int64_t n_targets, const double* target_pos,
                    double* out_pot);

/* ---- unaccelerated QBX, the GPU counterpart of the spec's direct_qbx ------ */
/* each associated target (association[i] =
 * centre id) gets the order-p_qbx local expansion of its centre formed from ALL
 * sources, evaluated at the target (Eq. (9)); conventional targets
 * (association[i] = -1) get the direct sum.  Same formulas and 1/(4 pi) as
 * qbxg_apply, so |apply - direct_qbx| measures the FMM error alone (Theorem 1).
 * p_qbx in [0, 8]; QBXG_ERR_INVALID_ARGUMENT on bad ids / radii / orders,
 * QBXG_ERR_DOMAIN when a conventional target coincides with a source. */
int qbxg_direct_qbx(int64_t n_sources, const double* source_pos, const double* weights,
                    const double* dipoles_or_null, int64_t n_centers, const double* center_pos,
                    const double* center_radius, int64_t n_targets, const double* target_pos,
                    const int32_t* association, int32_t p_qbx, double* out_pot);

/* ---- Helmholtz FMM (cfg.kernel = QBXG_KERNEL_HELMHOLTZ_SL or _SL_DL,
 * cfg.helmholtz_k > 0, p_fmm <= 20, p_qbx <= 6) ----------------------
 * Complex weights [n_sources][2] in, complex potentials [n_targets][2] out (caller
 * order), optional centre locals [n_centers][(p_qbx+1)^2][2] in the internal basis
 * L_n^m of  phi = sum L_n^m j_n(k|x-c|) Y_n^m(x-c)  (index n^2+n+m; orthonormal Y,
 * no Condon-Shortley phase; formulas in oracle/helm_oracle.cpp).  Stages 2-9 on the
 * same tree and lists as the Laplace path.  SL+DL: complex dipole moments
 * [n_sources][3][2] (m_x, m_y, m_z, each re, im) add m . grad_y G_k(x, y) -- e.g.
 * the Brakhage-Werner combination with w = -i eta q mu and
 * m = q mu n; dipoles_c must be NULL for the single layer.  On a sharded handle
 * (qbxg_create_sharded + qbxg_nccl_attach) every rank passes the whole density and
 * receives the whole result: owned upward pass, multipole broadcast, downward pass
 * for the rank's boxes, all-gather of the owned potentials / centre locals. */
int qbxg_apply_complex(qbxg_handle* h, const double* weights_c, const double* dipoles_c_or_null,
                       double* out_target_pot_c, double* out_center_coeffs_c, qbxg_timings* timings);

/* ---- Helmholtz single (+ double) layer, unaccelerated (BASELINE config 3) --
 * G_k = e^{ik|x-y|}/(4 pi |x-y|), complex weights and potentials interleaved
 * (re, im), optional complex dipoles [n_sources][3][2].  qbxg_helm_direct_sum:
 * pot[t] = sum_s w_s G_k(t, s) + m_s . grad_s G_k(t, s) (QBXG_ERR_DOMAIN on a
 * coincidence).  qbxg_helm_direct_qbx: the spec's direct_qbx for G_k -- each
 * associated target gets its centre's order-p_qbx local from all sources,
 *   L_n^m = ik sum_s w_s h_n(k|s-c|) conj(Y_n^m(s-c)), pot = sum L_n^m j_n(k|t-c|) Y_n^m(t-c)
 * (orthonormal Y without the Condon-Shortley phase), conventional targets the direct
 * sum.  No reference implementation exists; parity is against the
 * complex128 oracle in oracle/helm_oracle.cpp. */
int qbxg_helm_direct_sum(double k, int64_t n_sources, const double* source_pos, const double* weights_c,
                         const double* dipoles_c_or_null, int64_t n_targets, const double* target_pos,
                         double* out_pot_c);
int qbxg_helm_direct_qbx(double k, int64_t n_sources, const double* source_pos, const double* weights_c,
                         const double* dipoles_c_or_null, int64_t n_centers, const double* center_pos, int64_t n_targets, const double* target_pos,
                         const int32_t* association, int32_t p_qbx, double* out_pot_c);

/* ---- target association and area queries on the GPU --
 * Algorithm 3 (spec associate_targets) and
 * Algorithm 5 (spec area_query) over the tree
 * of a plan built from the sources and centres (its targets, if any, are ignored).
 * A locator holds that tree, the box-sorted sources with their danger radii and
 * the box-sorted centres on the device.
 *   qbxg_locator_create: source_danger_radius[n_sources] (the r_danger(s) of
 *     Algorithm 3, >= 0); center_side[n_centers] (int8 side tag, e.g. -1/+1) or
 *     NULL.  geom must hold the sources and centres the plan was built from.
 *   qbxg_associate_targets: target t is endangered iff |t - s| <= r_danger(s) for
 *     some source s; an endangered target is associated with the nearest centre c
 *     with |t - c| <= r_c (1 + eps_ta) (ties: lowest centre id), restricted to
 *     centres with center_side[c] == side_pref[t] when side_pref[t] != 0.
 *     out_association[t] = centre id, -1 (not endangered: conventional) or -2
 *     (endangered, no centre: flagged, counted in *out_n_flagged).  Distances are
 *     compared squared, (dx^2 + dy^2) + dz^2 rounded per operation.
 *   qbxg_area_query: the leaf boxes (plan box ids, ascending) whose closed cube
 *     intersects the closed l-inf ball B(r_i, c_i), i.e. |c_i,d - box_d| <= r_i + |b|
 *     for d = x, y, z.  out_starts[n_queries+1] is always written; out_leaves
 *     (NULL = counts only) is written when leaves_capacity >= out_starts[n_queries],
 *     else QBXG_ERR_INVALID_ARGUMENT after the counts.  side_pref without centre
 *     sides at create is QBXG_ERR_INVALID_ARGUMENT.
 *   The _device variants take device pointers and run on `stream` (NULL = the
 *   locator's stream), without host synchronisation. */
typedef struct qbxg_locator qbxg_locator;
int qbxg_locator_create(const qbxg_plan* plan, const qbxg_geometry* geom, const double* source_danger_radius,
                        const int8_t* center_side_or_null, qbxg_locator** out);
int qbxg_associate_targets(qbxg_locator* loc, int64_t n_targets, const double* target_pos, double eps_ta,
                           const int8_t* side_pref_or_null, int32_t* out_association, int64_t* out_n_flagged);
int qbxg_associate_targets_device(qbxg_locator* loc, int64_t n_targets, const double* d_target_pos, double eps_ta,
                                  const int8_t* d_side_pref_or_null, int32_t* d_out_association,
                                  unsigned long long* d_out_n_flagged, void* stream);
int qbxg_area_query(qbxg_locator* loc, int64_t n_queries, const double* centers, const double* radii,
                    int64_t* out_starts, int32_t* out_leaves, int64_t leaves_capacity);
void qbxg_locator_destroy(qbxg_locator* loc);

/* ---- misc ---------------------------------------------------------------- */
const char* qbxg_last_error(void);
int qbxg_device_count(int32_t* out);
/* fp64 DFMA throughput of `device` (TFLOP/s), the roofline denominator of the fp64 stages. */
int qbxg_measure_fp64_peak(int32_t device, double* out_tflops);
/* fp64 tensor-pipe (DMMA m8n8k4) throughput of `device` (TFLOP/s). */
int qbxg_measure_dmma_peak(int32_t device, double* out_tflops);
const char* qbxg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QBXG_H_ */
