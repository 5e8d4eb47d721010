"""Host-side mirror of the reference's qbx:: interface, over the C ABI.

Names follow the reference (/root/reference/proj/include/qbx3d/kernels.hpp and
SPEC.md): ``SourceEnsemble``, ``TargetSet``, ``direct_sum``, ``FmmConfig``,
``build_plan`` (build_tree + build_lists), ``execute``.  Errors are raised as
the reference raises them: ``ValueError`` for std::invalid_argument and
``ArithmeticError`` (``DomainError``) for std::domain_error.

Every numerical call lands in libqbxg.so (CUDA for sm_100a).  There is no CPU
fallback: without the library or a GPU the calls raise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)


class DomainError(ArithmeticError):
    """Mirror of std::domain_error (kernels.cpp:15, 22, 69-71)."""


class CudaError(RuntimeError):
    pass


def _check(status: int):
    if status == _abi.OK:
        return
    msg = _abi.lib().qbxg_last_error().decode(errors="replace")
    if status == _abi.ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == _abi.ERR_DOMAIN:
        raise DomainError(msg)
    if status in (_abi.ERR_CUDA, _abi.ERR_NO_DEVICE):
        raise CudaError(msg)
    raise RuntimeError(f"qbxg status {status}: {msg}")


def _ptr(a, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def _arr(p, n, dtype):
    if n == 0 or not p:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


# --------------------------------------------------------------------------- inputs
@dataclass
class SourceEnsemble:
    """kernels.hpp:18-29: positions (N,3), premultiplied weights (N,), optional dipole moments (N,3)."""
    positions: np.ndarray
    weights: np.ndarray
    dipole_moments: np.ndarray | None = None

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1, 3)
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float64).reshape(-1)
        if self.dipole_moments is not None and np.size(self.dipole_moments) == 0:
            self.dipole_moments = None
        if self.dipole_moments is not None:
            self.dipole_moments = np.ascontiguousarray(self.dipole_moments, dtype=np.float64).reshape(-1, 3)

    def size(self):
        return self.positions.shape[0]

    def has_dipoles(self):
        return self.dipole_moments is not None

    def total_abs_weight(self):
        return float(np.abs(self.weights).sum())


@dataclass
class TargetSet:
    """kernels.hpp:31-37: positions (M,3) and association (centre id or -1)."""
    positions: np.ndarray
    association: np.ndarray | None = None

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1, 3)
        if self.association is None:
            self.association = -np.ones(self.positions.shape[0], dtype=np.int32)
        self.association = np.ascontiguousarray(self.association, dtype=np.int32).reshape(-1)

    def size(self):
        return self.positions.shape[0]


@dataclass
class FmmConfig:
    """SPEC.md:414-417 (p_fmm, p_qbx, t_f, n_max, demotion threshold, level restriction)."""
    p_fmm: int = 15
    p_qbx: int = 5
    t_f: float = 0.9
    n_max: int = 64
    kernel: int = _abi.KERNEL_LAPLACE_SL
    w_far_demote: int = 0
    helmholtz_k: float = 0.0  # wavenumber, kernels 2 / 3 (Helmholtz single / single + double layer)
    level_restrict: int = 0   # 1 = subdivide until adjacent leaves differ by <= 1 level

    def to_c(self):
        return _abi.Config(self.p_fmm, self.p_qbx, self.t_f, self.n_max, self.kernel, float(self.helmholtz_k),
                           self.w_far_demote, int(self.level_restrict))

    @property
    def kq(self):
        return (self.p_qbx + 1) * (self.p_qbx + 2) // 2

    @property
    def kp(self):
        return (self.p_fmm + 1) * (self.p_fmm + 2) // 2


@dataclass
class Geometry:
    """Geometry bundle: sources, QBX centres (+radii), targets (+association)."""
    source_pos: np.ndarray
    center_pos: np.ndarray
    center_radius: np.ndarray
    target_pos: np.ndarray
    association: np.ndarray
    source_normal: np.ndarray | None = None
    quad_weight: np.ndarray | None = None
    density: np.ndarray | None = None
    n_triangles: int = 0
    n_volume_drawn: int = 0
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        self.source_pos = np.ascontiguousarray(self.source_pos, dtype=np.float64).reshape(-1, 3)
        self.center_pos = np.ascontiguousarray(self.center_pos, dtype=np.float64).reshape(-1, 3)
        self.center_radius = np.ascontiguousarray(self.center_radius, dtype=np.float64).reshape(-1)
        self.target_pos = np.ascontiguousarray(self.target_pos, dtype=np.float64).reshape(-1, 3)
        self.association = np.ascontiguousarray(self.association, dtype=np.int32).reshape(-1)

    @property
    def n_sources(self):
        return self.source_pos.shape[0]

    @property
    def n_centers(self):
        return self.center_pos.shape[0]

    @property
    def n_targets(self):
        return self.target_pos.shape[0]

    def to_c(self):
        return _abi.Geometry(self.n_sources, _ptr(self.source_pos), self.n_centers, _ptr(self.center_pos),
                             _ptr(self.center_radius), self.n_targets, _ptr(self.target_pos),
                             _ptr(self.association, C.c_int32))

    def weights(self, density=None):
        d = self.density if density is None else density
        return np.ascontiguousarray(self.quad_weight * d)

    def dipoles(self, density=None):
        d = self.density if density is None else density
        return np.ascontiguousarray(self.source_normal * (self.quad_weight * d)[:, None])


def geometry_spec(config_id: int, variant: int = 0, seed: int = 0, **overrides) -> _abi.GeometrySpec:
    spec = _abi.GeometrySpec()
    _check(_abi.lib().qbxg_geometry_spec_for_config(config_id, variant, seed, C.byref(spec)))
    for k, v in overrides.items():
        setattr(spec, k, v)
    return spec


def generate_geometry(spec: _abi.GeometrySpec) -> Geometry:
    L = _abi.lib()
    h = C.c_void_p()
    _check(L.qbxg_geometry_generate(C.byref(spec), C.byref(h)))
    try:
        v = _abi.GeneratedView()
        _check(L.qbxg_geometry_view(h, C.byref(v)))
        ns, nc, nt = v.n_sources, v.n_centers, v.n_targets
        g = Geometry(source_pos=_arr(v.source_pos, 3 * ns, np.float64), center_pos=_arr(v.center_pos, 3 * nc, np.float64),
                     center_radius=_arr(v.center_radius, nc, np.float64), target_pos=_arr(v.target_pos, 3 * nt, np.float64),
                     association=_arr(v.association, nt, np.int32),
                     source_normal=_arr(v.source_normal, 3 * ns, np.float64).reshape(-1, 3),
                     quad_weight=_arr(v.quad_weight, ns, np.float64),
                     density=_arr(v.density, ns * (2 if v.density_is_complex else 1), np.float64),
                     n_triangles=v.n_triangles, n_volume_drawn=v.n_volume_drawn)
        return g
    finally:
        L.qbxg_geometry_destroy(h)


def config_geometry(config_id: int, variant: int = 0, seed: int = 0, **overrides) -> Geometry:
    return generate_geometry(geometry_spec(config_id, variant, seed, **overrides))


CONFIG_ORDERS = {0: (10, 3, _abi.KERNEL_LAPLACE_SL), 1: (15, 5, _abi.KERNEL_LAPLACE_SL_DL),
                 2: (15, 5, _abi.KERNEL_LAPLACE_SL), 3: (20, 5, _abi.KERNEL_HELMHOLTZ_SL),
                 4: (15, 5, _abi.KERNEL_LAPLACE_SL_DL)}


def config_fmm(config_id: int, **overrides) -> FmmConfig:
    """FmmConfig of a BASELINE.json config.  List-3-far demotion (Remark 1,
    PAPER.md:2246-2256) uses the spec's cost-balance threshold p^3/q^2
    (SPEC.md:382); pass w_far_demote=0 to disable it."""
    p, q, k = CONFIG_ORDERS[config_id]
    cfg = FmmConfig(p_fmm=p, p_qbx=q, t_f=0.9, n_max=64, kernel=k, w_far_demote=(p ** 3) // max(q * q, 1),
                    helmholtz_k=3.0 if k in (_abi.KERNEL_HELMHOLTZ_SL, _abi.KERNEL_HELMHOLTZ_SL_DL) else 0.0)  # k = 3
    for key, v in overrides.items():
        setattr(cfg, key, v)
    return cfg


# --------------------------------------------------------------------------- plan
class Plan:
    """Host octree + interaction lists (Stage 1), built by libqbxg's host C++."""

    def __init__(self, cfg: FmmConfig, geom: Geometry, device: str = "host", gpu_lists: bool = True):
        """device="host": Stage 1 in host C++ (csrc/host/plan.cpp); device="gpu": the same
        plan bit for bit, octree (and, with gpu_lists, the lists) built on the GPU
        (csrc/cuda/plan_gpu.cu)."""
        self.cfg = cfg
        self.geom = geom
        self._c_cfg = cfg.to_c()
        self._c_geom = geom.to_c()
        self.handle = C.c_void_p()
        if device == "host":
            _check(_abi.lib().qbxg_plan_create(C.byref(self._c_cfg), C.byref(self._c_geom), C.byref(self.handle)))
        elif device == "gpu":
            _check(_abi.lib().qbxg_plan_create_gpu(C.byref(self._c_cfg), C.byref(self._c_geom),
                                                   1 if gpu_lists else 0, C.byref(self.handle)))
        else:
            raise ValueError("Plan: device must be 'host' or 'gpu'")
        self.view = _abi.PlanView()
        _check(_abi.lib().qbxg_plan_view_get(self.handle, C.byref(self.view)))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _abi.lib().qbxg_plan_destroy(h)
            self.handle = None

    # numpy copies of the tree
    def arrays(self):
        v = self.view
        nb = v.n_boxes
        out = dict(n_boxes=nb, n_levels=v.n_levels, root_center=np.array(v.root_center[:]), root_radius=v.root_radius,
                   box_center=_arr(v.box_center, 3 * nb, np.float64).reshape(-1, 3),
                   box_radius=_arr(v.box_radius, nb, np.float64), box_level=_arr(v.box_level, nb, np.int32),
                   box_parent=_arr(v.box_parent, nb, np.int32), child_starts=_arr(v.child_starts, nb + 1, np.int32),
                   box_flags=_arr(v.box_flags, nb, np.uint8))
        out["children"] = _arr(v.children, int(out["child_starts"][-1]), np.int32)
        out["level_starts"] = _arr(v.level_starts, v.n_levels + 1, np.int32)
        out["level_boxes"] = _arr(v.level_boxes, nb, np.int32)
        for role in ("src", "ctr", "tgt"):
            for kind in ("own_start", "own_count", "sub_start", "sub_count"):
                nm = f"{role}_{kind}"
                out[nm] = _arr(getattr(v, nm), nb, np.int32)
        out["src_perm"] = _arr(v.src_perm, v.n_sources, np.int32)
        out["ctr_perm"] = _arr(v.ctr_perm, v.n_centers, np.int32)
        out["tgt_perm"] = _arr(v.tgt_perm, v.n_conv_targets, np.int32)
        return out

    def list_csr(self, k: int):
        v = self.view
        starts = _arr(v.list_starts[k], v.n_boxes + 1, np.int64)
        boxes = _arr(v.list_boxes[k], int(starts[-1]), np.int32)
        return starts, boxes

    def list_hashes(self):
        return {name: int(self.view.list_hash[k]) for k, name in enumerate(_abi.LIST_NAMES)}

    def ledger(self) -> dict:
        L = _abi.Ledger()
        _check(_abi.lib().qbxg_plan_ledger(self.handle, C.byref(L)))
        d = {f: getattr(L, f) for f, _ in L._fields_}
        d["modeled"] = dict(zip(_abi.LIST_NAMES, L.modeled[:]))
        d["entries"] = dict(zip(_abi.LIST_NAMES, L.entries[:]))
        return d


class Locator:
    """Target association (Algorithm 3; spec associate_targets,
    SPEC.md:296-304) and area queries (Algorithm 5; spec
    area_query) on the GPU, over the tree of ``plan`` (built from
    the sources and centres of ``geom``).  ``danger_radius[s]`` is r_danger of
    source s; ``center_side`` (int8 per centre, optional) enables ``side_pref``."""

    def __init__(self, plan: "Plan", geom: Geometry, danger_radius, center_side=None):
        self.plan = plan
        self._c_geom = geom.to_c()
        self._danger = np.ascontiguousarray(danger_radius, dtype=np.float64)
        if self._danger.shape != (geom.n_sources,):
            raise ValueError("danger_radius must have one entry per source")
        cs = None if center_side is None else np.ascontiguousarray(center_side, dtype=np.int8)
        if cs is not None and cs.shape != (geom.n_centers,):
            raise ValueError("center_side must have one entry per centre")
        self.handle = C.c_void_p()
        _check(_abi.lib().qbxg_locator_create(plan.handle, C.byref(self._c_geom), _ptr(self._danger),
                                              None if cs is None else cs.ctypes.data, C.byref(self.handle)))

    def close(self):
        if getattr(self, "handle", None):
            _abi.lib().qbxg_locator_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()

    def associate(self, target_pos, eps_ta: float = 0.0, side_pref=None):
        """-> (association int32[n]: centre id / -1 conventional / -2 flagged, n_flagged)."""
        t = np.ascontiguousarray(target_pos, dtype=np.float64).reshape(-1, 3)
        sp = None if side_pref is None else np.ascontiguousarray(side_pref, dtype=np.int8)
        if sp is not None and sp.shape != (len(t),):
            raise ValueError("side_pref must have one entry per target")
        out = np.empty(len(t), dtype=np.int32)
        nf = C.c_int64(0)
        _check(_abi.lib().qbxg_associate_targets(self.handle, len(t), _ptr(t), float(eps_ta),
                                                 None if sp is None else sp.ctypes.data,
                                                 out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nf)))
        return out, int(nf.value)

    def associate_device(self, n: int, d_target_pos: int, eps_ta: float, d_side_pref: int | None, d_out: int,
                         d_n_flagged: int, stream: int | None = None):
        _check(_abi.lib().qbxg_associate_targets_device(self.handle, n, d_target_pos, float(eps_ta), d_side_pref,
                                                        d_out, d_n_flagged, stream))

    def area_query(self, centers, radii):
        """-> (starts int64[n+1], leaves int32): leaf box ids meeting each closed l-inf ball."""
        c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
        r = np.ascontiguousarray(radii, dtype=np.float64)
        if r.shape != (len(c),):
            raise ValueError("one radius per query centre")
        starts = np.zeros(len(c) + 1, dtype=np.int64)
        i64 = C.POINTER(C.c_int64)
        _check(_abi.lib().qbxg_area_query(self.handle, len(c), _ptr(c), _ptr(r), starts.ctypes.data_as(i64), None,
                                          0))
        leaves = np.zeros(max(1, int(starts[-1])), dtype=np.int32)
        _check(_abi.lib().qbxg_area_query(self.handle, len(c), _ptr(c), _ptr(r), starts.ctypes.data_as(i64),
                                          leaves.ctypes.data_as(C.POINTER(C.c_int32)), len(leaves)))
        return starts, leaves[:int(starts[-1])]


def danger_radius_of(geom: Geometry):
    """Per-source danger radius of the procedural configs: the expansion radius
    r = 0.5 sqrt(area) of the source's triangle (the radius the volume-target
    filter of BASELINE config 2 uses), read off centre 2s (csrc/host/geometry.cpp)."""
    return np.ascontiguousarray(geom.center_radius[0::2], dtype=np.float64)


def build_plan(cfg: FmmConfig, geom: Geometry) -> Plan:
    return Plan(cfg, geom)


# --------------------------------------------------------------------------- device engine
class FmmEngine:
    """One GPU's QBX-FMM apply (qbxg_create / qbxg_apply)."""

    def __init__(self, cfg: FmmConfig, geom: Geometry, plan: Plan | None = None, device: int = 0,
                 shard: tuple[int, int] | None = None):
        """shard=(n_ranks, rank): this process's part of a Morton-range sharded apply."""
        self.cfg = cfg
        self.geom = geom
        self.plan = plan if plan is not None else Plan(cfg, geom)
        self._c_cfg = cfg.to_c()
        self._c_geom = geom.to_c()
        self.handle = C.c_void_p()
        self.shard = shard
        if shard is None:
            _check(_abi.lib().qbxg_create(C.byref(self._c_cfg), C.byref(self._c_geom), self.plan.handle, device,
                                          C.byref(self.handle)))
        else:
            _check(_abi.lib().qbxg_create_sharded(C.byref(self._c_cfg), C.byref(self._c_geom), self.plan.handle,
                                                  device, shard[0], shard[1], C.byref(self.handle)))
        self.timings = _abi.Timings()

    # ---- sharded driving (multi-GPU)
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_abi.lib().qbxg_nccl_unique_id(buf))
        return buf.raw

    def attach_nccl(self, uid: bytes):
        _check(_abi.lib().qbxg_nccl_attach(self.handle, C.c_char_p(uid)))

    def apply_phase(self, phase: int, d_weights: int | None, d_dipoles: int | None, d_pot: int | None,
                    d_coeffs: int | None = None, stream: int | None = None):
        _check(_abi.lib().qbxg_apply_phase(self.handle, phase, C.c_void_p(d_weights or 0),
                                           C.c_void_p(d_dipoles or 0), C.c_void_p(d_pot or 0),
                                           C.c_void_p(d_coeffs or 0), C.c_void_p(stream or 0)))

    def multipole_buffer(self):
        ptr = C.c_void_p()
        row = C.c_int64()
        n = self.shard[0] if self.shard else 1
        cuts = (C.c_int32 * (n + 1))()
        _check(_abi.lib().qbxg_multipole_buffer(self.handle, C.byref(ptr), C.byref(row), cuts))
        return ptr.value, row.value, list(cuts)


    def close(self):
        if getattr(self, "handle", None):
            _abi.lib().qbxg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()

    def apply(self, weights, dipoles=None, want_centers=False):
        w = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
        m = None if dipoles is None else np.ascontiguousarray(dipoles, dtype=np.float64).reshape(-1)
        ns = self.geom.n_sources
        # SourceEnsemble::validate (kernels.cpp:27-38): sizes are checked before any copy
        if w.size != ns:
            raise ValueError(f"apply: {w.size} weights for {ns} sources")
        if m is not None and m.size != 3 * ns:
            raise ValueError(f"apply: {m.size // 3} dipole moments for {ns} sources")
        if m is None and self.cfg.kernel == _abi.KERNEL_LAPLACE_SL_DL:
            raise ValueError("apply: Laplace SL+DL requires dipole moments")
        pot = np.empty(self.geom.n_targets, dtype=np.float64)
        coeffs = np.empty(self.geom.n_centers * 2 * self.cfg.kq, dtype=np.float64) if want_centers else None
        _check(_abi.lib().qbxg_apply(self.handle, _ptr(w), _ptr(m), _ptr(pot), _ptr(coeffs), C.byref(self.timings)))
        if want_centers:
            c = coeffs.reshape(self.geom.n_centers, self.cfg.kq, 2)
            return pot, c[..., 0] + 1j * c[..., 1]
        return pot

    def apply_complex(self, weights, dipoles=None, want_centers=False):
        """Helmholtz single layer (kernel 2) or single + double layer (kernel 3): complex
        weights (N_S,) and, for kernel 3, complex dipole moments (N_S, 3) in; complex
        potentials out; centre locals (N_C, (q+1)^2) in the internal basis (include/qbxg.h)."""
        w = np.ascontiguousarray(weights, dtype=np.complex128).reshape(-1)
        if w.shape[0] != self.geom.n_sources:
            raise ValueError("apply_complex: weights do not match the geometry")
        m = None
        if dipoles is not None:
            m = np.ascontiguousarray(dipoles, dtype=np.complex128).reshape(-1)
            if m.shape[0] != 3 * self.geom.n_sources:
                raise ValueError("apply_complex: dipoles must have shape (n_sources, 3)")
        pot = np.empty(2 * self.geom.n_targets, dtype=np.float64)
        kq = (self.cfg.p_qbx + 1) ** 2
        cc = np.empty(2 * self.geom.n_centers * kq, dtype=np.float64) if want_centers else None
        _check(_abi.lib().qbxg_apply_complex(self.handle, _ptr(w.view(np.float64)),
                                             _ptr(None if m is None else m.view(np.float64)), _ptr(pot), _ptr(cc),
                                             C.byref(self.timings)))
        pot = pot.view(np.complex128)
        if want_centers:
            return pot, cc.view(np.complex128).reshape(self.geom.n_centers, kq)
        return pot

    def set_overlap(self, enable: bool):
        """Near field on a second stream beside M2L/P2L/L2L (default on); bitwise-identical results."""
        _check(_abi.lib().qbxg_set_overlap(self.handle, 1 if enable else 0))

    def apply_batch(self, weights, dipoles=None, want_centers=False):
        """Several densities at once (leading batch dimension): weights (R, N_S),
        dipoles (R, N_S, 3); returns potentials (R, N_T) [and centre coefficients
        (R, N_C, K_q) complex].  Same results as R calls of ``apply``."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.ndim != 2 or w.shape[1] != self.geom.n_sources:
            raise ValueError("apply_batch: weights must have shape (n_rhs, n_sources)")
        R = w.shape[0]
        m = None
        if dipoles is not None:
            m = np.ascontiguousarray(dipoles, dtype=np.float64).reshape(R, self.geom.n_sources, 3)
        pot = np.empty((R, self.geom.n_targets), dtype=np.float64)
        coeffs = np.empty((R, self.geom.n_centers, self.cfg.kq, 2), dtype=np.float64) if want_centers else None
        _check(_abi.lib().qbxg_apply_batch(self.handle, R, _ptr(w), _ptr(m), _ptr(pot), _ptr(coeffs),
                                           C.byref(self.timings)))
        if want_centers:
            return pot, coeffs[..., 0] + 1j * coeffs[..., 1]
        return pot

    def apply_batch_device(self, n_rhs: int, d_weights: int, d_dipoles: int | None, d_pot: int,
                           d_coeffs: int | None = None, stream: int | None = None):
        """Device-pointer batch apply (rhs-major arrays, see include/qbxg.h)."""
        _check(_abi.lib().qbxg_apply_batch_device(self.handle, int(n_rhs), C.c_void_p(d_weights),
                                                  C.c_void_p(d_dipoles or 0), C.c_void_p(d_pot),
                                                  C.c_void_p(d_coeffs or 0), C.c_void_p(stream or 0),
                                                  C.byref(self.timings)))

    def apply_device(self, d_weights: int, d_dipoles: int | None, d_pot: int, d_coeffs: int | None = None,
                     stream: int | None = None):
        """Device pointers (ints, e.g. torch tensor.data_ptr()) in original ordering."""
        _check(_abi.lib().qbxg_apply_device(self.handle, C.c_void_p(d_weights), C.c_void_p(d_dipoles or 0),
                                            C.c_void_p(d_pot), C.c_void_p(d_coeffs or 0), C.c_void_p(stream or 0),
                                            C.byref(self.timings)))

    def last_timings(self):
        t = self.timings
        return dict(zip(_abi.TIMER_NAMES, t.ms[:])), int(t.kernel_launches), int(t.h2d_bytes), int(t.d2h_bytes)




def exchange_local(engines):
    """Multipole exchange between sharded engines living in one process (device copies)."""
    arr = (C.c_void_p * len(engines))(*[e.handle for e in engines])
    _check(_abi.lib().qbxg_exchange_local(arr, len(engines)))


def exchange_results_local(engines, d_pots, d_coeffs=None):
    """Result all-gather between sharded engines in one process (device copies): after
    phase 2, every d_pots[r] (device pointer, n_targets doubles) holds all potentials."""
    n = len(engines)
    arr = (C.c_void_p * n)(*[e.handle for e in engines])
    pp = (C.c_void_p * n)(*d_pots)
    cp = (C.c_void_p * n)(*d_coeffs) if d_coeffs is not None else None
    _check(_abi.lib().qbxg_result_exchange_local(arr, n, pp, cp))


def plan_shard(plan: "Plan", n_ranks: int, rank: int):
    """Rank's box range cuts (n_ranks+1) and per-box role bits (_abi.SHARD_*)."""
    cuts = np.zeros(n_ranks + 1, dtype=np.int32)
    mask = np.zeros(plan.view.n_boxes, dtype=np.uint8)
    _check(_abi.lib().qbxg_plan_shard(plan.handle, n_ranks, rank, cuts.ctypes.data_as(_i32p),
                                      mask.ctypes.data_as(C.POINTER(C.c_uint8))))
    return cuts, mask

def execute(geom: Geometry, weights, dipoles, cfg: FmmConfig, want_centers=False, device=0):
    """SPEC.md:424 execute(bundle, density, FmmConfig) -> (potentials, ledger)."""
    plan = Plan(cfg, geom)
    eng = FmmEngine(cfg, geom, plan, device)
    try:
        out = eng.apply(weights, dipoles, want_centers=want_centers)
    finally:
        eng.close()
    return out, plan.ledger()


def adequately_separated(kind: str, a_center, a_half: float, b_center, b_half: float, t_f: float) -> bool:
    """SPEC.md:370-378 adequately_separated: kind "box_vs_tcr" (a < TCR(b)) or
    "tcr_vs_box" (TCR(a) < b); the predicate the host list builder uses."""
    k = {"box_vs_tcr": 0, "tcr_vs_box": 1}[kind]
    ca = np.ascontiguousarray(a_center, dtype=np.float64)
    cb = np.ascontiguousarray(b_center, dtype=np.float64)
    out = C.c_int32()
    _check(_abi.lib().qbxg_adequately_separated(k, _ptr(ca), float(a_half), _ptr(cb), float(b_half), float(t_f),
                                                C.byref(out)))
    return bool(out.value)


def direct_sum(sources: SourceEnsemble, targets: TargetSet) -> np.ndarray:
    """GPU counterpart of qbx::direct_sum (kernels.cpp:46-73)."""
    pot = np.empty(targets.size(), dtype=np.float64)
    m = sources.dipole_moments
    _check(_abi.lib().qbxg_direct_sum(sources.size(), _ptr(sources.positions), _ptr(sources.weights), _ptr(m),
                                      targets.size(), _ptr(targets.positions), _ptr(pot)))
    return pot


def direct_qbx(geom: Geometry, weights, dipoles=None, p_qbx: int = 5) -> np.ndarray:
    """Unaccelerated QBX on the GPU: every centre's local
    expansion from all sources, same formulas as ``FmmEngine.apply``."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    mu = None if dipoles is None else np.ascontiguousarray(dipoles, dtype=np.float64).reshape(-1, 3)
    if w.shape != (geom.n_sources,) or (mu is not None and mu.shape[0] != geom.n_sources):
        raise ValueError("direct_qbx: density shape does not match the geometry")
    pot = np.empty(geom.n_targets, dtype=np.float64)
    _check(_abi.lib().qbxg_direct_qbx(geom.n_sources, _ptr(geom.source_pos), _ptr(w), _ptr(mu), geom.n_centers,
                                      _ptr(geom.center_pos), _ptr(geom.center_radius), geom.n_targets,
                                      _ptr(geom.target_pos), _ptr(geom.association, C.c_int32),
                                      int(p_qbx), _ptr(pot)))
    return pot


def _as_cplx(w, n):
    w = np.ascontiguousarray(w, dtype=np.complex128).reshape(-1)
    if w.shape[0] != n:
        raise ValueError("weights do not match the number of sources")
    return w.view(np.float64)


def _as_cplx_dip(dipoles, n):
    if dipoles is None:
        return None
    m = np.ascontiguousarray(dipoles, dtype=np.complex128).reshape(-1)
    if m.shape[0] != 3 * n:
        raise ValueError("dipoles must have shape (n_sources, 3)")
    return m.view(np.float64)


def helm_direct_sum(k: float, source_pos, weights, target_pos, dipoles=None) -> np.ndarray:
    """Helmholtz G_k = e^{ik r}/(4 pi r) summed directly on the GPU (complex):
    sum_s w_s G_k(t, s) [+ m_s . grad_s G_k(t, s) with complex dipoles (N_S, 3)]."""
    pos = np.ascontiguousarray(source_pos, dtype=np.float64).reshape(-1, 3)
    tpos = np.ascontiguousarray(target_pos, dtype=np.float64).reshape(-1, 3)
    wc = _as_cplx(weights, pos.shape[0])
    mc = _as_cplx_dip(dipoles, pos.shape[0])
    out = np.empty(2 * tpos.shape[0], dtype=np.float64)
    _check(_abi.lib().qbxg_helm_direct_sum(float(k), pos.shape[0], _ptr(pos), _ptr(wc), _ptr(mc), tpos.shape[0],
                                           _ptr(tpos), _ptr(out)))
    return out.view(np.complex128)


def helm_direct_qbx(k: float, geom: Geometry, weights, p_qbx: int = 5, dipoles=None) -> np.ndarray:
    """Unaccelerated QBX for the Helmholtz single (+ double) layer on the GPU (complex potentials)."""
    wc = _as_cplx(weights, geom.n_sources)
    mc = _as_cplx_dip(dipoles, geom.n_sources)
    out = np.empty(2 * geom.n_targets, dtype=np.float64)
    _check(_abi.lib().qbxg_helm_direct_qbx(float(k), geom.n_sources, _ptr(geom.source_pos), _ptr(wc), _ptr(mc),
                                           geom.n_centers, _ptr(geom.center_pos), geom.n_targets,
                                           _ptr(geom.target_pos), _ptr(geom.association, C.c_int32), int(p_qbx),
                                           _ptr(out)))
    return out.view(np.complex128)


def device_count() -> int:
    n = C.c_int32(0)
    _check(_abi.lib().qbxg_device_count(C.byref(n)))
    return n.value


def measure_fp64_peak(device: int = 0) -> float:
    """Measured DFMA throughput (TFLOP/s) of the GPU: the fp64 roofline denominator."""
    v = C.c_double(0)
    _check(_abi.lib().qbxg_measure_fp64_peak(device, C.byref(v)))
    return v.value


def measure_dmma_peak(device: int = 0) -> float:
    """Measured fp64 tensor-pipe (DMMA) throughput (TFLOP/s)."""
    v = C.c_double(0)
    _check(_abi.lib().qbxg_measure_dmma_peak(device, C.byref(v)))
    return v.value
