"""ctypes mirror of include/qbxg.h (the C ABI).  Plumbing only: every compute
call goes through libqbxg.so; nothing here computes potentials."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqbxg.so")

NUM_LISTS = 6
NUM_TIMERS = 12
LIST_NAMES = ("U", "V", "W_close", "W_far", "X_close", "X_far")
TIMER_NAMES = ("h2d", "p2m", "m2m", "near", "m2l", "wfar", "p2l", "l2l", "l2qbxl", "eval", "d2h", "total")

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_DOMAIN = 2
ERR_CUDA = 3
ERR_NCCL = 4
ERR_INTERNAL = 5
ERR_NO_DEVICE = 6

KERNEL_LAPLACE_SL = 0
KERNEL_LAPLACE_SL_DL = 1
KERNEL_HELMHOLTZ_SL = 2
KERNEL_HELMHOLTZ_SL_DL = 3

BOX_TARGET, BOX_TARGET_ANCESTOR, BOX_HAS_SOURCES, BOX_LEAF = 1, 2, 4, 8

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class Config(C.Structure):
    _fields_ = [("p_fmm", C.c_int32), ("p_qbx", C.c_int32), ("t_f", C.c_double), ("n_max", C.c_int32),
                ("kernel", C.c_int32), ("helmholtz_k", C.c_double), ("w_far_demote", C.c_int32),
                ("level_restrict", C.c_int32)]


class Geometry(C.Structure):
    _fields_ = [("n_sources", C.c_int64), ("source_pos", _dp), ("n_centers", C.c_int64),
                ("center_pos", _dp), ("center_radius", _dp), ("n_targets", C.c_int64),
                ("target_pos", _dp), ("association", _i32p)]


class GeometrySpec(C.Structure):
    _fields_ = [("surface", C.c_int32), ("level", C.c_int32), ("nu", C.c_int32), ("nv", C.c_int32),
                ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("spacing", C.c_double),
                ("density", C.c_int32), ("reserved", C.c_int32), ("n_volume_targets", C.c_int64),
                ("volume_halfwidth", C.c_double), ("seed", C.c_uint64)]


class GeneratedView(C.Structure):
    _fields_ = [("n_triangles", C.c_int64), ("n_sources", C.c_int64), ("source_pos", _dp),
                ("source_normal", _dp), ("quad_weight", _dp), ("density", _dp),
                ("density_is_complex", C.c_int32), ("n_centers", C.c_int64), ("center_pos", _dp),
                ("center_radius", _dp), ("n_targets", C.c_int64), ("target_pos", _dp),
                ("association", _i32p), ("n_volume_drawn", C.c_int64)]


class PlanView(C.Structure):
    _fields_ = [("n_boxes", C.c_int32), ("n_levels", C.c_int32), ("root_center", C.c_double * 3),
                ("root_radius", C.c_double), ("box_center", _dp), ("box_radius", _dp),
                ("box_level", _i32p), ("box_parent", _i32p), ("child_starts", _i32p), ("children", _i32p),
                ("level_starts", _i32p), ("level_boxes", _i32p),
                ("src_own_start", _i32p), ("src_own_count", _i32p), ("src_sub_start", _i32p), ("src_sub_count", _i32p),
                ("ctr_own_start", _i32p), ("ctr_own_count", _i32p), ("ctr_sub_start", _i32p), ("ctr_sub_count", _i32p),
                ("tgt_own_start", _i32p), ("tgt_own_count", _i32p), ("tgt_sub_start", _i32p), ("tgt_sub_count", _i32p),
                ("n_sources", C.c_int64), ("n_centers", C.c_int64), ("n_conv_targets", C.c_int64),
                ("n_targets", C.c_int64), ("src_perm", _i32p), ("ctr_perm", _i32p), ("tgt_perm", _i32p),
                ("box_flags", _u8p), ("list_starts", _i64p * NUM_LISTS), ("list_boxes", _i32p * NUM_LISTS),
                ("list_hash", C.c_uint64 * NUM_LISTS), ("build_seconds_tree", C.c_double),
                ("build_seconds_lists", C.c_double)]


class Ledger(C.Structure):
    _fields_ = [("modeled", C.c_double * NUM_LISTS), ("modeled_total", C.c_double),
                ("entries", C.c_int64 * NUM_LISTS), ("pairs_qbx_near", C.c_int64), ("pairs_p2p_near", C.c_int64),
                ("pairs_wfar_centre", C.c_int64), ("pairs_wfar_target", C.c_int64),
                ("pairs_xfar_source", C.c_int64), ("n_m2m", C.c_int64), ("n_l2l", C.c_int64),
                ("n_p2m_sources", C.c_int64), ("n_l2qbxl_centres", C.c_int64), ("n_l2p_targets", C.c_int64),
                ("n_qbxl2p_targets", C.c_int64)]


class Timings(C.Structure):
    _fields_ = [("ms", C.c_double * NUM_TIMERS), ("kernel_launches", C.c_int32),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64)]


EXPORTED_SYMBOLS = (
    "qbxg_geometry_spec_for_config", "qbxg_geometry_generate", "qbxg_geometry_view", "qbxg_geometry_destroy",
    "qbxg_plan_create", "qbxg_plan_view_get", "qbxg_plan_ledger", "qbxg_plan_destroy",
    "qbxg_create", "qbxg_apply", "qbxg_apply_device", "qbxg_destroy", "qbxg_direct_sum",
    "qbxg_last_error", "qbxg_device_count", "qbxg_version", "qbxg_measure_fp64_peak",
    "qbxg_measure_dmma_peak", "qbxg_plan_shard", "qbxg_create_sharded", "qbxg_apply_phase",
    "qbxg_multipole_buffer", "qbxg_exchange_local", "qbxg_result_exchange_local", "qbxg_nccl_unique_id", "qbxg_nccl_attach",
    "qbxg_direct_qbx", "qbxg_apply_batch", "qbxg_apply_batch_device", "qbxg_set_overlap", "qbxg_helm_direct_sum", "qbxg_helm_direct_qbx",
    "qbxg_apply_complex", "qbxg_locator_create", "qbxg_associate_targets", "qbxg_associate_targets_device",
    "qbxg_area_query", "qbxg_locator_destroy", "qbxg_plan_create_gpu", "qbxg_adequately_separated",
)

SHARD_OWN, SHARD_SUBTREE, SHARD_STRADDLE, SHARD_DOWN = 1, 2, 4, 8


def _declare(lib):
    P = C.POINTER
    sig = {
        "qbxg_geometry_spec_for_config": ([C.c_int32, C.c_int32, C.c_uint64, P(GeometrySpec)], C.c_int),
        "qbxg_geometry_generate": ([P(GeometrySpec), P(C.c_void_p)], C.c_int),
        "qbxg_geometry_view": ([C.c_void_p, P(GeneratedView)], C.c_int),
        "qbxg_geometry_destroy": ([C.c_void_p], None),
        "qbxg_plan_create": ([P(Config), P(Geometry), P(C.c_void_p)], C.c_int),
        "qbxg_plan_create_gpu": ([P(Config), P(Geometry), C.c_int32, P(C.c_void_p)], C.c_int),
        "qbxg_plan_view_get": ([C.c_void_p, P(PlanView)], C.c_int),
        "qbxg_plan_ledger": ([C.c_void_p, P(Ledger)], C.c_int),
        "qbxg_plan_destroy": ([C.c_void_p], None),
        "qbxg_create": ([P(Config), P(Geometry), C.c_void_p, C.c_int32, P(C.c_void_p)], C.c_int),
        "qbxg_apply": ([C.c_void_p, _dp, _dp, _dp, _dp, P(Timings)], C.c_int),
        "qbxg_apply_device": ([C.c_void_p] * 6 + [P(Timings)], C.c_int),
        "qbxg_set_overlap": ([C.c_void_p, C.c_int32], C.c_int),
        "qbxg_apply_complex": ([C.c_void_p, _dp, _dp, _dp, _dp, P(Timings)], C.c_int),
        "qbxg_helm_direct_sum": ([C.c_double, C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, _dp], C.c_int),
        "qbxg_helm_direct_qbx": ([C.c_double, C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, C.c_int64, _dp, _i32p, C.c_int32,
                                  _dp], C.c_int),
        "qbxg_apply_batch": ([C.c_void_p, C.c_int32, _dp, _dp, _dp, _dp, P(Timings)], C.c_int),
        "qbxg_apply_batch_device": ([C.c_void_p, C.c_int32] + [C.c_void_p] * 5 + [P(Timings)], C.c_int),
        "qbxg_destroy": ([C.c_void_p], C.c_int),
        "qbxg_direct_sum": ([C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, _dp], C.c_int),
        "qbxg_direct_qbx": ([C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, _dp, C.c_int64, _dp, _i32p, C.c_int32, _dp],
                            C.c_int),
        "qbxg_last_error": ([], C.c_char_p),
        "qbxg_device_count": ([P(C.c_int32)], C.c_int),
        "qbxg_version": ([], C.c_char_p),
        "qbxg_measure_fp64_peak": ([C.c_int32, P(C.c_double)], C.c_int),
        "qbxg_measure_dmma_peak": ([C.c_int32, P(C.c_double)], C.c_int),
        "qbxg_plan_shard": ([C.c_void_p, C.c_int32, C.c_int32, _i32p, _u8p], C.c_int),
        "qbxg_create_sharded": ([P(Config), P(Geometry), C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                 P(C.c_void_p)], C.c_int),
        "qbxg_apply_phase": ([C.c_void_p, C.c_int32] + [C.c_void_p] * 5, C.c_int),
        "qbxg_multipole_buffer": ([C.c_void_p, P(C.c_void_p), _i64p, _i32p], C.c_int),
        "qbxg_exchange_local": ([P(C.c_void_p), C.c_int32], C.c_int),
        "qbxg_result_exchange_local": ([P(C.c_void_p), C.c_int32, P(C.c_void_p), P(C.c_void_p)], C.c_int),
        "qbxg_nccl_unique_id": ([C.c_char_p], C.c_int),
        "qbxg_nccl_attach": ([C.c_void_p, C.c_char_p], C.c_int),
        "qbxg_locator_create": ([C.c_void_p, P(Geometry), _dp, C.c_void_p, P(C.c_void_p)], C.c_int),
        "qbxg_associate_targets": ([C.c_void_p, C.c_int64, _dp, C.c_double, C.c_void_p, _i32p, _i64p], C.c_int),
        "qbxg_associate_targets_device": ([C.c_void_p, C.c_int64, C.c_void_p, C.c_double] + [C.c_void_p] * 4,
                                          C.c_int),
        "qbxg_area_query": ([C.c_void_p, C.c_int64, _dp, _dp, _i64p, _i32p, C.c_int64], C.c_int),
        "qbxg_locator_destroy": ([C.c_void_p], None),
        "qbxg_adequately_separated": ([C.c_int32, _dp, C.c_double, _dp, C.c_double, C.c_double, _i32p], C.c_int),
    }
    for name, (args, res) in sig.items():
        if not hasattr(lib, name):
            continue  # reported by missing_symbols()
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def missing_symbols(l=None):
    l = l or lib()
    return [n for n in EXPORTED_SYMBOLS if not hasattr(l, n)]


_lib = None


def lib(path: str | None = None):
    """Load libqbxg.so (built in-tree by __graft_entry__.build / make)."""
    global _lib
    if _lib is None or path is not None:
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(f"libqbxg.so not built ({p}); run `make -C paper_1805_06106_b200/csrc`")
        _lib = _declare(C.CDLL(p))
    return _lib
