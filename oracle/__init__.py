"""ORACLE -- test infrastructure only.

ctypes loader for oracle/liboracle.so (CPU restatement of the QBX-FMM path)
and oracle/_ref/libqbxref.so (the reference's own qbx::direct_sum compiled from
/root/reference/proj/src/kernels.cpp).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU legs may import this package; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqbxref.so")

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_o = None
_r = None


def lib():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.qbxo_last_error.restype = C.c_char_p
        L.qbxo_sph_harm.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp]
        L.qbxo_form_expansion.argtypes = [C.c_int, C.c_int64, _dp, _dp, _dp, _dp, C.c_int, _dp]
        L.qbxo_eval_expansion.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, _dp]
        L.qbxo_translate.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, C.c_int, _dp]
        L.qbxo_form_internal.argtypes = [C.c_int, C.c_int64, _dp, _dp, _dp, _dp, C.c_int, _dp]
        L.qbxo_eval_internal.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, _dp]
        L.qbxo_execute.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _i32p, _dp, _dp,
                                   _dp, _dp, _dp]
        L.qbxo_direct_qbx.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, _dp, C.c_int64, _dp, _i32p, C.c_int,
                                      _dp]
        L.qbxo_adequately_separated.argtypes = [C.c_int, _dp, C.c_double, _dp, C.c_double, C.c_double]
        L.qbxo_adequately_separated.restype = C.c_int
        L.qbxo_helm_last_error.restype = C.c_char_p
        L.qbxo_helm_ylm.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.qbxo_helm_bessel.argtypes = [C.c_int, C.c_double, _dp, _dp]
        L.qbxo_helm_gaunt.argtypes = [C.c_int] * 5 + [_dp]
        L.qbxo_helm_form.argtypes = [C.c_int, C.c_double, C.c_int64, _dp, _dp, _dp, _dp, C.c_int, _dp]
        L.qbxo_helm_eval.argtypes = [C.c_int, C.c_double, _dp, C.c_int, _dp, _dp, _dp]
        L.qbxo_helm_translate.argtypes = [C.c_int, C.c_double, _dp, C.c_int, _dp, _dp, C.c_int, _dp]
        L.qbxo_helm_direct_sum.argtypes = [C.c_double, C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, _dp]
        L.qbxo_helm_direct_qbx.argtypes = [C.c_double, C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, C.c_int64, _dp, _i32p,
                                           C.c_int, _dp]
        L.qbxo_helm_execute.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, _i32p, _dp, _dp, _dp,
                                        _dp]
        L.oracle_associate.argtypes = [C.c_int64, _dp, _dp, C.c_int64, _dp, _dp, C.c_void_p, C.c_int64, _dp,
                                       C.c_double, C.c_void_p, _i32p, _i64p]
        L.oracle_area_query.argtypes = [C.c_int32, _dp, _dp, _i32p, C.c_int64, _dp, _dp, _i64p, _i64p, _i32p]
        L.qbxo_lists_brute.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_int64, _i64p * 6, _i32p * 6, _i64p]
        _o = L
    return _o


def ref_lib():
    """The reference's own direct_sum (oracle/_ref).  None when not built."""
    global _r
    if _r is None:
        if not os.path.exists(REF_SO):
            try:
                build()
            except Exception:
                pass
        if not os.path.exists(REF_SO):
            return None
        L = C.CDLL(REF_SO)
        L.qbxref_last_error.restype = C.c_char_p
        L.qbxref_direct_sum.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_int64, _dp, _dp]
        L.qbxref_laplace_green.argtypes = [_dp, _dp, _dp]
        L.qbxref_laplace_dipole.argtypes = [_dp, _dp, _dp, _dp]
        _r = L
    return _r


def _p(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_dp)


def _chk(st, L):
    if st == 0:
        return
    msg = L.qbxo_last_error().decode() if L is _o else L.qbxref_last_error().decode()
    if st == 1:
        raise ValueError(msg)
    if st == 2:
        raise ArithmeticError(msg)
    raise RuntimeError(msg)


def sph_harm(n, m, theta, phi):
    out = np.zeros(2)
    _chk(lib().qbxo_sph_harm(n, m, theta, phi, out.ctypes.data_as(_dp)), _o)
    return complex(out[0], out[1])


def form_expansion(kind, pos, w, mu, center, p):
    """Paper normalisation (Eq. (5)/(10)); kind 'multipole' | 'local'; full table n^2+n+m."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    w = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
    out = np.zeros(2 * (p + 1) ** 2)
    _chk(lib().qbxo_form_expansion(0 if kind == "multipole" else 1, pos.shape[0], _p(pos), _p(w),
                                   _p(None if mu is None else np.asarray(mu).reshape(-1, 3)), _p(center), p,
                                   out.ctypes.data_as(_dp)), _o)
    return out[0::2] + 1j * out[1::2]


def eval_expansion(kind, coeffs, p, center, t):
    c = np.zeros(2 * (p + 1) ** 2)
    c[0::2] = np.real(coeffs)
    c[1::2] = np.imag(coeffs)
    out = np.zeros(1)
    _chk(lib().qbxo_eval_expansion(0 if kind == "multipole" else 1, _p(c), p, _p(center), _p(t),
                                   out.ctypes.data_as(_dp)), _o)
    return float(out[0])


def form_internal(kind, pos, w, mu, center, p):
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(2 * (p + 1) ** 2)
    _chk(lib().qbxo_form_internal(0 if kind == "multipole" else 1, pos.shape[0], _p(pos), _p(w),
                                  _p(None if mu is None else np.asarray(mu).reshape(-1, 3)), _p(center), p,
                                  out.ctypes.data_as(_dp)), _o)
    return out[0::2] + 1j * out[1::2]


def eval_internal(kind, coeffs, p, center, t):
    c = np.zeros(2 * (p + 1) ** 2)
    c[0::2] = np.real(coeffs)
    c[1::2] = np.imag(coeffs)
    out = np.zeros(1)
    _chk(lib().qbxo_eval_internal(0 if kind == "multipole" else 1, _p(c), p, _p(center), _p(t),
                                  out.ctypes.data_as(_dp)), _o)
    return float(out[0])


def translate(kind, coeffs, p, c, C_, q):
    k = {"M2M": 0, "M2L": 1, "L2L": 2}[kind]
    a = np.zeros(2 * (p + 1) ** 2)
    a[0::2] = np.real(coeffs)
    a[1::2] = np.imag(coeffs)
    out = np.zeros(2 * (q + 1) ** 2)
    _chk(lib().qbxo_translate(k, _p(a), p, _p(c), _p(C_), q, out.ctypes.data_as(_dp)), _o)
    return out[0::2] + 1j * out[1::2]


def execute(plan, geom, weights, dipoles=None, want_centers=False):
    """Stages 2-9 on the CPU over the product's host tree and lists (plan)."""
    cfg = plan.cfg
    pot = np.empty(geom.n_targets)
    kq = cfg.kq
    coeffs = np.empty(geom.n_centers * 2 * kq) if want_centers else None
    stages = np.zeros(8)
    keep = [np.ascontiguousarray(weights, dtype=np.float64), None if dipoles is None else
            np.ascontiguousarray(dipoles, dtype=np.float64)]
    _chk(lib().qbxo_execute(C.addressof(plan.view), cfg.p_fmm, cfg.p_qbx, cfg.t_f, _p(geom.source_pos),
                            _p(geom.center_pos), _p(geom.center_radius), _p(geom.target_pos),
                            geom.association.ctypes.data_as(_i32p), _p(keep[0]), _p(keep[1]),
                            pot.ctypes.data_as(_dp), None if coeffs is None else coeffs.ctypes.data_as(_dp),
                            stages.ctypes.data_as(_dp)), _o)
    if want_centers:
        c = coeffs.reshape(geom.n_centers, kq, 2)
        return pot, c[..., 0] + 1j * c[..., 1], stages
    return pot, stages


def direct_qbx(geom, weights, dipoles, q):
    pot = np.empty(geom.n_targets)
    _chk(lib().qbxo_direct_qbx(geom.n_sources, _p(geom.source_pos), _p(weights), _p(dipoles), geom.n_centers,
                               _p(geom.center_pos), _p(geom.center_radius), geom.n_targets, _p(geom.target_pos),
                               geom.association.ctypes.data_as(_i32p), q, pot.ctypes.data_as(_dp)), _o)
    return pot


def lists_brute(plan):
    """Definitional lists on the plan's tree: dict name -> (starts, boxes)."""
    v = plan.view
    nb = v.n_boxes
    cap = 4 * nb * nb + 16
    starts = [np.zeros(nb + 1, dtype=np.int64) for _ in range(6)]
    boxes = [np.zeros(cap, dtype=np.int32) for _ in range(6)]
    counts = np.zeros(6, dtype=np.int64)
    sp = (_i64p * 6)(*[s.ctypes.data_as(_i64p) for s in starts])
    bp = (_i32p * 6)(*[b.ctypes.data_as(_i32p) for b in boxes])
    st = lib().qbxo_lists_brute(C.addressof(v), plan.cfg.t_f, plan.cfg.w_far_demote, cap, sp, bp,
                                counts.ctypes.data_as(_i64p))
    if st != 0:
        raise RuntimeError("lists_brute capacity exceeded")
    names = ("U", "V", "W_close", "W_far", "X_close", "X_far")
    return {names[k]: (starts[k], boxes[k][:counts[k]].copy()) for k in range(6)}


def ref_direct_sum(pos, w, mu, tpos):
    """The reference's own qbx::direct_sum (kernels.cpp:46-73) via oracle/_ref."""
    L = ref_lib()
    if L is None:
        raise RuntimeError("oracle/_ref not built")
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    tpos = np.ascontiguousarray(tpos, dtype=np.float64).reshape(-1, 3)
    out = np.empty(tpos.shape[0])
    _chk(L.qbxref_direct_sum(pos.shape[0], _p(pos), _p(w), _p(mu), tpos.shape[0], _p(tpos),
                             out.ctypes.data_as(_dp)), L)
    return out


def execute_phase(plan, geom, weights, dipoles, mask, phase, Mbuf, want_centers=False):
    """Sharded oracle step (SURVEY.md §8e harness): mask from api.plan_shard,
    phase 1 fills Mbuf (n_boxes x (p+1)^2 complex as float64 pairs), phase 2
    consumes it.  Returns (pot, centre coefficients or None) for phase 2."""
    L = lib()
    if not hasattr(L, "_phase_declared"):
        L.qbxo_execute_phase.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _i32p, _dp, _dp, _dp, _dp,
                                         C.POINTER(C.c_uint8), C.c_int, _dp]
        L._phase_declared = True
    cfg = plan.cfg
    pot = np.zeros(geom.n_targets)
    coeffs = np.zeros(geom.n_centers * 2 * cfg.kq) if want_centers else None
    w = np.ascontiguousarray(weights, dtype=np.float64)
    mu = None if dipoles is None else np.ascontiguousarray(dipoles, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    _chk(L.qbxo_execute_phase(C.addressof(plan.view), cfg.p_fmm, cfg.p_qbx, _p(geom.source_pos), _p(geom.center_pos),
                              _p(geom.center_radius), _p(geom.target_pos), geom.association.ctypes.data_as(_i32p),
                              _p(w), _p(mu), pot.ctypes.data_as(_dp),
                              None if coeffs is None else coeffs.ctypes.data_as(_dp),
                              m.ctypes.data_as(C.POINTER(C.c_uint8)), phase, Mbuf.ctypes.data_as(_dp)), _o)
    if coeffs is not None:
        c = coeffs.reshape(geom.n_centers, cfg.kq, 2)
        return pot, c[..., 0] + 1j * c[..., 1]
    return pot, None


# ---- Helmholtz single layer (helm_oracle.cpp; parity unpinned, see its header) ----
def _hchk(st):
    if st != 0:
        raise RuntimeError(lib().qbxo_helm_last_error().decode())


def _cplx(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


def helm_ylm(n, m, v):
    out = np.zeros(2)
    _hchk(lib().qbxo_helm_ylm(n, m, _p(v), out.ctypes.data_as(_dp)))
    return complex(out[0], out[1])


def helm_bessel(P, x):
    j = np.zeros(P + 1)
    h = np.zeros(2 * (P + 1))
    _hchk(lib().qbxo_helm_bessel(P, x, j.ctypes.data_as(_dp), h.ctypes.data_as(_dp)))
    return j, h.view(np.complex128)


def helm_gaunt(n, m, n2, m2, l):
    out = np.zeros(1)
    _hchk(lib().qbxo_helm_gaunt(n, m, n2, m2, l, out.ctypes.data_as(_dp)))
    return float(out[0])


def _dip(mu, n):
    """complex dipoles (n, 3) -> 6n interleaved doubles (or None)"""
    if mu is None:
        return None
    return np.ascontiguousarray(np.asarray(mu, dtype=np.complex128).reshape(n, 3)).view(np.float64).reshape(-1)


def helm_form(kind, k, pos, w, center, P, mu=None):
    """kind 0: multipole (P2M), 1: local (P2L); w complex weights, mu complex dipoles (n, 3)."""
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(2 * (P + 1) ** 2)
    _hchk(lib().qbxo_helm_form(kind, k, pos.shape[0], _p(pos), _p(_cplx(w)), _p(_dip(mu, pos.shape[0])), _p(center),
                               P, out.ctypes.data_as(_dp)))
    return out.view(np.complex128)


def helm_eval(kind, k, coeffs, P, center, t):
    out = np.zeros(2)
    _hchk(lib().qbxo_helm_eval(kind, k, _p(_cplx(coeffs)), P, _p(center), _p(t), out.ctypes.data_as(_dp)))
    return complex(out[0], out[1])


def helm_translate(kind, k, coeffs, Pin, c, C_, Pout):
    """kind 0: M2M, 1: M2L, 2: L2L."""
    out = np.zeros(2 * (Pout + 1) ** 2)
    _hchk(lib().qbxo_helm_translate(kind, k, _p(_cplx(coeffs)), Pin, _p(c), _p(C_), Pout,
                                    out.ctypes.data_as(_dp)))
    return out.view(np.complex128)


def helm_direct_sum(k, pos, w, tpos, mu=None):
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    tpos = np.ascontiguousarray(tpos, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(2 * tpos.shape[0])
    _hchk(lib().qbxo_helm_direct_sum(k, pos.shape[0], _p(pos), _p(_cplx(w)), _p(_dip(mu, pos.shape[0])),
                                     tpos.shape[0], _p(tpos),
                                     out.ctypes.data_as(_dp)))
    return out.view(np.complex128)


def helm_direct_qbx(k, geom, w, q, mu=None):
    out = np.zeros(2 * geom.n_targets)
    _hchk(lib().qbxo_helm_direct_qbx(k, geom.n_sources, _p(geom.source_pos), _p(_cplx(w)),
                                     _p(_dip(mu, geom.n_sources)), geom.n_centers,
                                     _p(geom.center_pos), geom.n_targets, _p(geom.target_pos),
                                     geom.association.ctypes.data_as(_i32p), q, out.ctypes.data_as(_dp)))
    return out.view(np.complex128)


def helm_execute(plan, geom, k, p, q, w, want_centers=False, mu=None):
    """Stages 2-9 for the Helmholtz single (+ double) layer on the host plan (same tree and
    lists); mu: complex dipole moments (N_S, 3) or None."""
    pot = np.zeros(2 * geom.n_targets)
    cc = np.zeros(2 * geom.n_centers * (q + 1) ** 2) if want_centers else None
    _hchk(lib().qbxo_helm_execute(C.addressof(plan.view), k, p, q, _p(geom.source_pos), _p(geom.center_pos),
                                  _p(geom.target_pos), geom.association.ctypes.data_as(_i32p), _p(_cplx(w)),
                                  _p(_dip(mu, geom.n_sources)), pot.ctypes.data_as(_dp), None if cc is None else cc.ctypes.data_as(_dp)))
    pot = pot.view(np.complex128)
    if want_centers:
        return pot, cc.view(np.complex128).reshape(geom.n_centers, (q + 1) ** 2)
    return pot


def _i8(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int8)


def associate_targets(source_pos, danger_radius, center_pos, center_radius, target_pos, eps_ta=0.0,
                      center_side=None, side_pref=None):
    """Algorithm 3 by brute force (oracle/assoc_brute.cpp): association int32[n_t]
    (centre id, -1 not endangered, -2 flagged) and the flagged count."""
    sp = np.ascontiguousarray(source_pos, dtype=np.float64).reshape(-1, 3)
    cp = np.ascontiguousarray(center_pos, dtype=np.float64).reshape(-1, 3)
    tp = np.ascontiguousarray(target_pos, dtype=np.float64).reshape(-1, 3)
    dr = np.ascontiguousarray(danger_radius, dtype=np.float64)
    cr = np.ascontiguousarray(center_radius, dtype=np.float64)
    cs, tsd = _i8(center_side), _i8(side_pref)
    out = np.empty(len(tp), dtype=np.int32)
    nf = C.c_int64(0)
    lib().oracle_associate(len(sp), _p(sp), _p(dr), len(cp), _p(cp), _p(cr),
                           None if cs is None else cs.ctypes.data, len(tp), _p(tp), float(eps_ta),
                           None if tsd is None else tsd.ctypes.data, out.ctypes.data_as(_i32p), C.byref(nf))
    return out, int(nf.value)


def area_query(plan, centers, radii):
    """Algorithm 5 by the brute-force leaf scan: (starts int64[n+1], leaves int32)."""
    a = plan.arrays()
    qc = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    qr = np.ascontiguousarray(radii, dtype=np.float64)
    n = len(qc)
    bc = np.ascontiguousarray(a["box_center"])
    br = np.ascontiguousarray(a["box_radius"])
    cs = np.ascontiguousarray(a["child_starts"])
    cnt = np.zeros(n, dtype=np.int64)
    args = (int(a["n_boxes"]), _p(bc), _p(br), cs.ctypes.data_as(_i32p), n, _p(qc), _p(qr))
    lib().oracle_area_query(*args, cnt.ctypes.data_as(_i64p), None, None)
    starts = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=starts[1:])
    leaves = np.zeros(max(1, int(starts[-1])), dtype=np.int32)
    lib().oracle_area_query(*args, cnt.ctypes.data_as(_i64p), starts.ctypes.data_as(_i64p),
                            leaves.ctypes.data_as(_i32p))
    return starts, leaves[:int(starts[-1])]


def adequately_separated(kind: int, ca, ha: float, cb, hb: float, tf: float) -> bool:
    """Oracle restatement of SPEC.md:370-378 (kind 0 box_vs_tcr, 1 tcr_vs_box)."""
    a = np.ascontiguousarray(ca, dtype=np.float64)
    b = np.ascontiguousarray(cb, dtype=np.float64)
    return bool(lib().qbxo_adequately_separated(kind, a.ctypes.data_as(_dp), ha, b.ctypes.data_as(_dp), hb, tf))
