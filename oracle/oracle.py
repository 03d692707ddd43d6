"""ctypes wrapper of oracle.c (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

__all__ = ["build", "lib", "schedule", "keyframes", "bary_textbook", "fast_coeffs", "fast_eval",
           "render_fwd", "render_bwd", "num_threads", "closest_w", "soft_pair", "segments"]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain IEEE fp64: no -ffast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=c99", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _Scene(C.Structure):
    _fields_ = [("V", C.c_int), ("F", C.c_int), ("B", C.c_int), ("H", C.c_int), ("W", C.c_int),
                ("verts", C.c_void_p), ("faces", C.c_void_p), ("colors", C.c_void_p),
                ("cams", C.c_void_p), ("kind", C.c_void_p), ("vec", C.c_void_p),
                ("angle", C.c_void_p), ("pivot", C.c_void_p), ("n_sub", C.c_void_p),
                ("n_seg", C.c_void_p), ("rule", C.c_void_p), ("sub_range", C.c_void_p)]


class _Opts(C.Structure):
    _fields_ = [("mode", C.c_int), ("threads", C.c_int), ("check_fast", C.c_int),
                ("eps_amb", C.c_double), ("amb_val_tol", C.c_double), ("amb_z_rel", C.c_double),
                ("npix", C.c_int), ("pix", C.c_void_p), ("delta", C.c_double), ("soft_exact", C.c_int)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = C.CDLL(build())
            P = C.c_void_p
            _lib.om_schedule.argtypes = [C.c_int, C.c_int, C.c_int, P, P]
            _lib.om_keyframes.argtypes = [P, C.c_int, P, P, P]
            _lib.om_bary_textbook.argtypes = [P, P, C.c_double, C.c_double, P, P]
            _lib.om_fast_coeffs.argtypes = [P, P, P, P, C.c_double, C.c_double, P, P, P, P]
            _lib.om_fast_coeffs.restype = None
            _lib.om_fast_eval.argtypes = [P, P, P, P, C.c_double, C.c_double, C.c_double, P, P]
            _lib.om_render_fwd.argtypes = [P, P, P, P, C.c_int, P, P, P, P, P]
            _lib.om_render_bwd.argtypes = [P, P, P, P, P, P]
            _lib.om_num_threads.argtypes = [C.c_int]
            _lib.om_segments.argtypes = [P, C.c_int]
            _lib.om_closest_w.argtypes = [P, P, C.c_double, C.c_double, P, P, P, P, P]
            _lib.om_soft_pair.argtypes = [P, P, P, P, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                          C.c_double, P, P, P, P, P]
        return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _d(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a if shape is None else a.reshape(shape)


def _i(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class _Pack:
    """Holds the fp64/int32 copies alive while a call runs."""

    def __init__(self, sc, sub_range=None):
        self.verts = _d(sc.verts)
        self.faces = _i(sc.faces)
        self.colors = _d(sc.colors)
        self.cams = _d(sc.cams)
        m = sc.motion
        self.kind, self.vec, self.angle = _i(m["kind"]), _d(m["vec"]), _d(m["angle"])
        self.pivot, self.n_sub, self.n_seg, self.rule = _d(m["pivot"]), _i(m["n_sub"]), _i(m["n_seg"]), _i(m["rule"])
        self.sub_range = None if sub_range is None else _i(sub_range)
        self.s = _Scene(self.verts.shape[0], self.faces.shape[0], self.cams.shape[0], sc.H, sc.W,
                        _p(self.verts), _p(self.faces), _p(self.colors), _p(self.cams), _p(self.kind),
                        _p(self.vec), _p(self.angle), _p(self.pivot), _p(self.n_sub), _p(self.n_seg),
                        _p(self.rule), _p(self.sub_range))


def _opts(mode="binned", threads=0, check_fast=False, eps_amb=0.0, amb_val_tol=1e-5, amb_z_rel=1e-6,
          pixels=None, delta=0.0, soft_exact=False):
    pix = None if pixels is None else _i(pixels).reshape(-1, 3)
    o = _Opts(1 if mode == "binned" else 0, threads, int(check_fast), eps_amb, amb_val_tol, amb_z_rel,
              0 if pix is None else pix.shape[0], _p(pix), float(delta), int(soft_exact))
    return o, pix


def num_threads(req: int = 0) -> int:
    return lib().om_num_threads(req)


def schedule(N: int, S: int, rule: int = 0):
    s = np.zeros(N, np.int32)
    t = np.zeros(N, np.float64)
    if lib().om_schedule(N, S, rule, _p(s), _p(t)):
        raise ValueError("invalid schedule (N=%d, S=%d, rule=%d)" % (N, S, rule))
    return s, t


def segments(sc, b: int = 0) -> int:
    """Segment count of image b (n_seg, or the automatic rule for n_seg == 0; Q24)."""
    pk = _Pack(sc)
    return int(lib().om_segments(C.byref(pk.s), b))


def keyframes(sc, b: int = 0):
    """(S+1, V, 3) NDC x, y and view z; (S+1, V) valid; (S+1, V, 3) view coordinates."""
    pk = _Pack(sc)
    S = segments(sc, b)
    key = np.zeros((S + 1, sc.V, 3))
    valid = np.zeros((S + 1, sc.V), np.uint8)
    Q = np.zeros((S + 1, sc.V, 3))
    lib().om_keyframes(C.byref(pk.s), b, _p(key), _p(valid), _p(Q))
    return key, valid.astype(bool), Q


def bary_textbook(x, y, u, v):
    w = np.zeros(3)
    det = np.zeros(1)
    ok = lib().om_bary_textbook(_p(_d(x)), _p(_d(y)), float(u), float(v), _p(w), _p(det))
    return (w if ok else None), float(det[0])


def fast_coeffs(X0, Y0, X1, Y1, u, v):
    A1, A2, A3, a = np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3)
    lib().om_fast_coeffs(_p(_d(X0)), _p(_d(Y0)), _p(_d(X1)), _p(_d(Y1)), float(u), float(v),
                         _p(A1), _p(A2), _p(A3), _p(a))
    return A1, A2, A3, a


def fast_eval(X0, Y0, X1, Y1, u, v, t):
    w = np.zeros(3)
    den = np.zeros(1)
    ok = lib().om_fast_eval(_p(_d(X0)), _p(_d(Y0)), _p(_d(X1)), _p(_d(Y1)), float(u), float(v), float(t),
                            _p(w), _p(den))
    return (w if ok else None), float(den[0])


def render_fwd(sc, mode="binned", threads=0, ids_k=-1, eps_amb=0.0, check_fast=False, sub_range=None,
               frozen=None, pixels=None, colors=None, verts=None, delta=0.0, soft_exact=False):
    """Blurred RGBA (B,H,W,4) fp64 (or (npix,4) in pixel-list mode).
    delta > 0 adds the soft background alpha of Eq.10-15 (NEXT-1; soft_exact: Eq.12 instead of Eq.13).
    Returns dict(rgba, ids, amb_img, amb_ids, amb_win, stats, behind); the amb_* maps are the Q16
    exclusion masks: blurred value movable by > 1e-5, winner at ids_k ambiguous,
    winner ambiguous at some sub-frame."""
    import dataclasses
    if colors is not None or verts is not None:
        sc = dataclasses.replace(sc, colors=sc.colors if colors is None else colors,
                                 verts=sc.verts if verts is None else verts)
    pk = _Pack(sc, sub_range)
    o, pix = _opts(mode, threads, check_fast, eps_amb, pixels=pixels, delta=delta, soft_exact=soft_exact)
    shape = (pix.shape[0],) if pix is not None else (sc.B, sc.H, sc.W)
    rgba = np.zeros(shape + (4,))
    ids = np.full(shape, -1, np.int32)
    amb_i = np.zeros(shape, np.uint8)
    amb_d = np.zeros(shape, np.uint8)
    amb_w = np.zeros(shape, np.uint8)
    stats = np.zeros(4)
    fz = None if frozen is None else _i(frozen)
    on = eps_amb > 0
    r = lib().om_render_fwd(C.byref(pk.s), C.byref(o), _p(rgba), _p(ids), int(ids_k),
                            _p(amb_i) if on else None, _p(amb_d) if on else None, _p(amb_w) if on else None,
                            _p(fz), _p(stats))
    if r < 0:
        raise ValueError("oracle: invalid input")
    return dict(rgba=rgba, ids=ids, amb_img=amb_i.astype(bool), amb_ids=amb_d.astype(bool),
                amb_win=amb_w.astype(bool),
                stats=dict(max_fast_dev=stats[0], n_checked=stats[1], necessary_pairs=stats[2],
                           covered=stats[3]), behind=bool(r == 1))


def render_bwd(sc, grad_rgba, mode="binned", threads=0, sub_range=None, pixels=None, want_dkey=False,
               colors=None, verts=None, delta=0.0, soft_exact=False):
    """(dverts (V,3), dcolors (V,3)[, dkey list per image (S+1,V,2)]) in fp64.
    delta > 0: the alpha channel of grad_rgba also flows through the soft background (Eq.10-15)."""
    import dataclasses
    if colors is not None or verts is not None:
        sc = dataclasses.replace(sc, colors=sc.colors if colors is None else colors,
                                 verts=sc.verts if verts is None else verts)
    pk = _Pack(sc, sub_range)
    o, pix = _opts(mode, threads, pixels=pixels, delta=delta, soft_exact=soft_exact)
    g = _d(grad_rgba)
    dv = np.zeros((sc.V, 3))
    dc = np.zeros((sc.V, 3))
    Ss = [segments(sc, b) for b in range(sc.B)]
    nkey = int(sum((S + 1) * sc.V * 2 for S in Ss))
    dk = np.zeros(nkey) if want_dkey else None
    r = lib().om_render_bwd(C.byref(pk.s), C.byref(o), _p(g), _p(dv), _p(dc), _p(dk))
    if r < 0:
        raise ValueError("oracle: invalid input")
    if not want_dkey:
        return dv, dc
    out, off = [], 0
    for S in Ss:
        n = (int(S) + 1) * sc.V * 2
        out.append(dk[off:off + n].reshape(int(S) + 1, sc.V, 2))
        off += n
    return dv, dc, out


def closest_w(x, y, pu, pv, w_in=None):
    """Appendix A17-A18 closest-point weights of (pu, pv) on triangle (x, y): (what, dist2, edge,
    candidates (3,3), candidate dist2 (3,)).  edge = -1 when w_in says the point is inside."""
    what, d2, cand, cd = np.zeros(3), np.zeros(1), np.zeros(9), np.zeros(3)
    e = lib().om_closest_w(_p(_d(x)), _p(_d(y)), float(pu), float(pv), _p(None if w_in is None else _d(w_in)),
                           _p(what), _p(d2), _p(cand), _p(cd))
    return what, float(d2[0]), int(e), cand.reshape(3, 3), cd


def soft_pair(X0, Y0, X1, Y1, tau, u, v, delta, exact=False, eps=0.0):
    """One background term (Eq.10-14): dict(A, d, what, pstar, amb) or None if F(tau) is degenerate."""
    A, d, wh, pst, amb = np.zeros(1), np.zeros(1), np.zeros(3), np.zeros(2), np.zeros(1)
    ok = lib().om_soft_pair(_p(_d(X0)), _p(_d(Y0)), _p(_d(X1)), _p(_d(Y1)), float(tau), float(u), float(v),
                            float(delta), int(exact), float(eps), _p(A), _p(d), _p(wh), _p(pst), _p(amb))
    if not ok:
        return None
    return dict(A=float(A[0]), d=float(d[0]), what=wh, pstar=pst, amb=float(amb[0]))
