"""CPU oracle for TABI -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product path
(``paper_2602_07782_b200``) never imports it and shares no code with it.

The oracle itself is plain C (``tabi_oracle.c``, ``validate.c``); this module
builds it with gcc and marshals arguments through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRCS = [os.path.join(HERE, f) for f in ("tabi_oracle.c", "validate.c")]
KMAX = 64

OK, EINVAL, NO_FIT = 0, 1, 2
F_NO_HC, F_NO_BALANCE, F_ADJACENT_LOCKS_ONLY, F_PREROTATE, F_NO_OBB, F_EXACT_TAIL = (1, 2, 4, 8, 16,
                                                                            32)


def build(force: bool = False) -> str:
    """Compile the oracle (-O2 -ffp-contract=off, single thread, no SIMD intrinsics)."""
    newest = max(os.path.getmtime(s) for s in SRCS + [os.path.join(HERE, "oracle.h")])
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = ["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", LIB,
               *SRCS, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


class Proxy(C.Structure):
    _fields_ = [("w", C.c_int32), ("h", C.c_int32), ("area2", C.c_int64),
                ("xmin", C.c_int32), ("ymin", C.c_int32),
                ("rot90", C.c_int32), ("fx", C.c_int32), ("fy", C.c_int32), ("k", C.c_int32),
                ("top", C.c_int32 * KMAX), ("bot", C.c_int32 * KMAX),
                ("left", C.c_int32 * KMAX), ("right", C.c_int32 * KMAX),
                ("obb_j", C.c_int32), ("prerot", C.c_int32),
                ("umin", C.c_int64), ("umax", C.c_int64), ("vmin", C.c_int64), ("vmax", C.c_int64)]


class Prof(C.Structure):
    _fields_ = [("ws", C.c_int32), ("hs", C.c_int32), ("Wd", C.c_int32), ("Hd", C.c_int32),
                ("Dtop", C.POINTER(C.c_int32)), ("Dbot", C.POINTER(C.c_int32)),
                ("Dleft", C.POINTER(C.c_int32)), ("Dright", C.POINTER(C.c_int32))]


PLACEMENT_DTYPE = np.dtype([("tx", "<i4"), ("ty", "<i4"), ("scale_num", "<i4"),
                            ("scale_den", "<i4"), ("box_w", "<i4"), ("box_h", "<i4"),
                            ("rot90", "u1"), ("flip_x", "u1"), ("flip_y", "u1"),
                            ("mirror_x", "u1"), ("mode", "u1"), ("prerot", "u1"),
                            ("pad", "u1", (2,))])
assert PLACEMENT_DTYPE.itemsize == 32


class Spec(C.Structure):
    _fields_ = [("atlas_w", C.c_int32), ("atlas_h", C.c_int32), ("gutter", C.c_int32),
                ("scale_count", C.c_int32), ("local_aabb_count", C.c_int32),
                ("t_opt_bp", C.c_int32), ("flags", C.c_uint32)]


class Cand(C.Structure):
    _fields_ = [("success", C.c_int32), ("score", C.c_int32), ("rows", C.c_int32),
                ("knees_found", C.c_int32), ("knee_rows", C.c_int32),
                ("prefix_rows", C.c_int32), ("p", C.c_int32), ("switched_at", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("scale_index", C.c_int32), ("l2_stretch", C.c_double), ("rows", C.c_int32),
                ("knees_found", C.c_int32), ("knee_rows", C.c_int32),
                ("prefix_rows", C.c_int32), ("bad_chart", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        _lib.or_build_proxies.argtypes = [P, P, i32, C.c_float, C.c_float, i32, C.c_uint32, P, P]
        _lib.or_sort.argtypes = [P, i32, P]
        _lib.or_profile.argtypes = [P, i64, i64, i32, C.POINTER(Prof)]
        _lib.or_prof_free.argtypes = [C.POINTER(Prof)]
        _lib.or_offset.argtypes = [C.POINTER(Prof), C.POINTER(Prof)]
        _lib.or_offset.restype = i32
        _lib.or_locks.argtypes = [C.POINTER(Prof), C.POINTER(Prof), i32, P, P]
        _lib.or_fold_row.argtypes = [i32, i32, i32, i32, P, P, P]
        _lib.or_fold_row.restype = i32
        _lib.or_correct_y.argtypes = [i32, P, P, P, P, P]
        _lib.or_push_y.argtypes = [P, i32, i32, P, i32]
        _lib.or_push_y.restype = i32
        _lib.or_update_knee.argtypes = [P, i32, i32, P, P]
        _lib.or_find_knee.argtypes = [i32, P, i32]
        _lib.or_find_knee.restype = i32
        _lib.or_pack_candidate.argtypes = [P, P, i32, C.POINTER(Spec), i32, P, C.POINTER(Cand)]
        _lib.or_pack.argtypes = [P, P, i32, C.c_float, C.c_float, C.POINTER(Spec), P,
                                 C.POINTER(Info), P]
        _lib.or_validate.argtypes = [P, P, i32, C.c_float, C.c_float, i32, i32, i32, P, P]
        _lib.or_raster_chart.argtypes = [P, i32, C.c_float, C.c_float, P, P, i32, i32, i32, i32, P]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def make_spec(cs=None, **kw) -> Spec:
    d = dict(atlas_w=getattr(cs, "atlas_w", 64), atlas_h=getattr(cs, "atlas_h", 64),
             gutter=getattr(cs, "gutter", 1), scale_count=getattr(cs, "scale_count", 64),
             local_aabb_count=getattr(cs, "local_aabb_count", 10),
             t_opt_bp=getattr(cs, "t_opt_bp", 0), flags=0)
    d.update(kw)
    return Spec(**d)


def build_proxies(xy, start, k=10, res=(1.0, 1.0), flags=0):
    xy = np.ascontiguousarray(xy, dtype=np.float32)
    start = _i32(start)
    n = start.shape[0] - 1
    out = (Proxy * n)()
    bad = np.full(1, -1, dtype=np.int32)
    st = lib().or_build_proxies(_ptr(xy), _ptr(start), n, res[0], res[1], k, flags, out, _ptr(bad))
    return st, list(out), int(bad[0])


def sort_order(proxies):
    n = len(proxies)
    arr = (Proxy * n)(*proxies)
    perm = np.zeros(n, dtype=np.int32)
    lib().or_sort(arr, n, _ptr(perm))
    return perm


class Profile:
    """Python copy of one chart's dilated footprint (D11, D13)."""

    def __init__(self, proxy: Proxy, num: int, den: int, g: int):
        pr = Prof()
        ok = lib().or_profile(C.byref(proxy), num, den, g, C.byref(pr))
        if not ok:
            raise RuntimeError("or_profile failed")
        self.ws, self.hs, self.Wd, self.Hd = pr.ws, pr.hs, pr.Wd, pr.Hd
        self.Dtop = np.ctypeslib.as_array(pr.Dtop, (pr.Wd,)).copy()
        self.Dbot = np.ctypeslib.as_array(pr.Dbot, (pr.Wd,)).copy()
        self.Dleft = np.ctypeslib.as_array(pr.Dleft, (pr.Hd,)).copy()
        self.Dright = np.ctypeslib.as_array(pr.Dright, (pr.Hd,)).copy()
        self._c = pr

    def __del__(self):
        try:
            lib().or_prof_free(C.byref(self._c))
        except Exception:
            pass


def offset(a: Profile, b: Profile) -> int:
    return int(lib().or_offset(C.byref(a._c), C.byref(b._c)))


def locks(a: Profile, b: Profile, delta: int):
    la = np.zeros(1, dtype=np.int32)
    lb = np.zeros(1, dtype=np.int32)
    lib().or_locks(C.byref(a._c), C.byref(b._c), delta, _ptr(la), _ptr(lb))
    return bool(la[0]), bool(lb[0])


def fold_row(widths, offs, row_start, fold_w, hc):
    wd = _i32(widths)
    n = wd.shape[0]
    off = np.zeros(n, dtype=np.int32)
    off[:len(offs)] = offs
    x = np.full(n, -1, dtype=np.int32)
    end = lib().or_fold_row(n, row_start, fold_w, int(hc), _ptr(wd), _ptr(off), _ptr(x))
    return int(end), x[row_start:end + 1].tolist()


def correct_y(pairs, y):
    """pairs: list of (a, b, a_locked, b_locked)."""
    y = _i32(y).copy()
    if not pairs:
        return y.tolist()
    pa, pb, la, lb = (_i32([p[i] for p in pairs]) for i in range(4))
    lib().or_correct_y(len(pairs), _ptr(pa), _ptr(pb), _ptr(la), _ptr(lb), _ptr(y))
    return y.tolist()


def push_y(F, X, dtop, direction=0):
    F = _i32(F)
    d = _i32(dtop)
    return int(lib().or_push_y(_ptr(F), X, d.shape[0], _ptr(d), direction))


def make_prof(dtop, dbot, dleft, dright):
    """A Prof built from explicit arrays (hand-derived golden footprints)."""
    arrs = [_i32(a) for a in (dtop, dbot, dleft, dright)]
    pr = Prof()
    pr.Wd, pr.Hd = arrs[0].shape[0], arrs[2].shape[0]
    pr.ws, pr.hs = pr.Wd, pr.Hd
    pr.Dtop, pr.Dbot, pr.Dleft, pr.Dright = (a.ctypes.data_as(C.POINTER(C.c_int32)) for a in arrs)
    pr._keep = arrs
    return pr


def offset_raw(a: Prof, b: Prof) -> int:
    return int(lib().or_offset(C.byref(a), C.byref(b)))


def locks_raw(a: Prof, b: Prof, delta: int):
    la = np.zeros(1, dtype=np.int32)
    lb = np.zeros(1, dtype=np.int32)
    lib().or_locks(C.byref(a), C.byref(b), delta, _ptr(la), _ptr(lb))
    return bool(la[0]), bool(lb[0])


def update_knee(F, ltr, left, right):
    F = _i32(F)
    lr = np.array([left], dtype=np.int32)
    rr = np.array([right], dtype=np.int32)
    ok = lib().or_update_knee(_ptr(F), F.shape[0], int(ltr), _ptr(lr), _ptr(rr))
    return bool(ok), int(lr[0]), int(rr[0])


def find_knee(heights_units, atlas_h):
    h = np.ascontiguousarray(heights_units, dtype=np.int64)
    return int(lib().or_find_knee(h.shape[0], _ptr(h), atlas_h))


def pack(cs, res=(1.0, 1.0), with_cands=False, **spec_kw):
    """Full oracle pack of a chartgen.ChartSet. Returns (status, placements, info, cands)."""
    spec = make_spec(cs, **spec_kw)
    xy = np.ascontiguousarray(cs.xy, dtype=np.float32)
    start = _i32(cs.start)
    n = start.shape[0] - 1
    out = np.zeros(n, dtype=PLACEMENT_DTYPE)
    info = Info()
    cands = (Cand * spec.scale_count)() if with_cands else None
    st = lib().or_pack(_ptr(xy), _ptr(start), n, res[0], res[1], C.byref(spec), _ptr(out),
                       C.byref(info), cands)
    return st, out, info, (list(cands) if with_cands else None)


def pack_candidate(cs, m, res=(1.0, 1.0), **spec_kw):
    spec = make_spec(cs, **spec_kw)
    st, px, bad = build_proxies(cs.xy, cs.start, spec.local_aabb_count, res)
    assert st == OK, (st, bad)
    perm = sort_order(px)
    n = len(px)
    arr = (Proxy * n)(*px)
    out = np.zeros(n, dtype=PLACEMENT_DTYPE)
    cand = Cand()
    lib().or_pack_candidate(arr, _ptr(perm), n, C.byref(spec), m, _ptr(out), C.byref(cand))
    return cand, out


def validate(cs, placements, res=(1.0, 1.0), gutter=None):
    xy = np.ascontiguousarray(cs.xy, dtype=np.float32)
    start = _i32(cs.start)
    n = start.shape[0] - 1
    counts = np.zeros(4, dtype=np.int64)
    pl = np.ascontiguousarray(placements, dtype=PLACEMENT_DTYPE)
    g = cs.gutter if gutter is None else gutter
    ok = lib().or_validate(_ptr(xy), _ptr(start), n, res[0], res[1], cs.atlas_w, cs.atlas_h, g,
                           _ptr(pl), _ptr(counts))
    if not ok:
        raise RuntimeError("validator could not snap input")
    return {"overlap": int(counts[0]), "gutter": int(counts[1]), "oob": int(counts[2])}


def metrics(cs, placements, res=(1.0, 1.0), gutter=None):
    """Validator counts plus the atlas metrics:
    covered texels, occupancy = covered / (W H), and the L2 stretch
    (P:1027-1028): each chart map is a similarity of scale
    s_c = scale_num / scale_den, every triangle's stretch is 1/s_c, so the
    area-weighted RMS is sqrt(sum A_c / s_c^2 / sum A_c), A_c the snapped
    outline area (exact rationals here, one rounding at the end)."""
    from fractions import Fraction
    import math
    xy = np.ascontiguousarray(cs.xy, dtype=np.float32)
    start = _i32(cs.start)
    n = start.shape[0] - 1
    counts = np.zeros(4, dtype=np.int64)
    pl = np.ascontiguousarray(placements, dtype=PLACEMENT_DTYPE)
    g = cs.gutter if gutter is None else gutter
    ok = lib().or_validate(_ptr(xy), _ptr(start), n, res[0], res[1], cs.atlas_w, cs.atlas_h, g,
                           _ptr(pl), _ptr(counts))
    if not ok:
        raise RuntimeError("validator could not snap input")
    num = Fraction(0)
    den = 0
    for c in range(n):
        a, b = int(start[c]), int(start[c + 1])
        q = np.rint(xy[2 * a:2 * b].astype(np.float64).reshape(-1, 2) *
                    np.array([res[0], res[1]]) * 256.0).astype(np.int64)
        x, y = q[:, 0].tolist(), q[:, 1].tolist()
        a2 = abs(sum(x[i] * y[(i + 1) % len(x)] - x[(i + 1) % len(x)] * y[i]
                     for i in range(len(x))))
        s = Fraction(int(pl["scale_num"][c]), int(pl["scale_den"][c]))
        num += Fraction(a2) / (s * s)
        den += a2
    return {"overlap": int(counts[0]), "gutter": int(counts[1]), "oob": int(counts[2]),
            "covered": int(counts[3]),
            "occupancy": int(counts[3]) / (cs.atlas_w * cs.atlas_h),
            "l2_stretch": math.sqrt(num / den)}


def raster_chart(poly_xy, placement, x0, y0, nx, ny, res=(1.0, 1.0)):
    xy = np.ascontiguousarray(poly_xy, dtype=np.float32).reshape(-1)
    pl = np.ascontiguousarray(np.asarray([placement], dtype=PLACEMENT_DTYPE))
    mask = np.zeros((ny, nx), dtype=np.uint8)
    lib().or_raster_chart(_ptr(xy), xy.shape[0] // 2, res[0], res[1], None, _ptr(pl), x0, y0, nx,
                          ny, _ptr(mask))
    return mask
