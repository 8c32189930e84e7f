"""Thin ctypes binding of the TABI C ABI (include/tabi.h).

Argument marshalling only: every step of the packing runs in the CUDA kernels
of ``libtabi.so``. There is no CPU fallback -- if the library or a GPU is
missing, these calls raise.

Inputs may be numpy arrays (host; the library copies them in and the result
out inside the call) or CUDA torch tensors (device pointers, run on
``torch.cuda.current_stream()``); torch is used only for device memory and
streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtabi.so")

OK, EINVAL, NO_FIT, ECUDA, ECAPACITY, PENDING = 0, 1, 2, 3, 4, 5
F_NO_HC, F_NO_BALANCE, F_ADJACENT_LOCKS_ONLY, F_PREROTATE, F_NO_OBB, F_EXACT_TAIL = (1, 2, 4, 8, 16,
                                                                            32)
# Ablation / baseline modes on the same kernels (the ablation table after
# P:1060): spec overrides for spec_of(cs, **ABLATIONS[name]).
#   tight_only    = horizontal + vertical compacting, no balance (no knees,
#                   static L/R alternation);
#   balanced_only = balance without tightening: plain AABB proxies (k = 1, no
#                   OBB bound), no horizontal compacting;
#   chameleon     = Chameleon: AABBs, fold + push, strict alternation.
ABLATIONS = {
    "tabi": dict(flags=0),
    "tight_only": dict(flags=F_NO_BALANCE),
    "balanced_only": dict(flags=F_NO_HC | F_NO_OBB, local_aabb_count=1),
    "chameleon": dict(flags=F_NO_HC | F_NO_BALANCE | F_NO_OBB, local_aabb_count=1),
}
STATUS_NAMES = {0: "ok", 1: "invalid argument", 2: "no candidate scale fits", 3: "CUDA error",
                4: "capacity exceeded"}


class TabiError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"tabi status {status} ({STATUS_NAMES.get(status, '?')}) {msg}".strip())
        self.status = status


class Spec(C.Structure):
    _fields_ = [("atlas_w", C.c_int32), ("atlas_h", C.c_int32), ("gutter", C.c_int32),
                ("scale_count", C.c_int32), ("local_aabb_count", C.c_int32),
                ("t_opt_bp", C.c_int32), ("flags", C.c_uint32)]


class Info(C.Structure):
    _fields_ = [("scale_index", C.c_int32), ("fused", C.c_int32), ("l2_stretch", C.c_double),
                ("rows", C.c_int32), ("knees_found", C.c_int32), ("knee_rows", C.c_int32),
                ("prefix_rows", C.c_int32), ("bad_chart", C.c_int32), ("gpu_launches", C.c_int32),
                ("stage_ms", C.c_float * 8), ("work_pack", C.c_int64),
                ("work_profile", C.c_int64), ("device_ms", C.c_float), ("reserved", C.c_int32)]


class Validation(C.Structure):
    _fields_ = [("overlap", C.c_int64), ("gutter", C.c_int64), ("oob", C.c_int64),
                ("covered", C.c_int64), ("occupancy", C.c_double), ("l2_stretch", C.c_double),
                ("bad_chart", C.c_int32), ("gpu_launches", C.c_int32)]


class BatchInfo(C.Structure):
    _fields_ = [("device_ms", C.c_float), ("stage_ms", C.c_float * 4), ("gpu_launches", C.c_int32),
                ("candidates_evaluated", C.c_int32), ("batched_atlases", C.c_int32),
                ("solo_atlases", C.c_int32), ("work_pack", C.c_int64), ("work_profile", C.c_int64),
                ("cycles", C.c_int64 * 3), ("tail_ms", C.c_float), ("busy_frac", C.c_float),
                ("ranks_in_flight", C.c_int32), ("reserved", C.c_int32)]


PLACEMENT_DTYPE = np.dtype([("tx", "<i4"), ("ty", "<i4"), ("scale_num", "<i4"),
                            ("scale_den", "<i4"), ("box_w", "<i4"), ("box_h", "<i4"),
                            ("rot90", "u1"), ("flip_x", "u1"), ("flip_y", "u1"),
                            ("mirror_x", "u1"), ("mode", "u1"), ("prerot", "u1"),
                            ("pad", "u1", (2,))])
assert PLACEMENT_DTYPE.itemsize == 32

PROXY_DTYPE = np.dtype([("w", "<i4"), ("h", "<i4"), ("area2", "<i8"), ("xmin", "<i4"),
                        ("ymin", "<i4"), ("rot90", "<i4"), ("fx", "<i4"), ("fy", "<i4"),
                        ("k", "<i4"), ("top", "<i4", (64,)), ("bot", "<i4", (64,)),
                        ("left", "<i4", (64,)), ("right", "<i4", (64,)), ("obb_j", "<i4"),
                        ("prerot", "<i4"), ("umin", "<i8"), ("umax", "<i8"), ("vmin", "<i8"),
                        ("vmax", "<i8")])
CAND_DTYPE = np.dtype([(f, "<i4") for f in ("success", "score", "rows", "knees_found",
                                            "knee_rows", "prefix_rows", "p", "evaluated",
                                            "switched_at", "reserved")] +
                      [("apre_lo", "<u8"), ("apre_hi", "<u8")])
assert CAND_DTYPE.itemsize == 56

_lib = None


def lib():
    """Load libtabi.so (built in-tree by ``paper_2602_07782_b200.build``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TabiError(ECUDA, f"native library missing: {LIB_PATH} (run build())")
        L = C.CDLL(LIB_PATH)
        P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.tabi_ctx_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, i32, i64, i32]
        L.tabi_ctx_destroy.argtypes = [P]
        L.tabi_pack.argtypes = [P, P, P, i32, C.c_float, C.c_float, C.POINTER(Spec), P,
                                C.POINTER(Info), C.c_int, P]
        L.tabi_pack_async.argtypes = [P, P, P, i32, C.c_float, C.c_float, C.POINTER(Spec), P, P]
        L.tabi_pack_wait.argtypes = [P, C.POINTER(Info)]
        L.tabi_pack_query.argtypes = [P]
        L.tabi_status_str.restype = C.c_char_p
        L.tabi_status_str.argtypes = [C.c_int]
        L.tabi_last_error.restype = C.c_char_p
        L.tabi_last_error.argtypes = [P]
        L.tabi_debug_proxies.argtypes = [P, P]
        L.tabi_debug_perm.argtypes = [P, P]
        L.tabi_debug_candidates.argtypes = [P, P]
        L.tabi_debug_profile.argtypes = [P, i32, i32, P, P, P, P, P]
        L.tabi_debug_offsets.argtypes = [P, i32, P, P]
        L.tabi_debug_trace.argtypes = [P, P]
        L.tabi_debug_trace_raster.argtypes = [P, P]
        L.tabi_debug_latency_floor.argtypes = [C.c_int, P]
        L.tabi_shard_plan.argtypes = [i32, P, i32, P]
        L.tabi_pack_batch.argtypes = [P, i32, i32, P, P, P, P, P, P, P]
        L.tabi_pack_many.argtypes = [P, i32, P, P, P, P, C.POINTER(Spec), P, P, P,
                                     C.POINTER(BatchInfo), C.c_int, P]
        L.tabi_validate.argtypes = [P, P, P, i32, C.c_float, C.c_float, i32, i32, i32, P,
                                    C.POINTER(Validation), C.c_int, P]
        _lib = L
    return _lib


EXPORTS = ["tabi_ctx_create", "tabi_ctx_destroy", "tabi_pack", "tabi_pack_async",
           "tabi_pack_wait", "tabi_pack_query", "tabi_status_str",
           "tabi_last_error", "tabi_debug_proxies", "tabi_debug_perm", "tabi_debug_candidates",
           "tabi_debug_profile", "tabi_debug_offsets", "tabi_debug_trace",
           "tabi_debug_trace_raster", "tabi_shard_plan", "tabi_pack_batch", "tabi_pack_many",
           "tabi_validate", "tabi_debug_latency_floor"]


def latency_floor(device: int = 0) -> dict:
    """ns per packer building block (tabi_debug_latency_floor)."""
    out = np.zeros(8, dtype=np.float64)
    st = lib().tabi_debug_latency_floor(device, _ptr(out))
    if st != OK:
        raise TabiError(st, "tabi_debug_latency_floor")
    return dict(barrier_ns=out[0], barrier_smem_exchange_ns=out[1], block_max_ns=out[2],
                smem_atomic_barrier_ns=out[3], l2_dependent_load_ns=out[4], sm_mhz=out[5])


def concat_chart_sets(chart_sets):
    """Marshal independent chart sets into tabi_pack_many's layout: outlines
    back to back, GLOBAL vertex offsets, per-atlas chart offsets and
    resolutions.  Returns (xy float32[2V], chart_start int32[N+1],
    atlas_start int32[A+1], res_xy float32[2A])."""
    xys, starts, abase, res = [], [], [0], []
    vo = 0
    for cs in chart_sets:
        st = np.asarray(cs.start, dtype=np.int64)
        xys.append(np.asarray(cs.xy, dtype=np.float32))
        starts.append((st[:-1] + vo).astype(np.int32))
        vo += int(st[-1])
        abase.append(abase[-1] + cs.n_charts)
        r = getattr(cs, "res", 1.0)
        res.extend((r, r))
    starts.append(np.array([vo], dtype=np.int32))
    return (np.concatenate(xys), np.concatenate(starts), np.asarray(abase, dtype=np.int32),
            np.asarray(res, dtype=np.float32))


def shard_plan(n_charts, n_gpus: int) -> np.ndarray:
    """LPT assignment of atlases to GPUs (tabi_shard_plan; host code, no GPU)."""
    nc = np.ascontiguousarray(n_charts, dtype=np.int32)
    out = np.zeros(nc.shape[0], dtype=np.int32)
    st = lib().tabi_shard_plan(nc.shape[0], _ptr(nc), n_gpus, _ptr(out))
    if st != OK:
        raise TabiError(st, "tabi_shard_plan")
    return out


def pack_batch(contexts, chart_sets, specs):
    """Pack independent atlases on several contexts (one host thread each).
    Returns (status, [placements], [Info])."""
    n = len(chart_sets)
    xys = [np.ascontiguousarray(cs.xy, dtype=np.float32) for cs in chart_sets]
    starts = [np.ascontiguousarray(cs.start, dtype=np.int32) for cs in chart_sets]
    outs = [np.zeros(cs.n_charts, dtype=PLACEMENT_DTYPE) for cs in chart_sets]
    infos = (Info * n)()
    ctx_arr = (C.c_void_p * len(contexts))(*[c.h.value for c in contexts])
    xy_arr = (C.c_void_p * n)(*[a.ctypes.data for a in xys])
    st_arr = (C.c_void_p * n)(*[a.ctypes.data for a in starts])
    out_arr = (C.c_void_p * n)(*[a.ctypes.data for a in outs])
    nch = np.array([cs.n_charts for cs in chart_sets], dtype=np.int32)
    res = np.array([[cs.res, cs.res] for cs in chart_sets], dtype=np.float32).reshape(-1)
    spec_arr = (Spec * n)(*specs)
    st = lib().tabi_pack_batch(ctx_arr, len(contexts), n, xy_arr, st_arr, _ptr(nch), _ptr(res),
                               spec_arr, out_arr, infos)
    return st, outs, list(infos)


def _ptr(a):
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def make_spec(atlas_w, atlas_h, gutter=1, scale_count=64, local_aabb_count=10, t_opt_bp=0,
              flags=0) -> Spec:
    return Spec(atlas_w, atlas_h, gutter, scale_count, local_aabb_count, t_opt_bp, flags)


def spec_of(cs, **kw) -> Spec:
    d = dict(gutter=cs.gutter, scale_count=cs.scale_count, local_aabb_count=cs.local_aabb_count,
             t_opt_bp=cs.t_opt_bp, flags=0)
    d.update(kw)
    return make_spec(cs.atlas_w, cs.atlas_h, **d)


def _torch_stream(device):
    """Handle of torch's current stream on `device` for the C ABI.  torch's
    default stream is the legacy NULL stream (handle 0), which the ABI reads as
    "the context's own stream"; pass cudaStreamLegacy (1) instead so the pack
    stays ordered with the torch work that produced its inputs."""
    import torch
    h = torch.cuda.current_stream(device).cuda_stream
    return h if h else 1


class Context:
    """One device workspace + stream (``tabi_ctx``)."""

    def __init__(self, device: int = 0, max_charts: int = 1 << 16, max_vertices: int = 1 << 20,
                 max_atlas_side: int = 16384):
        h = C.c_void_p()
        st = lib().tabi_ctx_create(C.byref(h), device, max_charts, max_vertices, max_atlas_side)
        if st != OK:
            raise TabiError(st, "tabi_ctx_create")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().tabi_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return lib().tabi_last_error(self.h).decode()

    def pack(self, xy, start, spec: Spec, res=(1.0, 1.0), out=None, stream=None,
             raise_on_error=True):
        """Pack one atlas. Host numpy inputs -> host numpy placements; CUDA tensors
        (xy float32, start int32, out uint8[32*N]) -> device placements.
        Returns (status, placements, Info)."""
        on_device = hasattr(xy, "is_cuda") and xy.is_cuda
        n = int(start.shape[0]) - 1
        info = Info()
        if on_device:
            import torch
            if out is None:
                out = torch.empty(n * PLACEMENT_DTYPE.itemsize, dtype=torch.uint8, device=xy.device)
            if stream is None:
                stream = _torch_stream(xy.device)
            st = lib().tabi_pack(self.h, _ptr(xy), _ptr(start), n, res[0], res[1], C.byref(spec),
                                 _ptr(out), C.byref(info), 1, C.c_void_p(stream))
        else:
            xy = np.ascontiguousarray(xy, dtype=np.float32)
            start = np.ascontiguousarray(start, dtype=np.int32)
            if out is None:
                out = np.zeros(n, dtype=PLACEMENT_DTYPE)
            st = lib().tabi_pack(self.h, _ptr(xy), _ptr(start), n, res[0], res[1], C.byref(spec),
                                 _ptr(out), C.byref(info), 0,
                                 C.c_void_p(stream) if stream else None)
        if raise_on_error and st not in (OK, NO_FIT):
            raise TabiError(st, f"bad_chart={info.bad_chart} {self.last_error()}")
        return st, out, info

    def pack_async(self, xy, start, spec: Spec, res=(1.0, 1.0), out=None, stream=None):
        """Enqueue one pack (tabi_pack_async) from CUDA tensors and return the
        device placement buffer at once; the inputs must stay alive and unchanged
        until ``wait()``.  Raises on errors found before enqueueing."""
        import torch
        n = int(start.shape[0]) - 1
        if out is None:
            out = torch.empty(n * PLACEMENT_DTYPE.itemsize, dtype=torch.uint8, device=xy.device)
        if stream is None:
            stream = _torch_stream(xy.device)
        st = lib().tabi_pack_async(self.h, _ptr(xy), _ptr(start), n, res[0], res[1], C.byref(spec),
                                   _ptr(out), C.c_void_p(stream))
        if st != OK:
            raise TabiError(st, self.last_error())
        self._pending = (xy, start, out)  # keep the buffers alive until wait()
        return out

    def query(self) -> int:
        """tabi_pack_query: PENDING while the asynchronous pack runs, OK once done."""
        return lib().tabi_pack_query(self.h)

    def wait(self, raise_on_error=True):
        """tabi_pack_wait: (status, device placements, Info) of the pending pack."""
        info = Info()
        st = lib().tabi_pack_wait(self.h, C.byref(info))
        out = (getattr(self, "_pending", None) or (None, None, None))[2]
        self._pending = None
        if raise_on_error and st not in (OK, NO_FIT):
            raise TabiError(st, f"bad_chart={info.bad_chart} {self.last_error()}")
        return st, out, info

    def validate(self, xy, start, placements, atlas_w, atlas_h, gutter=1, res=(1.0, 1.0),
                 stream=None, raise_on_error=True):
        """GPU validator + metrics (tabi_validate): overlap / gutter / oob /
        covered texel counts, occupancy and L2 stretch of ``placements``.
        Host numpy inputs, or CUDA tensors (placements as uint8[32*N]).
        Returns a dict."""
        on_device = hasattr(xy, "is_cuda") and xy.is_cuda
        n = int(start.shape[0]) - 1
        v = Validation()
        if on_device:
            import torch
            if stream is None:
                stream = _torch_stream(xy.device)
            st = lib().tabi_validate(self.h, _ptr(xy), _ptr(start), n, res[0], res[1], atlas_w,
                                     atlas_h, gutter, _ptr(placements), C.byref(v), 1,
                                     C.c_void_p(stream))
        else:
            xy = np.ascontiguousarray(xy, dtype=np.float32)
            start = np.ascontiguousarray(start, dtype=np.int32)
            pl = np.ascontiguousarray(placements, dtype=PLACEMENT_DTYPE)
            st = lib().tabi_validate(self.h, _ptr(xy), _ptr(start), n, res[0], res[1], atlas_w,
                                     atlas_h, gutter, _ptr(pl), C.byref(v), 0,
                                     C.c_void_p(stream) if stream else None)
        if raise_on_error and st != OK:
            raise TabiError(st, f"bad_chart={v.bad_chart} {self.last_error()}")
        return dict(status=st, overlap=v.overlap, gutter=v.gutter, oob=v.oob, covered=v.covered,
                    occupancy=v.occupancy, l2_stretch=v.l2_stretch, bad_chart=v.bad_chart,
                    gpu_launches=v.gpu_launches)

    def pack_many(self, xy, chart_start, atlas_start, spec: Spec, res_xy=None, out=None,
                  stream=None, raise_on_error=True):
        """Pack many independent atlases as one device pipeline (tabi_pack_many).
        xy / chart_start (global vertex offsets) / out: host numpy arrays or CUDA
        tensors (out uint8[32*N]); atlas_start and res_xy are host arrays.
        Returns (status, placements, [Info], atlas_status int32[A], BatchInfo)."""
        on_device = hasattr(xy, "is_cuda") and xy.is_cuda
        abase = np.ascontiguousarray(atlas_start, dtype=np.int32)
        A = abase.shape[0] - 1
        N = int(abase[-1])
        infos = (Info * A)()
        ast = np.zeros(A, dtype=np.int32)
        bi = BatchInfo()
        rp = None
        if res_xy is not None:
            res_xy = np.ascontiguousarray(res_xy, dtype=np.float32)
            rp = _ptr(res_xy)
        if on_device:
            import torch
            if out is None:
                out = torch.empty(N * PLACEMENT_DTYPE.itemsize, dtype=torch.uint8, device=xy.device)
            if stream is None:
                stream = _torch_stream(xy.device)
            st = lib().tabi_pack_many(self.h, A, _ptr(xy), _ptr(chart_start), _ptr(abase), rp,
                                      C.byref(spec), _ptr(out), infos, _ptr(ast), C.byref(bi), 1,
                                      C.c_void_p(stream))
        else:
            if not (isinstance(xy, np.ndarray) and xy.dtype == np.float32 and xy.flags.c_contiguous):
                xy = np.ascontiguousarray(xy, dtype=np.float32)
            chart_start = np.ascontiguousarray(chart_start, dtype=np.int32)
            if out is None:
                out = np.zeros(N, dtype=PLACEMENT_DTYPE)
            st = lib().tabi_pack_many(self.h, A, _ptr(xy), _ptr(chart_start), _ptr(abase), rp,
                                      C.byref(spec), _ptr(out), infos, _ptr(ast), C.byref(bi), 0,
                                      C.c_void_p(stream) if stream else None)
        if raise_on_error and st not in (OK, NO_FIT):
            raise TabiError(st, self.last_error())
        return st, out, list(infos), ast, bi

    def pack_set(self, cs, res=None, **spec_kw):
        r = (cs.res, cs.res) if res is None else res
        return self.pack(cs.xy, cs.start, spec_of(cs, **spec_kw), res=r)

    # ---- introspection of the last pack ----
    def proxies(self, n):
        out = np.zeros(n, dtype=PROXY_DTYPE)
        self._chk(lib().tabi_debug_proxies(self.h, _ptr(out)))
        return out

    def perm(self, n):
        out = np.zeros(n, dtype=np.int32)
        self._chk(lib().tabi_debug_perm(self.h, _ptr(out)))
        return out

    def candidates(self, M):
        out = np.zeros(M, dtype=CAND_DTYPE)
        self._chk(lib().tabi_debug_candidates(self.h, _ptr(out)))
        return out

    def profile(self, m, s, max_len=1 << 16):
        wh = np.zeros(2, dtype=np.int32)
        bufs = [np.zeros(max_len, dtype=np.int32) for _ in range(4)]
        st = lib().tabi_debug_profile(self.h, m, s, _ptr(wh), *[_ptr(b) for b in bufs])
        if st == NO_FIT:
            return None
        self._chk(st)
        Wd, Hd = int(wh[0]), int(wh[1])
        return Wd, Hd, bufs[0][:Wd], bufs[1][:Wd], bufs[2][:Hd], bufs[3][:Hd]

    def offsets(self, m, n):
        off = np.zeros(n, dtype=np.int32)
        lk = np.zeros(n, dtype=np.uint8)
        self._chk(lib().tabi_debug_offsets(self.h, m, _ptr(off), _ptr(lk)))
        return off, lk

    def trace(self):
        """Fused-kernel timeline of the last wave (tabi_debug_trace): dict of ns."""
        out = np.zeros(16, dtype=np.int64)
        self._chk(lib().tabi_debug_trace(self.h, _ptr(out)))
        keys = ("raster_end", "pack_end", "pack_wait", "raster_wait", "tiles", "fused")
        d = dict(zip(keys, (int(v) for v in out[:6])))
        r16 = np.zeros(16, dtype=np.int64)
        self._chk(lib().tabi_debug_trace_raster(self.h, _ptr(r16)))
        d["raster_phases"] = dict(zip(("fetch", "cells", "big", "pairs_int", "pairs_bnd",
                                       "publish", "setup"), (int(v) for v in r16[:7])))
        d["alg1_passes"] = int(r16[7])  # trace build: Alg. 1 passes of wave slot 0
        d["first_row_ns"] = dict(zip(("tile0_cells", "tile0_published", "fold_unblocked",
                                      "row0_done", "tile0_raw", "tile0_setup", "tile0_pairs_start",
                                      "tile0_pairs_end"), (int(v) for v in r16[8:16])))
        d["phases"] = dict(zip(("knee", "fold", "hc_locks", "push", "alg1", "score", "commit",
                                "findknee", "push_stage", "commit_stage"),
                               (int(v) for v in out[6:16])))
        return d

    def _chk(self, st):
        if st != OK:
            raise TabiError(st, self.last_error())
