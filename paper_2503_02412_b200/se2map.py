"""Thin ctypes binding of libse2map.so (include/se2map.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; there is no Python or CPU
fallback.  If the extension is missing this module raises at import time.
Names follow the C ABI: ``init``, ``update_elevation``, ``shift_window``, ``assess_se2``,
``query``, ``download`` (+ the ``Se2Map`` convenience class).  Arrays may be NumPy (host) or
torch CUDA tensors (device, passed by data pointer with SE2M_MEM_DEVICE).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_LIB_PATH = os.environ.get("SE2M_LIB") or _build.LIB  # SE2M_LIB: A/B-test an alternative build
if not os.path.exists(_LIB_PATH):
    raise ImportError(
        "libse2map.so is not built (%s); run __graft_entry__.build() — there is no CPU fallback" % _LIB_PATH)

SE2M_OK, SE2M_ERR_INVALID_ARG, SE2M_ERR_OOM, SE2M_ERR_CUDA, SE2M_ERR_UNSUPPORTED, SE2M_ERR_OUT_OF_RANGE, \
    SE2M_ERR_STATE, SE2M_ERR_NCCL = range(8)
SE2M_FULL, SE2M_INCREMENTAL = 0, 1
SE2M_MEM_HOST, SE2M_MEM_DEVICE = 0, 1
SE2M_SHARD_NONE, SE2M_SHARD_YAW, SE2M_SHARD_ROWS = 0, 1, 2

EXPORTS = ["se2m_default_params", "se2m_init", "se2m_destroy", "se2m_update_elevation", "se2m_shift_window",
           "se2m_assess_se2", "se2m_query", "se2m_download", "se2m_get_origin", "se2m_stencil_info",
           "se2m_synchronize", "se2m_launch_count", "se2m_last_error", "se2m_tile_info", "se2m_shard_plan",
           "se2m_download_compact", "se2m_compute_sdf", "se2m_download_sdf", "se2m_sdf_from_mask",
           "se2m_query_trilinear", "se2m_integrate_scan", "se2m_download_elevation", "se2m_inpaint",
           "se2m_download_inpainted", "se2m_download_compact_rep", "se2m_step",
           "se2m_owned_rows", "se2m_halo_size", "se2m_halo_pack", "se2m_halo_unpack", "se2m_halo_plan",
           "se2m_chain_segments", "se2m_query_async", "se2m_exchange_halo", "se2m_nccl_unique_id",
           "se2m_query_trilinear_async", "se2m_debug_phases", "se2m_nccl_selftest"]


class Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_yaw", ctypes.c_int32),
                ("shard_mode", ctypes.c_int32), ("resolution", ctypes.c_double),
                ("ellipse_ex", ctypes.c_double), ("ellipse_ey", ctypes.c_double),
                ("w_r", ctypes.c_double * 3), ("kappa_max", ctypes.c_double),
                ("phi_x_max", ctypes.c_double), ("phi_y_max", ctypes.c_double),
                ("robot_x", ctypes.c_double), ("robot_y", ctypes.c_double),
                ("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("device", ctypes.c_int32),
                ("chain_segments", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p),
                ("fe_z_min", ctypes.c_double), ("fe_z_max", ctypes.c_double), ("fe_gate", ctypes.c_double),
                ("fe_ray_eps", ctypes.c_double), ("fe_prior_var", ctypes.c_double),
                ("inpaint", ctypes.c_int32), ("step_graph", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


class Pose(ctypes.Structure):
    """se2m_pose: row-major 3x3 rotations / covariances (NEXT-1 front-end)."""
    _fields_ = [("R_B", ctypes.c_double * 9), ("p_B", ctypes.c_double * 3), ("R_BS", ctypes.c_double * 9),
                ("p_BS", ctypes.c_double * 3), ("Sigma_S", ctypes.c_double * 9), ("Sigma_R", ctypes.c_double * 9),
                ("Sigma_B", ctypes.c_double * 9)]

    @classmethod
    def from_arrays(cls, R_B, p_B, R_BS, p_BS, Sigma_S, Sigma_R, Sigma_B):
        q = cls()
        for name, v in (("R_B", R_B), ("p_B", p_B), ("R_BS", R_BS), ("p_BS", p_BS), ("Sigma_S", Sigma_S),
                        ("Sigma_R", Sigma_R), ("Sigma_B", Sigma_B)):
            flat = np.ascontiguousarray(v, dtype=np.float64).ravel()
            setattr(q, name, (ctypes.c_double * len(flat))(*flat))
        return q


_lib = ctypes.CDLL(_LIB_PATH)
if os.environ.get("SE2M_LIB"):  # an A/B build may predate some entry points: give the missing ones a stub
    class _Missing:
        def __init__(self, name):
            self.name = name

        def __call__(self, *a):
            raise RuntimeError("%s is not exported by %s" % (self.name, _LIB_PATH))

    class _LibView:
        def __init__(self, lib):
            self._lib = lib

        def __getattr__(self, name):
            try:
                return getattr(self._lib, name)
            except AttributeError:
                stub = _Missing(name)
                setattr(self, name, stub)
                return stub
    _lib = _LibView(_lib)
_vp, _i32, _i64, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_lib.se2m_default_params.argtypes = [ctypes.POINTER(Params)]
_lib.se2m_default_params.restype = None
_lib.se2m_init.argtypes = [ctypes.POINTER(Params), ctypes.POINTER(_vp)]
_lib.se2m_destroy.argtypes = [_vp]
_lib.se2m_destroy.restype = None
_lib.se2m_update_elevation.argtypes = [_vp, _i32, _i32, _i32, _i32, _vp, _i64, _vp, _i32]
_lib.se2m_shift_window.argtypes = [_vp, _f64, _f64, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]
_lib.se2m_assess_se2.argtypes = [_vp, _i32]
_lib.se2m_query.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.se2m_download.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i32]
_lib.se2m_get_origin.argtypes = [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
_lib.se2m_stencil_info.argtypes = [_vp, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]
_lib.se2m_synchronize.argtypes = [_vp]
_lib.se2m_download_compact.argtypes = [_vp, _vp, _vp, _i32]
_lib.se2m_compute_sdf.argtypes = [_vp, _f64]
_lib.se2m_download_sdf.argtypes = [_vp, _vp, _i32]
_lib.se2m_sdf_from_mask.argtypes = [_vp, _i32, _i32, _i32, _f64, _f64, _vp, _i32, _i32]
_lib.se2m_query_trilinear.argtypes = [_vp, _i64, _vp, _i32, _vp, _vp]
_lib.se2m_integrate_scan.argtypes = [_vp, _vp, _i64, ctypes.POINTER(Pose), _i32, _vp]
_lib.se2m_download_elevation.argtypes = [_vp, _vp, _vp, _i32]
_lib.se2m_inpaint.argtypes = [_vp]
_lib.se2m_owned_rows.argtypes = [_vp, _vp, ctypes.POINTER(_i32)]
_lib.se2m_step.argtypes = [_vp, _f64, _f64, _vp, _i64, _i64, _i64, _i32, _i32, _i32, ctypes.POINTER(_i32),
                           ctypes.POINTER(_i32)]
_lib.se2m_download_compact_rep.argtypes = [_vp, _vp, _vp, _i32]
_lib.se2m_download_inpainted.argtypes = [_vp, _vp, _i32]
_lib.se2m_tile_info.argtypes = [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]
_lib.se2m_shard_plan.argtypes = [ctypes.POINTER(Params)] + [ctypes.POINTER(_i32)] * 6
_lib.se2m_query_async.argtypes = [_vp, _i64, _vp, _vp, _i32]
_lib.se2m_chain_segments.argtypes = [_vp, ctypes.POINTER(_i32)]
_lib.se2m_halo_size.argtypes = [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]
_lib.se2m_halo_pack.argtypes = [_vp, _i32, _vp]
_lib.se2m_halo_unpack.argtypes = [_vp, _i32, _vp]
_lib.se2m_halo_plan.argtypes = [ctypes.POINTER(Params), _i64, _i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                _vp]
_lib.se2m_exchange_halo.argtypes = [_vp]
_lib.se2m_debug_phases.argtypes = [_vp, _vp, _i64, _i32, ctypes.POINTER(_i64)]
_lib.se2m_query_trilinear_async.argtypes = [_vp, _i64, _vp, _i32, _vp, _i32]
_lib.se2m_nccl_unique_id.argtypes = [_vp, _i32, ctypes.POINTER(_i32)]
_lib.se2m_nccl_selftest.argtypes = [_i32, _i64, ctypes.POINTER(_i32)]
_lib.se2m_launch_count.argtypes = [_vp]
_lib.se2m_launch_count.restype = _i64
_lib.se2m_last_error.argtypes = [_vp]
_lib.se2m_last_error.restype = ctypes.c_char_p
for _name in ("se2m_init", "se2m_update_elevation", "se2m_shift_window", "se2m_assess_se2", "se2m_query",
              "se2m_download", "se2m_get_origin", "se2m_stencil_info", "se2m_synchronize", "se2m_tile_info",
              "se2m_shard_plan", "se2m_download_compact", "se2m_compute_sdf", "se2m_download_sdf",
              "se2m_sdf_from_mask", "se2m_query_trilinear", "se2m_integrate_scan",
              "se2m_download_elevation", "se2m_halo_size", "se2m_halo_pack", "se2m_halo_unpack",
              "se2m_halo_plan", "se2m_chain_segments", "se2m_query_async", "se2m_exchange_halo",
              "se2m_nccl_unique_id", "se2m_query_trilinear_async", "se2m_debug_phases", "se2m_nccl_selftest"):
    getattr(_lib, _name).restype = ctypes.c_int


def lib():
    return _lib


class Se2mError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("se2map status %d: %s" % (status, msg))
        self.status = status


def default_params(**kw) -> Params:
    """se2m_default_params + overrides; nccl_unique_id may be given as the 128 bytes of nccl_unique_id()."""
    p = Params()
    _lib.se2m_default_params(ctypes.byref(p))
    for k, v in kw.items():
        if k == "w_r":
            p.w_r = (ctypes.c_double * 3)(*v)
        elif k == "nccl_unique_id" and isinstance(v, (bytes, bytearray)):
            buf = ctypes.create_string_buffer(bytes(v), len(v))
            p._nccl_id_buf = buf                        # keep alive until se2m_init copied it
            p.nccl_unique_id = ctypes.addressof(buf)
        else:
            setattr(p, k, v)
    return p


def nccl_unique_id():
    """(128-byte NCCL unique id, NCCL version code) made by the library's NCCL (host-only, no GPU): one rank
    makes it and sends it to the others over the caller's bootstrap channel (e.g. torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    ver = _i32()
    st = _lib.se2m_nccl_unique_id(buf, 128, ctypes.byref(ver))
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    return buf.raw, ver.value


def nccl_selftest(device=0, count=1 << 20):
    """se2m_nccl_selftest: a one-rank NCCL communicator on `device` sends `count` floats to itself through the
    calls se2m_exchange_halo makes; returns the loaded NCCL's version code, raises Se2mError on any failure."""
    ver = _i32()
    st = _lib.se2m_nccl_selftest(int(device), int(count), ctypes.byref(ver))
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    return ver.value


def _ptr(a):
    """(address, mem kind, keepalive) of a NumPy array or a torch tensor."""
    if a is None:
        return None, SE2M_MEM_HOST, None
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        return a.data_ptr(), (SE2M_MEM_DEVICE if a.is_cuda else SE2M_MEM_HOST), a
    a = np.ascontiguousarray(a)
    return a.ctypes.data, SE2M_MEM_HOST, a


def _cuda_ptr(t):
    if not (hasattr(t, "is_cuda") and t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _ptr_nocopy(a):
    if a is None:
        return None, SE2M_MEM_HOST, None
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        return a.data_ptr(), (SE2M_MEM_DEVICE if a.is_cuda else SE2M_MEM_HOST), a
    return a.ctypes.data, SE2M_MEM_HOST, a


def _check_async_buffers(xyt, out, rows):
    """Asynchronous calls read xyt and write out after the call returned, so nothing may be converted or copied
    here (a temporary would be freed first): validate instead — xyt (n, 3) float64 C-contiguous, out (rows, n)
    float32 C-contiguous, both host or both device."""
    def desc(a):
        if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
            return str(a.dtype).replace("torch.", ""), tuple(a.shape), a.is_contiguous(), a.is_cuda
        return str(a.dtype), tuple(a.shape), bool(a.flags["C_CONTIGUOUS"]), False
    dx, sx, cx, gx = desc(xyt)
    do, so, co, go = desc(out)
    n = sx[0] if len(sx) == 2 else -1
    if dx != "float64" or len(sx) != 2 or sx[1] != 3 or not cx:
        raise ValueError("xyt must be a C-contiguous (n, 3) float64 array")
    if do != "float32" or so != (rows, n) or not co:
        raise ValueError("out must be a C-contiguous (%d, n) float32 array" % rows)
    if gx != go:
        raise ValueError("xyt and out must both be host or both be device memory")


def shard_plan(params: Params) -> dict:
    """Host-only share of this rank (no GPU needed): representative bins and tile-row ownership."""
    v = [_i32() for _ in range(6)]
    st = _lib.se2m_shard_plan(ctypes.byref(params), *[ctypes.byref(x) for x in v])
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    keys = ("n_rep", "k_lo", "k_hi", "tile_y", "row_mod", "row_rank")
    return {k: x.value for k, x in zip(keys, v)}


def halo_plan(params: Params, J_M: int, sender: int, last: int) -> dict:
    """Host-only (no GPU): the row-band halo slabs rank `sender` sends for window origin row J_M — the
    first world row of each slab (None past the end of the list); last = 0: the first rows of its tile rows
    (sent to rank sender - 1), 1: the last rows (sent to rank sender + 1).  See se2m_halo_plan."""
    cap, rows = _i32(), _i32()
    st = _lib.se2m_halo_plan(ctypes.byref(params), J_M, sender, last, ctypes.byref(cap), ctypes.byref(rows), None)
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    first = np.empty(cap.value, np.int64)
    st = _lib.se2m_halo_plan(ctypes.byref(params), J_M, sender, last, ctypes.byref(cap), ctypes.byref(rows),
                             first.ctypes.data)
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    return {"cap": cap.value, "slab_rows": rows.value,
            "first_rows": [int(v) if v != np.iinfo(np.int64).min else None for v in first]}


def sdf_from_mask(mask, resolution: float, d_max: float, device: int = 0):
    """NEXT-2 stand-alone: signed distance field (metres) of obstacle masks [layers][ny][nx] (host NumPy)."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    shp = m.shape
    ny, nx = shp[-2], shp[-1]
    layers = int(np.prod(shp[:-2])) if len(shp) > 2 else 1
    out = np.empty(shp, np.float32)
    st = _lib.se2m_sdf_from_mask(m.ctypes.data, nx, ny, layers, resolution, d_max, out.ctypes.data,
                                 SE2M_MEM_HOST, device)
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    return out


def init(params: Params):
    h = _vp()
    st = _lib.se2m_init(ctypes.byref(params), ctypes.byref(h))
    if st != SE2M_OK:
        raise Se2mError(st, _lib.se2m_last_error(None).decode())
    return h


class Se2Map:
    """Owns one se2m_map handle."""

    def __init__(self, params: Params | None = None, **kw):
        self.params = params if params is not None else default_params(**kw)
        self.h = init(self.params)

    # -- lifecycle -------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            _lib.se2m_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st, ok=(SE2M_OK,)):
        if st not in ok:
            raise Se2mError(st, _lib.se2m_last_error(self.h).decode())
        return st

    # -- C-ABI calls -----------------------------------------------------------------
    def update_elevation(self, heights, known=None, i0: int = 0, j0: int = 0):
        """heights: (h, w) float32 NumPy array or CUDA tensor; known: same shape uint8 or None."""
        hh, w = heights.shape
        if hasattr(heights, "is_cuda"):                      # torch tensor (host or device)
            if heights.dtype.__repr__() != "torch.float32" or heights.stride(1) != 1:
                raise ValueError("heights tensor must be float32 with unit column stride")
            ld = heights.stride(0)
            if known is not None and (known.shape != heights.shape or known.stride(0) != ld or known.stride(1) != 1):
                raise ValueError("known must have the layout of heights")
        else:                                                # NumPy: row views are passed without a copy
            if heights.dtype != np.float32 or heights.strides[1] != 4 or heights.strides[0] % 4:
                heights = np.ascontiguousarray(heights, dtype=np.float32)
            ld = heights.strides[0] // 4
            if known is not None:
                known = np.asarray(known, dtype=np.uint8)
                if known.shape != heights.shape or known.strides != (ld, 1):
                    kk = np.zeros((hh, ld), np.uint8)
                    kk[:, :w] = known
                    known = kk[:, :w]
        hp, mem, keep = _ptr_nocopy(heights)
        kp, mem2, keep2 = _ptr_nocopy(known)
        if known is not None and mem2 != mem:
            raise ValueError("heights and known must both be host or both be device memory")
        return self._check(_lib.se2m_update_elevation(self.h, i0, j0, w, hh, hp, ld, kp, mem))

    def shift_window(self, x: float, y: float):
        di, dj = _i32(), _i32()
        self._check(_lib.se2m_shift_window(self.h, x, y, ctypes.byref(di), ctypes.byref(dj)))
        return di.value, dj.value

    def step(self, x: float, y: float, world, world_I0: int, world_J0: int):
        """H1 + H2 + H9 in one call: recentre on (x, y), fill the entered cells from `world` (a float32 CUDA
        tensor of world heights whose element [0, 0] is world cell (world_I0, world_J0)), assess
        INCREMENTAL.  Returns (di, dj)."""
        if not (hasattr(world, "is_cuda") and world.is_cuda) or world.stride(1) != 1:
            raise ValueError("world must be a CUDA tensor with unit column stride")
        wh, ww = world.shape
        di, dj = _i32(), _i32()
        self._check(_lib.se2m_step(self.h, x, y, world.data_ptr(), world.stride(0), world_I0, world_J0, ww, wh,
                                   SE2M_MEM_DEVICE, ctypes.byref(di), ctypes.byref(dj)))
        return di.value, dj.value

    def assess_se2(self, mode: int = SE2M_FULL):
        return self._check(_lib.se2m_assess_se2(self.h, mode))

    def query(self, xyt):
        xyt = np.ascontiguousarray(xyt, dtype=np.float64).reshape(-1, 3)
        n = len(xyt)
        out = {k: np.empty(n, np.float32) for k in ("risk", "pitch", "roll", "z")}
        out["trav"] = np.empty(n, np.uint8)
        st = _lib.se2m_query(self.h, n, xyt.ctypes.data, out["risk"].ctypes.data, out["pitch"].ctypes.data,
                             out["roll"].ctypes.data, out["z"].ctypes.data, out["trav"].ctypes.data)
        self._check(st, ok=(SE2M_OK, SE2M_ERR_OUT_OF_RANGE))
        out["status"] = st
        return out

    def query_async(self, xyt, out):
        """Queue the lookups of xyt (n x 3 float64: host array — pinned buffers are read / written in place by the
        kernel, pageable ones staged — or CUDA tensor) into out (5 x n float32, same memory kind: risk, pitch,
        roll, z, trav as rows); valid after synchronize().  Both buffers must stay alive and untouched until then."""
        _check_async_buffers(xyt, out, 5)
        xp, mem, _ = _ptr_nocopy(xyt)
        op, _, _ = _ptr_nocopy(out)
        return self._check(_lib.se2m_query_async(self.h, xyt.shape[0], xp, op, mem))

    def download(self, planes=("risk", "pitch", "roll", "z", "trav"), out=None):
        """Whole planes in logical [k][j][i] order as NumPy arrays (or into ``out`` dict of arrays/tensors)."""
        P = self.params
        shape = (P.n_yaw, P.ny, P.nx)
        res = {}
        ptrs = []
        mem = SE2M_MEM_HOST
        for name in ("risk", "pitch", "roll", "z", "trav"):
            if name not in planes:
                ptrs.append(None)
                continue
            if out is not None and name in out:
                a = out[name]
            else:
                a = np.empty(shape, np.uint8 if name == "trav" else np.float32)
            p, mem_a, keep = _ptr(a)
            mem = mem_a
            res[name] = a
            ptrs.append(p)
        self._check(_lib.se2m_download(self.h, *ptrs, mem))
        return res

    def download_compact(self, out=None):
        """(risk_h float16 [k][j][i], trav bits u32 [k][j][ceil(nx/32)]) in logical order (host NumPy by default)."""
        P = self.params
        wpr = (P.nx + 31) // 32
        if out is None:
            out = {"risk_h": np.empty((P.n_yaw, P.ny, P.nx), np.float16),
                   "trav_bits": np.empty((P.n_yaw, P.ny, wpr), np.uint32)}
        rp, mem, k1 = _ptr_nocopy(out.get("risk_h"))
        bp, mem2, k2 = _ptr_nocopy(out.get("trav_bits"))
        if out.get("risk_h") is not None and out.get("trav_bits") is not None and mem != mem2:
            raise ValueError("both outputs must be host or both device")
        mem = mem if out.get("risk_h") is not None else mem2
        self._check(_lib.se2m_download_compact(self.h, rp, bp, mem))
        return out

    def owned_rows(self):
        """Logical rows of the window this rank owns (all rows unless row-band sharded)."""
        n = _i32()
        self._check(_lib.se2m_owned_rows(self.h, None, ctypes.byref(n)))
        rows = np.empty(n.value, np.int32)
        self._check(_lib.se2m_owned_rows(self.h, rows.ctypes.data, ctypes.byref(n)))
        return rows

    def download_compact_rep(self, out=None):
        """Representative planes only (Risk and traversability are pi-periodic in theta: plane k serves bins k
        and k + n_yaw/2).  Host outputs (pinned, for overlap) are filled asynchronously: call synchronize()
        before reading them."""
        P = self.params
        n_rep = P.n_yaw // 2 if P.n_yaw % 2 == 0 else P.n_yaw
        wpr = (P.nx + 31) // 32
        if out is None:
            rows = len(self.owned_rows())
            out = {"risk_h": np.empty((n_rep, rows, P.nx), np.float16),
                   "trav_bits": np.empty((n_rep, rows, wpr), np.uint32)}
        rp, mem, k1 = _ptr_nocopy(out.get("risk_h"))
        bp, mem2, k2 = _ptr_nocopy(out.get("trav_bits"))
        if out.get("risk_h") is not None and out.get("trav_bits") is not None and mem != mem2:
            raise ValueError("both outputs must be host or both device")
        mem = mem if out.get("risk_h") is not None else mem2
        self._check(_lib.se2m_download_compact_rep(self.h, rp, bp, mem))
        return out

    def compute_sdf(self, d_max: float = 2.0):
        return self._check(_lib.se2m_compute_sdf(self.h, d_max))

    def download_sdf(self):
        P = self.params
        out = np.empty((P.n_yaw, P.ny, P.nx), np.float32)
        self._check(_lib.se2m_download_sdf(self.h, out.ctypes.data, SE2M_MEM_HOST))
        return out

    def query_trilinear(self, xyt, field: int = 0):
        """field 0 = risk, 1 = sdf: (value (n,), grad (n, 3), status)."""
        xyt = np.ascontiguousarray(xyt, dtype=np.float64).reshape(-1, 3)
        n = len(xyt)
        v = np.empty(n, np.float32)
        g = np.empty((n, 3), np.float32)
        st = _lib.se2m_query_trilinear(self.h, n, xyt.ctypes.data, field, v.ctypes.data, g.ctypes.data)
        self._check(st, ok=(SE2M_OK, SE2M_ERR_OUT_OF_RANGE))
        return v, g, st

    def query_trilinear_async(self, xyt, out, field: int = 0):
        """Queue trilinear lookups of xyt (n x 3 float64, C-contiguous: host array — pinned buffers are read /
        written in place by the kernel, pageable ones staged — or CUDA tensor) into out (4 x n float32, same memory
        kind: value, d/dx, d/dy, d/dtheta); valid after synchronize().  Both buffers must stay alive and untouched
        until then."""
        _check_async_buffers(xyt, out, 4)
        xp, mem, _ = _ptr_nocopy(xyt)
        op, _, _ = _ptr_nocopy(out)
        return self._check(_lib.se2m_query_trilinear_async(self.h, xyt.shape[0], xp, field, op, mem))

    def integrate_scan(self, points, pose: Pose):
        """NEXT-1: one LiDAR frame (points (n, 3) float32 sensor frame: NumPy host or CUDA tensor).
        Returns counts (used, outside map, outside band, bad variance, ray-reset events)."""
        if hasattr(points, "is_cuda"):
            pp, mem, keep = _ptr_nocopy(points)
            n = points.shape[0]
        else:
            points = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
            pp, mem, keep = points.ctypes.data, SE2M_MEM_HOST, points
            n = len(points)
        cnt = np.zeros(5, np.int64)
        self._check(_lib.se2m_integrate_scan(self.h, pp, n, ctypes.byref(pose), mem, cnt.ctypes.data))
        return cnt

    def download_elevation(self):
        P = self.params
        h = np.empty((P.ny, P.nx), np.float32)
        v = np.empty((P.ny, P.nx), np.float32)
        self._check(_lib.se2m_download_elevation(self.h, h.ctypes.data, v.ctypes.data, SE2M_MEM_HOST))
        return h, v

    def inpaint(self):
        """NEXT-4: refresh the nearest-neighbour inpainted view (raises if no cell is known)."""
        self._check(_lib.se2m_inpaint(self.h))

    def download_inpainted(self):
        P = self.params
        h = np.empty((P.ny, P.nx), np.float32)
        self._check(_lib.se2m_download_inpainted(self.h, h.ctypes.data, SE2M_MEM_HOST))
        return h

    def origin(self):
        I, J = _i64(), _i64()
        self._check(_lib.se2m_get_origin(self.h, ctypes.byref(I), ctypes.byref(J)))
        return I.value, J.value

    def stencil_info(self, k: int):
        n, r = _i32(), _i32()
        self._check(_lib.se2m_stencil_info(self.h, k, ctypes.byref(n), ctypes.byref(r)))
        return n.value, r.value

    def tile_info(self):
        tx, ty = _i32(), _i32()
        self._check(_lib.se2m_tile_info(self.h, ctypes.byref(tx), ctypes.byref(ty)))
        return tx.value, ty.value

    def synchronize(self):
        return self._check(_lib.se2m_synchronize(self.h))

    def chain_segments(self) -> int:
        """Yaw-chain segments S (S = n_rep: no chain)."""
        v = _i32()
        self._check(_lib.se2m_chain_segments(self.h, ctypes.byref(v)))
        return v.value

    # -- row-band halo exchange (SE2M_SHARD_ROWS, world_size > 1) ----------------------------------
    def halo_size(self):
        """(cap, slab_rows): a halo buffer holds cap x slab_rows x nx float32."""
        cap, rows = _i32(), _i32()
        self._check(_lib.se2m_halo_size(self.h, ctypes.byref(cap), ctypes.byref(rows)))
        return cap.value, rows.value

    def halo_pack(self, dir: int, dst):
        """Outgoing slabs toward rank g + dir (dir = -1 / +1) into the CUDA tensor dst (asynchronous)."""
        return self._check(_lib.se2m_halo_pack(self.h, dir, _cuda_ptr(dst)))

    def halo_unpack(self, src, frm: int):
        """Write the slabs received from rank g + frm (frm = -1 / +1) into the map (asynchronous)."""
        return self._check(_lib.se2m_halo_unpack(self.h, frm, _cuda_ptr(src)))

    def exchange_halo(self):
        """se2m_exchange_halo: pack, NCCL send / recv to ranks g -+ 1 and unpack, all inside the library on the
        map's stream (needs the map created with nccl_unique_id).  Call after update_elevation of the rank's own
        rows and before assess_se2."""
        return self._check(_lib.se2m_exchange_halo(self.h))

    def debug_phases(self, max_records: int = 1 << 17, reset: bool = True):
        """SE2M_PHASES builds only: the assess kernels' per-warp phase records as a structured NumPy array."""
        dt = np.dtype([("t", np.uint64, 6), ("bx", np.int32), ("by", np.int32), ("mode", np.int32), ("flags", np.int32)])
        out = np.zeros(max_records, dt)
        n = _i64()
        self._check(_lib.se2m_debug_phases(self.h, out.ctypes.data, max_records, 1 if reset else 0, ctypes.byref(n)))
        return out[:min(n.value, max_records)]

    def launch_count(self) -> int:
        return int(_lib.se2m_launch_count(self.h))
