"""FP64 CPU oracle for the SE(2) traversability hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2503_02412_b200``) never imports it, and this package never imports the product
path: the two share no code, header, table or constant generator.  Only the seeded input
generators in ``synth/`` serve both.

Contents
--------
* ``se2_oracle.c`` (compiled to ``liboracle.so``): Algorithm 1 (§V.B) per
  state, in IEEE double, step by step in the paper's order, with a textbook cyclic-Jacobi
  eigen-solver.  Threaded over states with POSIX threads.
* ``Window`` (below): the robot-centric window of Eq. 4 (§V.A) written out in
  plain Python on LOGICAL arrays (no ring buffer): ``shift`` recomputes the origin by Eq. 4 in
  double, copies retained cells bit-exactly into a fresh array and marks exposed cells unknown.
* ``query_index``: world (x, y, theta) -> (logical cell, nearest yaw bin) (reading R3/R6).

Parity: pinned by ``tests/test_oracle_pins.py`` (pins Q1-Q12 of DESIGN.md) and the independent
NumPy brute force in ``tests/bruteforce.py`` (Q5).  On non-planar terrain the per-state values
are pinned only by the invariants Q3-Q8 and the brute force; readings R1, R2, R8 and R14 are
readings of the paper, not confirmable from it ("parity unpinned" for those readings only;
see DESIGN.md §oracle).  ``sdf`` (NEXT-2) is pinned by tests/test_oracle_sdf.py (SPEC examples, scipy's
exact EDT, the 1-Lipschitz property); its reading R24 (centre-to-centre distance, unknown = obstacle) is
parity unpinned as a reading.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "se2_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
GCC_FLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (IEEE double, no FP contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("n_yaw", ctypes.c_int32),
                ("pad0", ctypes.c_int32), ("resolution", ctypes.c_double),
                ("ex", ctypes.c_double), ("ey", ctypes.c_double), ("w", ctypes.c_double * 3),
                ("kappa_max", ctypes.c_double), ("phi_x_max", ctypes.c_double),
                ("phi_y_max", ctypes.c_double)]


class _Result(ctypes.Structure):
    _fields_ = [("risk", ctypes.c_double), ("pitch", ctypes.c_double), ("roll", ctypes.c_double),
                ("z", ctypes.c_double), ("kappa", ctypes.c_double), ("gap", ctypes.c_double),
                ("lam", ctypes.c_double * 3), ("n", ctypes.c_double * 3),
                ("trav", ctypes.c_int32), ("status", ctypes.c_int32),
                ("n_points", ctypes.c_int32), ("early", ctypes.c_int32)]


RESULT_DTYPE = np.dtype([("risk", "f8"), ("pitch", "f8"), ("roll", "f8"), ("z", "f8"),
                         ("kappa", "f8"), ("gap", "f8"), ("lam", "f8", 3), ("n", "f8", 3),
                         ("trav", "i4"), ("status", "i4"), ("n_points", "i4"), ("early", "i4")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        assert _lib.orc_result_size() == RESULT_DTYPE.itemsize == ctypes.sizeof(_Result)
        assert _lib.orc_params_size() == ctypes.sizeof(_Params)
        P, F, U8, I32 = (ctypes.c_void_p,) * 4
        _lib.orc_assess_states.argtypes = [P, F, U8, ctypes.c_int64, I32, P, ctypes.c_int]
        _lib.orc_assess_state.argtypes = [P, F, U8, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_uint64, P]
        _lib.orc_eig3.argtypes = [P, P, P]
        _lib.orc_sdf_layer.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, P,
                                       ctypes.c_int]
    return _lib


@dataclass
class Params:
    """Alg. 1 constant inputs + the grid."""
    nx: int
    ny: int
    resolution: float
    n_yaw: int
    ex: float = 0.8
    ey: float = 0.5
    w: tuple = (0.4, 0.3, 0.3)
    kappa_max: float = 0.1
    phi_x_max: float = 0.52
    phi_y_max: float = 0.52

    def c(self) -> _Params:
        p = _Params()
        p.nx, p.ny, p.n_yaw, p.pad0 = self.nx, self.ny, self.n_yaw, 0
        p.resolution, p.ex, p.ey = self.resolution, self.ex, self.ey
        p.w = (ctypes.c_double * 3)(*self.w)
        p.kappa_max, p.phi_x_max, p.phi_y_max = self.kappa_max, self.phi_x_max, self.phi_y_max
        return p


def _prep(params: Params, heights, known):
    h = np.ascontiguousarray(heights, dtype=np.float32)
    assert h.shape == (params.ny, params.nx), (h.shape, params.ny, params.nx)
    k = None if known is None else np.ascontiguousarray(known, dtype=np.uint8)
    if k is not None:
        assert k.shape == h.shape
    return h, k


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def assess_all(params: Params, heights, known=None, nthreads: int | None = None) -> np.ndarray:
    """Alg. 1 for every state; structured array of shape (n_yaw, ny, nx), layout [k][j][i]."""
    h, k = _prep(params, heights, known)
    out = np.zeros(params.n_yaw * params.ny * params.nx, dtype=RESULT_DTYPE)
    cp = params.c()
    rc = lib().orc_assess_states(ctypes.byref(cp), h.ctypes.data,
                                 None if k is None else k.ctypes.data, 0, None,
                                 out.ctypes.data, nthreads or default_threads())
    if rc:
        raise ValueError("oracle: invalid parameters (rc=%d)" % rc)
    return out.reshape(params.n_yaw, params.ny, params.nx)


def assess_states(params: Params, heights, ijk, known=None, nthreads: int | None = None) -> np.ndarray:
    """Alg. 1 for a list of states ijk (n, 3) = (i, j, k) in window coordinates."""
    h, k = _prep(params, heights, known)
    ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
    out = np.zeros(len(ijk), dtype=RESULT_DTYPE)
    if len(ijk) == 0:
        return out
    cp = params.c()
    rc = lib().orc_assess_states(ctypes.byref(cp), h.ctypes.data,
                                 None if k is None else k.ctypes.data, len(ijk), ijk.ctypes.data,
                                 out.ctypes.data, nthreads or default_threads())
    if rc:
        raise ValueError("oracle: invalid parameters or state index (rc=%d)" % rc)
    return out


def assess_state(params: Params, heights, i: int, j: int, k: int, known=None, shuffle_seed: int = 0):
    """One state; ``shuffle_seed`` != 0 permutes the gathered points (pin Q8)."""
    h, kn = _prep(params, heights, known)
    out = np.zeros(1, dtype=RESULT_DTYPE)
    cp = params.c()
    rc = lib().orc_assess_state(ctypes.byref(cp), h.ctypes.data, None if kn is None else kn.ctypes.data,
                                i, j, k, shuffle_seed, out.ctypes.data)
    if rc:
        raise MemoryError("oracle: allocation failed")
    return out[0]


def eig3(C) -> tuple[np.ndarray, np.ndarray]:
    """Cyclic-Jacobi eigen-decomposition (ascending eigenvalues, eigenvectors as columns)."""
    A = np.ascontiguousarray(C, dtype=np.float64).reshape(3, 3)
    lam = np.zeros(3)
    V = np.zeros((3, 3))
    lib().orc_eig3(A.ctypes.data, lam.ctypes.data, V.ctypes.data)
    return lam, V


def sdf(obstacle, r: float, d_max: float, nthreads: int | None = None) -> np.ndarray:
    """Signed distance field (metres) of obstacle masks [..., ny, nx] (reading R24): free cells
    get the distance to the nearest obstacle cell, obstacle cells minus the distance to the nearest free
    cell, clamped to +-d_max.  Brute force over all cell pairs, one layer at a time."""
    ob = np.ascontiguousarray(obstacle, dtype=np.uint8)
    shape = ob.shape
    ny, nx = shape[-2], shape[-1]
    layers = ob.reshape(-1, ny, nx)
    out = np.empty(layers.shape, dtype=np.float64)
    for L in range(len(layers)):
        lay = np.ascontiguousarray(layers[L])
        o = np.empty((ny, nx), dtype=np.float64)
        rc = lib().orc_sdf_layer(lay.ctypes.data, nx, ny, r, d_max, o.ctypes.data, nthreads or default_threads())
        if rc:
            raise ValueError("oracle sdf: bad arguments")
        out[L] = o
    return out.reshape(shape)


# ---------------------------------------------------------------------------------------
# Window (Eq. 4) and query, on logical arrays.
# ---------------------------------------------------------------------------------------
def window_origin(x: float, y: float, r: float, nx: int, ny: int) -> tuple[int, int]:
    """Eq. 4: p_M = l_res * floor(x / l_res).  Reading R6: the window is
    [floor(x/r) - nx//2, floor(x/r) - nx//2 + nx) in world cells.  IEEE double floor of
    x / r (reading R7: 1.2 / 0.1 -> 11)."""
    I_r = math.floor(x / r)
    J_r = math.floor(y / r)
    return I_r - nx // 2, J_r - ny // 2


class Window:
    """Robot-centric elevation window on logical arrays."""

    def __init__(self, nx: int, ny: int, r: float, x: float, y: float):
        self.nx, self.ny, self.r = nx, ny, r
        self.I_M, self.J_M = window_origin(x, y, r, nx, ny)
        self.heights = np.zeros((ny, nx), dtype=np.float32)
        self.known = np.zeros((ny, nx), dtype=np.uint8)
        self.var = np.zeros((ny, nx), dtype=np.float32)   # cell height variance (front-end, NEXT-1)

    def shift(self, x: float, y: float) -> tuple[int, int]:
        """Recentre (Eq. 4); retained cells keep their values bit-exactly, cells that enter
        the window are unknown (PAPER.md:103 'set the state of grids that are no longer
        within the map to unknown')."""
        I_M, J_M = window_origin(x, y, self.r, self.nx, self.ny)
        di, dj = I_M - self.I_M, J_M - self.J_M
        h = np.zeros_like(self.heights)
        k = np.zeros_like(self.known)
        v = np.zeros_like(self.var)
        for j in range(self.ny):
            for i in range(self.nx):
                oi, oj = i + di, j + dj            # old logical index of new cell (i, j)
                if 0 <= oi < self.nx and 0 <= oj < self.ny:
                    h[j, i] = self.heights[oj, oi]
                    k[j, i] = self.known[oj, oi]
                    v[j, i] = self.var[oj, oi]
        self.heights, self.known, self.var = h, k, v
        self.I_M, self.J_M = I_M, J_M
        return di, dj

    def write_world(self, I0: int, J0: int, values: np.ndarray, known=None):
        """Write world-indexed values (rows J0.., cols I0..) that fall inside the window."""
        hgt, wid = values.shape
        for jj in range(hgt):
            for ii in range(wid):
                i, j = I0 + ii - self.I_M, J0 + jj - self.J_M
                if 0 <= i < self.nx and 0 <= j < self.ny:
                    self.heights[j, i] = values[jj, ii]
                    self.known[j, i] = 1 if known is None else known[jj, ii]


def query_index(x: float, y: float, theta: float, I_M: int, J_M: int, nx: int, ny: int,
                r: float, n_yaw: int):
    """World (x, y, theta) -> (i, j, k) or None when outside the window.  Cell by reading R6
    (world cell I covers [I r, (I+1) r)); nearest yaw bin k = floor((theta+pi)/dtheta + 1/2)
    mod n_yaw (reading R3: theta_k = -pi + k dtheta)."""
    i = math.floor(x / r) - I_M
    j = math.floor(y / r) - J_M
    dth = 2.0 * math.pi / n_yaw
    k = math.floor((theta + math.pi) / dth + 0.5) % n_yaw
    if not (0 <= i < nx and 0 <= j < ny):
        return None
    return i, j, k
