"""FP64/integer oracle of nearest-neighbour inpainting (NEXT-4) — TEST INFRASTRUCTURE ONLY
(oracle/__init__.py: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline use oracle/).

PAPER.md:95 (§V, Fig. 3): "the elevation map ... can be inpainted by classical methods"
(§VII.B-1): "Both methods utilize nearest-neighbor interpolation for elevation inpainting".  The paper
does not define "nearest" further; reading R31, after SPEC S:168-176: every unknown cell of
the window takes the height of its nearest known cell of the window — Euclidean distance on grid
indices — with ties going to the known cell that comes first in row-major (j, i) order; known cells are
unchanged; a window without any known cell is an error.

Written as the definition: for each unknown cell, the squared distance to every known cell, the first
minimum in row-major order (np.nonzero enumerates in row-major order, np.argmin returns the first
minimum).  Integer arithmetic only; heights are copied, never computed.

Pinned by tests/test_oracle_inpaint.py (SPEC examples, tie cases, an independent exact EDT, a pure-Python
brute force); the tie rule of R31 is a reading (the paper is silent): parity unpinned as a reading.
"""
from __future__ import annotations

import numpy as np


def inpaint_nearest(heights: np.ndarray, known: np.ndarray):
    """heights (ny, nx) float32, known (ny, nx) bool/uint8 (logical window order).
    Returns (inpainted float32 (ny, nx), site (ny, nx, 2) int64 = (j, i) of the cell each value comes
    from).  Raises ValueError if no cell is known."""
    h = np.asarray(heights, dtype=np.float32)
    k = np.asarray(known).astype(bool)
    if h.shape != k.shape or h.ndim != 2:
        raise ValueError("heights and known must be 2-D arrays of the same shape")
    kj, ki = np.nonzero(k)                    # known cells in row-major order
    if kj.size == 0:
        raise ValueError("inpaint: no known cell in the window")
    ny, nx = h.shape
    out = h.copy()
    site = np.empty((ny, nx, 2), dtype=np.int64)
    jj, ii = np.mgrid[0:ny, 0:nx]
    site[..., 0], site[..., 1] = jj, ii
    kj64, ki64 = kj.astype(np.int64), ki.astype(np.int64)
    for j in range(ny):
        cols = np.nonzero(~k[j])[0]
        if cols.size == 0:
            continue
        # (unknown cells of row j) x (known cells): squared Euclidean distance on grid indices
        d2 = (kj64[None, :] - j) ** 2 + (ki64[None, :] - cols[:, None].astype(np.int64)) ** 2
        best = np.argmin(d2, axis=1)          # first minimum = row-major first among ties
        out[j, cols] = h[kj[best], ki[best]]
        site[j, cols, 0] = kj[best]
        site[j, cols, 1] = ki[best]
    return out, site
