"""Pins for the NEXT-4 inpainting oracle (oracle/inpaint.py).  CPU only."""
import numpy as np
import pytest
from scipy import ndimage

from oracle.inpaint import inpaint_nearest


def test_spec_examples():
    """one known cell -> uniform field; fully known -> identity; all unknown -> error."""
    rng = np.random.default_rng(0)
    h = rng.normal(size=(9, 11)).astype(np.float32)
    k = np.zeros((9, 11), bool)
    k[3, 7] = True
    out, _ = inpaint_nearest(h, k)
    assert np.all(out == h[3, 7])
    out, site = inpaint_nearest(h, np.ones_like(k))
    assert np.array_equal(out, h)
    assert np.array_equal(site[..., 0], np.mgrid[0:9, 0:11][0])
    with pytest.raises(ValueError):
        inpaint_nearest(h, np.zeros_like(k))


def test_tie_rule_row_major():
    """Equidistant known cells: the one first in row-major (j, i) order wins (reading R31)."""
    h = np.arange(25, dtype=np.float32).reshape(5, 5)
    k = np.zeros((5, 5), bool)
    k[0, 2] = k[2, 0] = True          # (1, 1) is at squared distance 2 from both
    out, site = inpaint_nearest(h, k)
    assert tuple(site[1, 1]) == (0, 2) and out[1, 1] == h[0, 2]
    k = np.zeros((5, 5), bool)
    k[2, 0] = k[2, 4] = True          # (2, 2): same row, distance 2 to both -> smaller i
    out, site = inpaint_nearest(h, k)
    assert tuple(site[2, 2]) == (2, 0)
    k = np.zeros((5, 5), bool)
    k[4, 2] = k[2, 4] = True          # (3, 3): (2, 4) precedes (4, 2)
    _, site = inpaint_nearest(h, k)
    assert tuple(site[3, 3]) == (2, 4)


@pytest.mark.parametrize("frac", [0.5, 0.9, 0.99])
def test_distances_match_exact_edt(frac):
    """The chosen site is at the exact Euclidean distance transform's distance (scipy.ndimage, an
    independent exact EDT), i.e. it is a nearest known cell; values are copies of that cell."""
    rng = np.random.default_rng(int(frac * 100))
    ny, nx = 40, 57
    h = rng.normal(size=(ny, nx)).astype(np.float32)
    k = rng.random((ny, nx)) > frac
    k[rng.integers(ny), rng.integers(nx)] = True
    out, site = inpaint_nearest(h, k)
    edt = ndimage.distance_transform_edt(~k)
    jj, ii = np.mgrid[0:ny, 0:nx]
    d2 = (site[..., 0] - jj) ** 2 + (site[..., 1] - ii) ** 2
    assert np.array_equal(np.rint(edt ** 2).astype(np.int64), d2)
    assert np.array_equal(out, h[site[..., 0], site[..., 1]])
    assert np.array_equal(out[k], h[k])


def test_pure_python_brute_force():
    """Triple loop over cells and known cells (strict < keeps the first in row-major order)."""
    rng = np.random.default_rng(4)
    ny, nx = 7, 9
    h = rng.normal(size=(ny, nx)).astype(np.float32)
    k = rng.random((ny, nx)) > 0.6
    out, _ = inpaint_nearest(h, k)
    for j in range(ny):
        for i in range(nx):
            if k[j, i]:
                assert out[j, i] == h[j, i]
                continue
            best, val = None, None
            for jj in range(ny):
                for ii in range(nx):
                    if k[jj, ii]:
                        d = (jj - j) ** 2 + (ii - i) ** 2
                        if best is None or d < best:
                            best, val = d, h[jj, ii]
            assert out[j, i] == val
