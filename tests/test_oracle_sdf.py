"""Pins for the SDF oracle (NEXT-2).  CPU only.

Independent reference: scipy.ndimage.distance_transform_edt (exact Euclidean distance transform, a
library routine) applied to the obstacle set and to the free set.
"""
import math

import numpy as np
import pytest
from scipy import ndimage

import oracle


def test_spec_examples():
    r = 0.1
    ob = np.zeros((9, 9), np.uint8)
    ob[4, 4] = 1
    s = oracle.sdf(ob, r, 10.0)
    assert abs(s[4, 5] - r) < 1e-15 and abs(s[3, 4] - r) < 1e-15       # 4-neighbour of one obstacle
    assert abs(s[5, 5] - r * math.sqrt(2)) < 1e-15
    assert abs(s[4, 4] + r) < 1e-15                                       # a single obstacle cell: -r
    ob = np.zeros((9, 9), np.uint8)
    ob[3:6, 3:6] = 1
    s = oracle.sdf(ob, r, 10.0)
    assert abs(s[4, 4] + 2 * r) < 1e-15 and abs(s[3, 4] + r) < 1e-15     # 3x3 block: centre -2r, edge -r
    assert np.all(oracle.sdf(np.zeros((5, 6), np.uint8), r, 0.7) == 0.7)   # no obstacles: +d_max
    assert np.all(oracle.sdf(np.ones((5, 6), np.uint8), r, 0.7) == -0.7)   # no free cells: -d_max


@pytest.mark.parametrize("seed,d_max", [(0, 100.0), (1, 0.45), (2, 1.3)])
def test_matches_scipy_edt_and_lipschitz(seed, d_max):
    rng = np.random.default_rng(seed)
    r = 0.05
    ob = (rng.random((48, 56)) < 0.08).astype(np.uint8)
    ob[10:20, 30:45] = 1
    s = oracle.sdf(ob, r, d_max)
    free_d = ndimage.distance_transform_edt(ob == 0) * r      # distance of free cells to the nearest obstacle
    obst_d = ndimage.distance_transform_edt(ob == 1) * r      # distance of obstacle cells to the nearest free
    ref = np.where(ob == 1, -np.minimum(obst_d, d_max), np.minimum(free_d, d_max))
    assert np.max(np.abs(s - ref)) < 1e-12
    # 1-Lipschitz between 4-neighbours on each side of the boundary
    assert np.all(np.abs(np.diff(s, axis=1)) <= r * 2 + 1e-12)
    assert np.all(np.abs(np.diff(s, axis=0)) <= r * 2 + 1e-12)
    assert np.all(s[ob == 1] < 0) and np.all(s[ob == 0] > 0)
