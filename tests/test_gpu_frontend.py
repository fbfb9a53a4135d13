"""GPU parity of the NEXT-1 front-end (se2m_integrate_scan) against the FP64 oracle (oracle/frontend.py):
several LiDAR frames with window shifts in between; heights, known mask and variances are compared
after every frame (the arithmetic is FP64 in a fixed order on both sides: bit-identical expected), then
the whole pipeline (front-end + Algorithm 1) is compared with the oracle's assessment of its own map.
"""
import math

import numpy as np
import pytest

import oracle
from oracle.frontend import FrontendParams, Pose, integrate_scan
from synth.lidar import scan
from synth.terrain import Hills
from tests.gpu_common import make_map, oracle_params
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _gpu_pose(fr):
    from paper_2503_02412_b200 import se2map as S
    return S.Pose.from_arrays(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S, fr.Sigma_R, fr.Sigma_B)


@pytest.mark.parametrize("pose_noise", [0.0, 0.01])
def test_frontend_frames_bit_exact_and_pipeline_parity(pose_noise):
    terrain = Hills(seed=21)
    nx, ny, r, n_yaw = 100, 100, 0.1, 36
    path = [(0.37, 0.61, 0.3), (0.81, 0.44, 0.1), (1.56, 0.9, 0.6), (1.57, 0.91, 0.6)]
    m = make_map(nx, ny, r, n_yaw, robot=path[0][:2])
    w = oracle.Window(nx, ny, r, *path[0][:2])
    P = FrontendParams()
    for f, (x, y, yaw) in enumerate(path):
        d = m.shift_window(x, y)
        assert d == w.shift(x, y)
        fr = scan(terrain, x, y, yaw, seed=100 + f, pose_noise=pose_noise, n_az=600)
        cnt = m.integrate_scan(fr.points_s, _gpu_pose(fr))
        st, n_reset = integrate_scan(w, fr.points_s, Pose(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S,
                                                                 fr.Sigma_R, fr.Sigma_B), P)
        assert list(cnt[:4]) == [int((st == s_).sum()) for s_ in range(4)], (cnt, np.bincount(st, minlength=4))
        assert (n_reset == 0) == (cnt[4] == 0)
        h, v = m.download_elevation()
        known_g = ~np.isnan(h)
        assert np.array_equal(known_g, w.known.astype(bool)), f
        assert np.array_equal(h[known_g], w.heights[known_g]), f
        assert np.array_equal(v[known_g], w.var[known_g]), f
    assert known_g.mean() > 0.3
    # whole pipeline: Algorithm 1 on the fused map vs the oracle on its own fused map
    m.assess_se2(1)
    g = m.download()
    orc = oracle.assess_all(oracle_params(nx, ny, r, n_yaw), w.heights, w.known)
    rep = compare(g, orc)
    print(rep)
    assert rep["ok"], rep
