"""PnP RANSAC (geometry.py:414-474, tracking.py:208) with device hypothesis
scoring (ec3r_ransac_draws + ec3r_pnp_score) against the reference's own
outputs (tests/golden/pnp.npz, made by make_golden.py from the unmodified
reference): the reference's test_geometry scenes, noisy / outlier / planar
problems up to 1,500 correspondences, a count-tie case, NoConsensus and
TooFewCorrespondences.  Inlier masks and ratios are bit-exact and the models
identical (the winning hypothesis is the same draw, so the reference's own
host refits see identical inputs).  The minimal EPnP stays the reference's
host code, so these tests need it importable (baseline/_ref)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref_geometry():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2510_02080_b200.types import reference_module
    try:
        return reference_module("submap_slam.geometry")
    except ImportError:
        pytest.skip("the reference's host EPnP (baseline/_ref) is not installed")


def _case(g, c, rg):
    pts, pix, Kv, cf = g[f"c{c}_pts"], g[f"c{c}_pix"], g[f"c{c}_K"], g[f"c{c}_cfg"]
    k = rg.CameraIntrinsics(fx=Kv[0], fy=Kv[1], cx=Kv[2], cy=Kv[3], width=int(Kv[4]), height=int(Kv[5]))
    cfg = rg.RansacConfig(seed=int(cf[0]), min_inliers=int(cf[1]), pixel_threshold=float(cf[2]),
                          max_iterations=int(cf[3]), confidence=float(cf[4]))
    corrs = [rg.Correspondence2D3D(pix[i], pts[i], i) for i in range(len(pts))]
    return corrs, k, cfg


def _check(g, c, r):
    status = str(g[f"c{c}_status"])
    if status != "ok":
        assert isinstance(r, Exception) and type(r).__name__ == status, (c, r)
        return
    assert not isinstance(r, Exception), (c, r)
    np.testing.assert_array_equal(r.inlier_mask, g[f"c{c}_mask"], err_msg=f"case {c}")
    assert r.inlier_ratio == float(g[f"c{c}_ratio"])
    np.testing.assert_array_equal(np.asarray(r.model.rotation.q), g[f"c{c}_q"])
    np.testing.assert_array_equal(np.asarray(r.model.translation), g[f"c{c}_t"])


def test_pnp_golden_cases(golden, ref_geometry):
    from paper_2510_02080_b200 import geometry
    g = golden("pnp")
    for c in range(int(g["n_cases"])):
        corrs, k, cfg = _case(g, c, ref_geometry)
        try:
            r = geometry.solve_pnp_ransac(corrs, k, cfg)
        except Exception as e:  # the reference's exception types
            r = e
        _check(g, c, r)


def test_pnp_batched_equals_golden(golden, ref_geometry):
    """All cases in one solve_pnp_ransac_batch call (hypotheses of every
    problem scored in shared launches)."""
    from paper_2510_02080_b200 import geometry
    g = golden("pnp")
    probs, seeds, cfgs = [], [], []
    for c in range(int(g["n_cases"])):
        corrs, k, cfg = _case(g, c, ref_geometry)
        probs.append((corrs, k))
        cfgs.append(cfg)
    # one config per batch: group the cases by their (min_inliers, threshold, budget)
    groups = {}
    for c, cfg in enumerate(cfgs):
        groups.setdefault((cfg.min_inliers, cfg.pixel_threshold, cfg.max_iterations), []).append(c)
    for cs in groups.values():
        stats = {}
        res = geometry.solve_pnp_ransac_batch([probs[c] for c in cs], cfgs[cs[0]], seeds=[cfgs[c].seed for c in cs],
                                              stats=stats)
        for c, r in zip(cs, res):
            _check(g, c, r)
    assert stats.get("hypotheses_scored", 0) > 0
