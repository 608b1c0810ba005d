"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz were
produced by tests/golden/make_golden.py running the unmodified reference)."""

import numpy as np
import pytest

from oracle import fuse as ofuse
from oracle import ref_numpy as ref
from tests.conftest import mapping_submaps

STATUS = {"ok": ref.STATUS_OK, "TooFewCorrespondences": ref.STATUS_TOO_FEW,
          "ValueError": ref.STATUS_SHAPE, "AllZeroConfidence": ref.STATUS_ALL_ZERO,
          "DegenerateConfiguration": ref.STATUS_DEGENERATE}


def test_registration_cases(golden):
    g = golden("registration")
    for i in range(int(g["n_cases"])):
        w = g[f"c{i}_w"] if bool(g[f"c{i}_hasw"]) else None
        s, q, t, rms, st = ref.align_point_sets(g[f"c{i}_p"], g[f"c{i}_q"], w,
                                                bool(g[f"c{i}_withscale"]))
        assert st == STATUS[str(g[f"c{i}_status"])], i
        if st != ref.STATUS_OK:
            continue
        assert abs(s - float(g[f"c{i}_s"])) <= 1e-12 * abs(s), i
        np.testing.assert_allclose(ref.canonical_quat(q), ref.canonical_quat(g[f"c{i}_quat"]),
                                   atol=1e-12)
        np.testing.assert_allclose(t, g[f"c{i}_t"], atol=1e-10)
        assert abs(rms - float(g[f"c{i}_rms"])) <= 1e-12


def test_inverse_project_bit_exact(golden):
    g = golden("mapping")
    sms, _ = mapping_submaps(g)
    sm = sms[0]
    pts, conf, fids, pix = ref.inverse_project(sm["depth"], sm["conf"], sm["frame_ids"],
                                               sm["pose_q"], sm["pose_t"], sm["K"])
    np.testing.assert_array_equal(pts, g["ip_points"])
    np.testing.assert_array_equal(conf, g["ip_conf"])
    np.testing.assert_array_equal(fids, g["ip_fids"])
    np.testing.assert_array_equal(pix, g["ip_pixels"])


@pytest.mark.parametrize("j", [1, 2])
def test_shared_correspondences_and_edges(golden, j):
    g = golden("mapping")
    sms, _ = mapping_submaps(g)
    p, q, w = ref.shared_correspondences(sms[j], sms[j - 1])
    np.testing.assert_array_equal(p, g[f"e{j}_p"])
    np.testing.assert_array_equal(q, g[f"e{j}_q"])
    np.testing.assert_array_equal(w, g[f"e{j}_w"])
    e = ref.registration_edge(sms[j], sms[j - 1])
    np.testing.assert_array_equal(e["keep"], g[f"e{j}_keep"])
    assert e["status"] == ref.STATUS_OK
    assert e["count"] == int(g[f"e{j}_count"])
    assert abs(e["s"] - float(g[f"e{j}_s"])) < 1e-12
    np.testing.assert_allclose(ref.canonical_quat(e["q"]), ref.canonical_quat(g[f"e{j}_quat"]),
                               atol=1e-12)
    np.testing.assert_allclose(e["t"], g[f"e{j}_t"], atol=1e-12)
    assert abs(e["rms"] - float(g[f"e{j}_rms"])) < 1e-12


def test_chained_global_poses(golden):
    """register_submap (mapping.py:200-204): global = partner.global o T."""
    g = golden("mapping")
    sms, globs = mapping_submaps(g)
    cur = (1.0, np.array([1.0, 0, 0, 0]), np.zeros(3))
    for j in range(1, len(sms)):
        e = ref.registration_edge(sms[j], sms[j - 1])
        cur = ref.sim3_compose(globs[j - 1], (e["s"], e["q"], e["t"]))
        s, q, t = globs[j]
        assert abs(cur[0] - s) < 1e-12
        np.testing.assert_allclose(ref.canonical_quat(cur[1]), ref.canonical_quat(q), atol=1e-12)
        np.testing.assert_allclose(cur[2], t, atol=1e-12)


def test_fused_cloud_bit_exact_and_keys(golden):
    g = golden("mapping")
    sms, globs = mapping_submaps(g)
    pts, conf = ref.fused_cloud(sms, globs)
    np.testing.assert_array_equal(pts, g["fused_points"])
    np.testing.assert_array_equal(conf, g["fused_conf"])
    f = ofuse.fuse_points(pts, conf, 0.02)
    assert f["count"].sum() == f["n_in"] == int((conf > 0).sum())
    assert np.all(np.diff(f["keys"]) > 0)
    cells = ref.unpack(f["keys"])
    np.testing.assert_array_equal(ref.pack(cells), f["keys"])
    lo = cells * 0.02
    assert np.all(f["centroid"] >= lo - 1e-9) and np.all(f["centroid"] <= lo + 0.02 + 1e-9)


def test_streamed_fusion_equals_fuse_submaps(golden):
    """fuse_submaps_streamed (the bounded-memory oracle the configs[3] GPU
    parity test uses) against fuse_submaps on the golden submaps, one submap
    per chunk so every shared voxel goes through the partial merge."""
    g = golden("mapping")
    sms, globs = mapping_submaps(g)
    for cell in (0.02, 0.05):
        a = ofuse.fuse_submaps(sms, globs, cell)
        b = ofuse.fuse_submaps_streamed(sms, globs, cell, chunk=1)
        np.testing.assert_array_equal(a["keys"], b["keys"])
        np.testing.assert_array_equal(a["count"], b["count"])
        assert a["n_in"] == b["n_in"] and a["n_out_of_range"] == b["n_out_of_range"]
        np.testing.assert_allclose(b["centroid"], a["centroid"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(b["wsum"], a["wsum"], rtol=1e-12)


def test_match_cases(golden):
    g = golden("match")
    for i in range(int(g["n_cases"])):
        a = g[f"c{i}_a"].astype(np.float64)
        b = g[f"c{i}_b"].astype(np.float64)
        exp = g[f"c{i}_matches"]
        got = np.array(ref.match_descriptors(a, b, 0.8), np.int64).reshape(-1, 2)
        np.testing.assert_array_equal(got, exp)
        np.testing.assert_array_equal(ref.match_descriptors_vec(a, b, 0.8), exp)


def test_retrieval_cases(golden):
    g = golden("retrieval")
    for i in range(int(g["n_cases"])):
        st = ref.SimilarityState()
        tg, tl = g[f"c{i}_tau"]
        for c in range(2):
            res = ref.update_similarity(st, g[f"c{i}_kf"], g[f"c{i}_pooled"],
                                        int(g[f"c{i}_stride"]), int(g[f"c{i}_excl"]), tg, tl)
            pairs = np.array([p for p, _ in res], np.int64).reshape(-1, 2)
            np.testing.assert_array_equal(pairs, g[f"c{i}_call{c}_pairs"])
            np.testing.assert_allclose([s for _, s in res], g[f"c{i}_call{c}_scores"],
                                       rtol=0, atol=1e-15)
        keys = np.array(sorted(st.scores), np.int64).reshape(-1, 2)
        np.testing.assert_array_equal(keys, g[f"c{i}_matrix_keys"])


# --------------------------------------------------------------------------
# native-kernel plugin slot (_kernels/_numpy.py): nn_query / raycast

def test_kernels_nn_query_cases(golden):
    from oracle import kernels as ok
    g = golden("kernels")
    for i in range(int(g["n_nn"])):
        d, ix = ok.nn_query(g[f"nn{i}_query"], g[f"nn{i}_ref"], float(g[f"nn{i}_cell"]))
        np.testing.assert_array_equal(ix, g[f"nn{i}_idx"], err_msg=f"case {i}")
        np.testing.assert_array_equal(d, g[f"nn{i}_dist"], err_msg=f"case {i}")
    d, ix = ok.nn_query(np.zeros((3, 3)), np.zeros((0, 3)), 0.1)
    np.testing.assert_array_equal(d, g["nn_empty_ref_dist"])
    np.testing.assert_array_equal(ix, g["nn_empty_ref_idx"])


def test_kernels_raycast_case(golden):
    from oracle import kernels as ok
    g = golden("kernels")
    boxes = [(b[0], b[1]) for b in g["rc_boxes"]]
    t = ok.raycast(g["rc_origins"], g["rc_dirs"], g["rc_room_min"], g["rc_room_max"], boxes)
    np.testing.assert_array_equal(t, g["rc_t"])


def test_local_candidates_cases(golden):
    from oracle import local as ol
    g = golden("local")
    for i in range(int(g["n_cases"])):
        np.testing.assert_array_equal(ol.visible_counts(g[f"c{i}_pos"], g[f"c{i}_poses"], g[f"c{i}_intr"]),
                                      g[f"c{i}_counts"], err_msg=f"case {i}")
        assert ol.local_candidates(g[f"c{i}_pos"], g[f"c{i}_kf"], g[f"c{i}_poses"], g[f"c{i}_intr"],
                                   float(g["tau_p"])) == g[f"c{i}_cand"].tolist()


def _ransac_case(g, i):
    c = g[f"c{i}_cfg"]
    return g[f"c{i}_src"], g[f"c{i}_dst"], float(c[0]), float(c[1]), int(c[2]), int(c[3])


def test_ransac_homography_cases(golden):
    """oracle/ransac.py == the reference on its own test scenes + mixtures."""
    from oracle import ransac as orr
    g = golden("ransac")
    for i in range(int(g["n_cases"])):
        src, dst, thr, conf, iters, seed = _ransac_case(g, i)
        h, m, r = orr.estimate_homography_ransac(src, dst, thr, conf, iters, seed)
        np.testing.assert_array_equal(m, g[f"c{i}_mask"], err_msg=f"case {i}")
        assert r == float(g[f"c{i}_ratio"])
        np.testing.assert_allclose(h, g[f"c{i}_model"], rtol=0, atol=1e-9 * np.abs(h).max())


def test_ransac_rng_replay_matches_numpy_choice(golden):
    """The PCG64 + Generator.choice replay K9 runs on the device reproduces
    the reference's hypothesis order (geometry.py:612)."""
    from oracle import ransac as orr
    g = golden("ransac")
    keys = [k for k in g.files if k.startswith("draws_")]
    assert len(keys) == 5
    for k in keys:
        _, n, seed = k.split("_")
        rp = orr.Pcg64Replay(int(seed))
        np.testing.assert_array_equal(np.array([rp.choice4(int(n)) for _ in range(len(g[k]))]), g[k], err_msg=k)


def test_ransac_host_walk_reproduces_sequential_loop(golden):
    """geometry.walk_counts over the full-budget counts picks the hypothesis
    the reference's adaptive loop keeps."""
    from oracle import ransac as orr
    from paper_2510_02080_b200.geometry import walk_counts
    from paper_2510_02080_b200.types import RansacConfig
    g = golden("ransac")
    for i in (0, 1, 21, 24, 28, 30, 35, 36, 37):
        src, dst, thr, conf, iters, seed = _ransac_case(g, i)
        counts = orr.hypotheses(src, dst, thr, iters, seed)
        b = walk_counts(counts, len(src), RansacConfig(pixel_threshold=thr, confidence=conf, max_iterations=iters,
                                                       seed=seed))
        if b < 0:
            assert float(g[f"c{i}_ratio"]) == 0.0
            continue
        rng = np.random.default_rng(seed)
        for _ in range(b + 1):
            smp = rng.choice(len(src), size=4, replace=False)
        h = orr.dlt(src[smp], dst[smp])
        best = orr.transfer_errors(h, src, dst) < thr
        assert int(best.sum()) == counts[b]
        # the reference's final mask is the refit's when it keeps at least as many
        assert g[f"c{i}_mask"].sum() >= best.sum()


def test_ransac_batched_walk_equals_per_row_walk():
    from paper_2510_02080_b200.geometry import walk_counts, walk_counts_batch
    from paper_2510_02080_b200.types import RansacConfig
    rng = np.random.default_rng(3)
    counts = rng.integers(-1, 60, size=(40, 300))
    counts[5] = -1
    counts[7, :] = 0
    ns = rng.integers(60, 200, size=40)
    cfg = RansacConfig(max_iterations=300)
    np.testing.assert_array_equal(walk_counts_batch(counts, ns, cfg),
                                  [walk_counts(counts[p], int(ns[p]), cfg) for p in range(40)])
