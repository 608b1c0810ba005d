"""Drop-in proof: the reference's OWN test suites (pkg/tests, installed with
the package into baseline/_ref by tools/install_reference.sh) run with the
reference's hot-path names rebound to this package (binding.install(), the
runtime form of INTEGRATION.md §1).  Every call those tests make to
align_point_sets, inverse_project, match_descriptors, update_similarity,
detect_local_candidates, verify_candidate, estimate_homography_ransac,
nn_query / raycast and Mapping then goes through the CUDA path."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITES = ["test_registration.py", "test_mapping.py", "test_tracking.py", "test_loops.py", "test_backend.py",
          "test_geometry.py", "test_evaluation.py"]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "ref_tests")), reason="reference not installed in baseline/_ref")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_through_binding(suite):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, REF]), EC3R_REFERENCE_SRC=REF)
    cmd = [sys.executable, "-m", "pytest", os.path.join("ref_tests", suite), "-p", "no:cacheprovider",
           "-p", "tests.ref_binding_plugin", "--rootdir", REF]
    r = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-40:])
    assert r.returncode == 0, tail
    assert "rebound" in r.stdout, tail
    print(tail)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "submap_slam")), reason="reference not installed in baseline/_ref")
def test_reference_pipeline_end_to_end_through_binding():
    """The reference Pipeline, unmodified, on its numpy path and then bound
    to the B200 path: identical decisions and events, poses within 1e-5,
    fused cloud within 1e-6 m (tests/dropin_pipeline.py)."""
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, REF]), EC3R_REFERENCE_SRC=REF)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dropin_pipeline.py"), "150"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-30:])
    assert r.returncode == 0, tail
    print(tail)
