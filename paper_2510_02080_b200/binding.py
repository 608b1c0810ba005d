"""Runtime form of the maintainer binding of INTEGRATION.md §1: rebinds the
reference package's hot-path functions to this package's, in the defining
module and in every reference module that imported the name, so unmodified
reference code (its pipeline, its tests) runs through the B200 path.

    from paper_2510_02080_b200 import binding
    binding.install()        # submap_slam must be importable

Bindings (reference file:line -> this package):
  registration.align_point_sets / weighted_umeyama / normalize_confidences
      (registration.py:28-112)                 -> registration.*
  backend.inverse_project (backend.py:78-101)  -> backend.inverse_project
  tracking.match_descriptors / match_to_map (tracking.py:143-194)
                                               -> tracking.*
  loops.update_similarity / detect_local_candidates / verify_candidate
      (loops.py:114-153,184-243)               -> loops.*
  geometry.estimate_homography_ransac (geometry.py:594-640)
                                               -> geometry.estimate_homography_ransac
  geometry.solve_pnp_ransac (geometry.py:414-474, its EPnP / Gauss-Newton
      helpers stay the reference's)            -> geometry.solve_pnp_ransac
  _kernels.nn_query / nn_dists / raycast (_kernels/__init__.py:12-33)
                                               -> kernels.*
  mapping.Mapping (mapping.py:80-338)          -> mapping.b200_mapping_class(Mapping)
There is no fallback: install() raises when the library or a GPU is missing
(the reference's SUBMAP_SLAM_KERNELS=native contract).
"""

from __future__ import annotations

import importlib

_installed: list = []


def _targets():
    from . import backend, geometry, kernels, loops, mapping, registration, tracking

    return [
        ("registration", "align_point_sets", registration.align_point_sets,
         ("registration", "mapping", "geometry", "evaluation")),
        ("registration", "weighted_umeyama", registration.weighted_umeyama, ("registration",)),
        ("registration", "normalize_confidences", registration.normalize_confidences, ("registration",)),
        ("backend", "inverse_project", backend.inverse_project, ("backend", "mapping")),
        ("tracking", "match_descriptors", tracking.match_descriptors, ("tracking", "loops")),
        ("tracking", "match_to_map", tracking.match_to_map, ("tracking",)),
        ("loops", "update_similarity", loops.update_similarity, ("loops", "pipeline")),
        ("loops", "detect_local_candidates", loops.detect_local_candidates, ("loops", "pipeline")),
        ("loops", "verify_candidate", loops.verify_candidate, ("loops", "pipeline")),
        ("geometry", "estimate_homography_ransac", geometry.estimate_homography_ransac, ("geometry", "loops")),
        ("geometry", "solve_pnp_ransac", geometry.solve_pnp_ransac, ("geometry", "tracking")),
        ("_kernels", "nn_query", kernels.nn_query, ("_kernels", "evaluation")),
        ("_kernels", "nn_dists", kernels.nn_dists, ("_kernels", "evaluation")),
        ("_kernels", "raycast", kernels.raycast, ("_kernels",)),
        ("mapping", "Mapping", None, ("mapping", "pipeline")),
    ]


def install() -> list:
    """Rebind; returns the list of (module, name) rebound.  Idempotent."""
    if _installed:
        return list(_installed)
    from . import _lib
    from .mapping import b200_mapping_class

    _lib.lib()  # fail loudly without the library / a device
    for owner, name, fn, users in _targets():
        if fn is None:  # Mapping: subclass the reference class once
            base = getattr(importlib.import_module(f"submap_slam.{owner}"), name)
            fn = b200_mapping_class(base)
            fn.__name__ = fn.__qualname__ = "Mapping"
        for mod_name in users:
            mod = importlib.import_module(f"submap_slam.{mod_name}")
            if hasattr(mod, name):
                _installed.append((mod_name, name, getattr(mod, name)))
                setattr(mod, name, fn)
    return [(m, n) for m, n, _ in _installed]


def uninstall() -> None:
    while _installed:
        mod_name, name, orig = _installed.pop()
        setattr(importlib.import_module(f"submap_slam.{mod_name}"), name, orig)
