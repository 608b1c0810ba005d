"""B200-native (sm_100a) dense data-parallel path of EC3R-SLAM
(arxiv 2510.02080), behind the reference ``submap_slam`` API.

Modules mirror the reference modules they replace on the hot path:
  registration  align_point_sets / weighted_umeyama   (registration.py)
  backend       inverse_project, FramePool             (backend.py)
  mapping       batched registration edges, voxel fusion, Mapping drop-in
  tracking      match_descriptors / match_to_map       (tracking.py)
  loops         update_similarity                      (loops.py)
  dist          multi-GPU sharding (one process per GPU, NCCL)
All compute goes through the C ABI in include/ec3r_b200.h
(libec3r_b200.so); there is no CPU fallback.
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401
