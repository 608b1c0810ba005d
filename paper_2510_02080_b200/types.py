"""Value types and exception taxonomy of the reference API.

When the reference package ``submap_slam`` is importable (the integration
case: this package is bound into the reference's host code), its own classes
are re-exported so every value returned here IS a reference object
(Sim3Transform, Rotation3, SubmapCloud, the exception types ...).  On a
machine without the reference (e.g. the GPU test box) the same names resolve
to minimal mirrors with the same constructors, attributes and the operations
this path uses.  Only value types live here — there is no compute dispatch.

Mirrors follow liegroups.py:43-281, backend.py:51-68, geometry.py:28-45 and
errors.py:4-65.
"""

from __future__ import annotations

import math
import os
import sys
from dataclasses import dataclass

import numpy as np

_src = os.environ.get("EC3R_REFERENCE_SRC")
if _src and _src not in sys.path:
    sys.path.append(_src)

try:  # pragma: no cover - exercised when the reference is installed
    from submap_slam import errors as _ref_errors
    from submap_slam.backend import ReconstructionOutput, SubmapCloud
    from submap_slam.geometry import CameraIntrinsics
    from submap_slam.liegroups import Pose3, Rotation3, Sim3Transform

    SubmapSlamError = _ref_errors.SubmapSlamError
    TooFewCorrespondences = _ref_errors.TooFewCorrespondences
    DegenerateConfiguration = _ref_errors.DegenerateConfiguration
    AllZeroConfidence = _ref_errors.AllZeroConfidence
    NoSharedKeyframes = _ref_errors.NoSharedKeyframes
    MissingEmbedding = _ref_errors.MissingEmbedding
    NoConsensus = _ref_errors.NoConsensus
    REFERENCE_TYPES = True
except ImportError:
    REFERENCE_TYPES = False

    class SubmapSlamError(Exception):
        """errors.py:4"""

    class TooFewCorrespondences(SubmapSlamError):
        """errors.py:12"""

    class DegenerateConfiguration(SubmapSlamError):
        """errors.py:20"""

    class AllZeroConfidence(SubmapSlamError):
        """errors.py:24"""

    class NoSharedKeyframes(SubmapSlamError):
        """errors.py:52"""

    class MissingEmbedding(SubmapSlamError):
        """errors.py:48"""

    class NoConsensus(SubmapSlamError):
        """errors.py:16"""

    def _quat_mul(a, b):
        aw, ax, ay, az = a
        bw, bx, by, bz = b
        return np.array([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                         aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw])

    def _quat_rotate(q, pts):
        w = q[0]
        v = q[1:]
        uv = 2.0 * np.cross(v, pts)
        return pts + w * uv + np.cross(v, uv)

    def _matrix_to_quat(m):
        t = np.trace(m)
        if t > 0:
            r = math.sqrt(1.0 + t)
            s = 0.5 / r
            q = np.array([0.5 * r, (m[2, 1] - m[1, 2]) * s, (m[0, 2] - m[2, 0]) * s, (m[1, 0] - m[0, 1]) * s])
        else:
            i = int(np.argmax(np.diag(m)))
            j, k = (i + 1) % 3, (i + 2) % 3
            r = math.sqrt(1.0 + m[i, i] - m[j, j] - m[k, k])
            s = 0.5 / r
            q = np.empty(4)
            q[0] = (m[k, j] - m[j, k]) * s
            q[1 + i] = 0.5 * r
            q[1 + j] = (m[j, i] + m[i, j]) * s
            q[1 + k] = (m[k, i] + m[i, k]) * s
        return q / np.linalg.norm(q)

    @dataclass(frozen=True, eq=False)
    class Rotation3:
        q: np.ndarray

        def __post_init__(self):
            q = np.asarray(self.q, dtype=float)
            q = q / np.linalg.norm(q)
            q.flags.writeable = False
            object.__setattr__(self, "q", q)

        @staticmethod
        def identity():
            return Rotation3(np.array([1.0, 0.0, 0.0, 0.0]))

        @staticmethod
        def from_matrix(m):
            return Rotation3(_matrix_to_quat(np.asarray(m, dtype=float)))

        def matrix(self):
            w, x, y, z = self.q
            return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                             [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                             [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])

        def apply(self, pts):
            return _quat_rotate(self.q, np.asarray(pts, dtype=float))

        def compose(self, other):
            return Rotation3(_quat_mul(self.q, other.q))

        def inverse(self):
            return Rotation3(np.array([self.q[0], -self.q[1], -self.q[2], -self.q[3]]))

        def approx_equal(self, other, tol=1e-9):
            d = min(np.linalg.norm(self.q - other.q), np.linalg.norm(self.q + other.q))
            return float(d) <= tol

    @dataclass(frozen=True, eq=False)
    class Pose3:
        rotation: Rotation3
        translation: np.ndarray

        def __post_init__(self):
            t = np.asarray(self.translation, dtype=float).reshape(3).copy()
            t.flags.writeable = False
            object.__setattr__(self, "translation", t)

        @staticmethod
        def identity():
            return Pose3(Rotation3.identity(), np.zeros(3))

        def apply(self, pts):
            return self.rotation.apply(pts) + self.translation

        def compose(self, other):
            return Pose3(self.rotation.compose(other.rotation),
                         self.rotation.apply(other.translation) + self.translation)

        def inverse(self):
            rinv = self.rotation.inverse()
            return Pose3(rinv, -rinv.apply(self.translation))

        def to_sim3(self):
            return Sim3Transform(1.0, self.rotation, self.translation)

    @dataclass(frozen=True, eq=False)
    class Sim3Transform:
        scale: float
        rotation: Rotation3
        translation: np.ndarray

        def __post_init__(self):
            s = float(self.scale)
            if not s > 0:
                raise ValueError(f"scale must be positive, got {s}")
            object.__setattr__(self, "scale", s)
            t = np.asarray(self.translation, dtype=float).reshape(3).copy()
            t.flags.writeable = False
            object.__setattr__(self, "translation", t)

        @staticmethod
        def identity():
            return Sim3Transform(1.0, Rotation3.identity(), np.zeros(3))

        def matrix(self):
            out = np.eye(4)
            out[:3, :3] = self.scale * self.rotation.matrix()
            out[:3, 3] = self.translation
            return out

        def apply(self, pts):
            return self.scale * self.rotation.apply(pts) + self.translation

        def compose(self, other):
            return Sim3Transform(self.scale * other.scale, self.rotation.compose(other.rotation),
                                 self.scale * self.rotation.apply(other.translation) + self.translation)

        def inverse(self):
            rinv = self.rotation.inverse()
            sinv = 1.0 / self.scale
            return Sim3Transform(sinv, rinv, -sinv * rinv.apply(self.translation))

    @dataclass(frozen=True, eq=False)
    class CameraIntrinsics:
        fx: float
        fy: float
        cx: float
        cy: float
        width: int
        height: int

    @dataclass(frozen=True, eq=False)
    class ReconstructionOutput:
        frame_ids: tuple
        depths: np.ndarray
        confidences: np.ndarray
        poses: tuple
        intrinsics: CameraIntrinsics
        call_index: int = -1

    @dataclass(frozen=True, eq=False)
    class SubmapCloud:
        points: np.ndarray
        confidences: np.ndarray
        frame_ids: np.ndarray
        pixels: np.ndarray


try:  # pragma: no cover
    from submap_slam.geometry import RansacConfig, RansacResult
except ImportError:
    @dataclass
    class RansacConfig:
        """geometry.py:59-66."""

        pixel_threshold: float = 2.0
        confidence: float = 0.999
        max_iterations: int = 1000
        min_inliers: int = 10
        min_parallax_deg: float = 1.0
        seed: int = 0

    @dataclass
    class RansacResult:
        """geometry.py:69-73."""

        model: object
        inlier_mask: np.ndarray
        inlier_ratio: float


try:  # pragma: no cover
    from submap_slam.geometry import Correspondence2D3D
except ImportError:
    @dataclass(frozen=True, eq=False)
    class Correspondence2D3D:
        """geometry.py:52-56."""

        pixel: np.ndarray
        point: np.ndarray
        point_id: int = -1


def sim3_to_vec(t) -> np.ndarray:
    """Any Sim3Transform / Pose3 -> the ABI's 8 doubles {s, q(4), t(3)}."""
    s = float(getattr(t, "scale", 1.0))
    return np.concatenate([[s], np.asarray(t.rotation.q, float), np.asarray(t.translation, float)])


def vec_to_sim3(v) -> "Sim3Transform":
    v = np.asarray(v, dtype=float)
    return Sim3Transform(float(v[0]), Rotation3(v[1:5]), v[5:8])


def intrinsics_vec(k) -> np.ndarray:
    return np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)


def reference_module(name: str):
    """A module of the reference package (host code this path delegates to:
    EPnP / Gauss-Newton, pose-graph LM), importable as installed, from
    EC3R_REFERENCE_SRC, or from the offline install under baseline/_ref."""
    import importlib

    try:
        return importlib.import_module(name)
    except ImportError:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        for p in (os.environ.get("EC3R_REFERENCE_SRC"), os.path.join(root, "baseline", "_ref")):
            if p and os.path.isdir(p) and p not in sys.path:
                sys.path.append(p)
        return importlib.import_module(name)
