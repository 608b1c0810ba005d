"""Drop-in for the reference's native-kernel plugin slot ``submap_slam._kernels``
(``_kernels/__init__.py:12-33``): ``raycast``, ``nn_query`` and ``nn_dists``
with the numpy-in / numpy-out semantics of ``_kernels/_numpy.py``, computed by
K7 (``csrc/nn.cu``) on the B200 and bit-identical to the reference.

The reference looks for a compiled module ``_core`` exporting exactly these
three names; INTEGRATION.md shows the two-line alias a maintainer adds so
that ``SUBMAP_SLAM_KERNELS=native`` picks this module.  ``*_device`` variants
take and return CUDA tensors (no host round trip) for callers that keep their
clouds on the GPU.  There is no CPU fallback: without CUDA every call raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

BACKEND = "b200"


def backend_name() -> str:
    return BACKEND


def _dev_f64(x) -> torch.Tensor:
    t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, 3)))
    return t.to("cuda", non_blocking=False)


def nn_query_device(query: torch.Tensor, ref: torch.Tensor, cell_size: float, stream=None):
    """query (nq, 3), ref (nr, 3) float64 CUDA tensors -> (dist (nq,) float64,
    idx (nq,) int64) CUDA tensors (nn_query, _numpy.py:66-132)."""
    L = _lib.lib()
    query = query.reshape(-1, 3).to(torch.float64).contiguous()
    ref = ref.reshape(-1, 3).to(torch.float64).contiguous()
    nq, nr = int(query.shape[0]), int(ref.shape[0])
    dist = torch.empty(nq, dtype=torch.float64, device=query.device)
    idx = torch.empty(nq, dtype=torch.int64, device=query.device)
    if nq == 0:
        return dist, idx
    ws = _lib.workspace(L.ec3r_nn_workspace(nr, nq), query.device, "nn")
    _lib.check(L.ec3r_nn_query(_lib.ptr(query), nq, _lib.ptr(ref) if nr else None, nr, float(cell_size),
                               _lib.ptr(dist), _lib.ptr(idx), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)),
               "ec3r_nn_query")
    return dist, idx


def nn_query(query, ref, cell_size):
    """Directed nearest neighbours query -> ref via grid hashing; returns
    (distances float64, ref_indices int64) exactly as _numpy.nn_query."""
    _lib.lib()
    q = np.asarray(query, dtype=float).reshape(-1, 3)
    r = np.asarray(ref, dtype=float).reshape(-1, 3)
    if len(q) == 0:
        return np.zeros(0), np.zeros(0, dtype=np.int64)
    d, i = nn_query_device(_dev_f64(q), _dev_f64(r), cell_size)
    return d.cpu().numpy(), i.cpu().numpy()


def nn_dists(query, ref, cell_size):
    """Directed nearest-neighbour distances query -> ref (see nn_query)."""
    return nn_query(query, ref, cell_size)[0]


def raycast_device(origins: torch.Tensor, dirs: torch.Tensor, room_min, room_max, boxes, stream=None):
    L = _lib.lib()
    origins = origins.reshape(-1, 3).to(torch.float64).contiguous()
    dirs = dirs.reshape(-1, 3).to(torch.float64).contiguous()
    solids = [(room_min, room_max)] + [(a, b) for a, b in boxes]
    sol = np.ascontiguousarray(np.concatenate([np.concatenate([np.asarray(a, float).reshape(3),
                                                               np.asarray(b, float).reshape(3)])
                                               for a, b in solids]).reshape(-1, 6))
    n = int(origins.shape[0])
    out = torch.empty(n, dtype=torch.float64, device=origins.device)
    _lib.check(L.ec3r_raycast(_lib.ptr(origins), _lib.ptr(dirs), n, sol.ctypes.data, len(solids), _lib.ptr(out),
                              _lib.stream_ptr(stream)), "ec3r_raycast")
    return out


def raycast(origins, dirs, room_min, room_max, boxes):
    """First-hit ray parameter against the room shell and solid boxes; 0
    where a ray hits nothing (_numpy.raycast semantics)."""
    _lib.lib()
    o = _dev_f64(origins)
    d = _dev_f64(dirs)
    return raycast_device(o, d, room_min, room_max, list(boxes)).cpu().numpy()
