"""ctypes binding of the C ABI (include/ec3r_b200.h) — the only way this
package reaches the GPU.  There is no CPU fallback: a missing library or a
machine without CUDA raises immediately."""

from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EC3R_B200_LIB", os.path.join(_HERE, "libec3r_b200.so"))

ST_OK, ST_SKIP, ST_TOO_FEW, ST_ALL_ZERO, ST_DEGENERATE, ST_NONPOS_SCALE = range(6)

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double
_SZ = C.c_size_t

# name -> (restype, argtypes)
_PROTOS = {
    "ec3r_abi_version": (_I, []),
    "ec3r_kernel_launches": (C.c_uint64, []),
    "ec3r_timing_enable": (None, [_I]),
    "ec3r_timing_get": (_I, [_I, _P, _P]),
    "ec3r_sim3_apply": (_I, [_P, _I64, _P, _P, _P]),
    "ec3r_last_error": (C.c_char_p, []),
    "ec3r_inverse_project_workspace": (_SZ, [_I, _I, _I]),
    "ec3r_inverse_project": (_I, [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ec3r_inverse_project_f64": (_I, [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ec3r_register_edges_workspace": (_SZ, [_I]),
    "ec3r_register_edges": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _I, _D, _I, _I, _P, _P, _P, _P, _P, _P,
                                 _P, _SZ, _P]),
    "ec3r_chain_poses": (_I, [_P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P]),
    "ec3r_umeyama_workspace": (_SZ, [_I]),
    "ec3r_umeyama_batched": (_I, [_P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _SZ, _P]),
    "ec3r_vhash_create": (_I, [C.POINTER(_P), _I64, _D, _P]),
    "ec3r_vhash_create_sized": (_I, [C.POINTER(_P), _I64, _I64, _I64, _D, _P]),
    "ec3r_vhash_destroy": (_I, [_P]),
    "ec3r_vhash_capacity": (_I64, [_P]),
    "ec3r_vhash_clear": (_I, [_P, _P]),
    "ec3r_vhash_diag_log": (_I, [_P, _P, _I64, _P]),
    "ec3r_vhash_diag_replay": (_I, [_P, _P, _P, _I64, _I, _P]),
    "ec3r_vhash_insert_frames": (_I, [_P, _P, _P, _I, _I, _P, _P, _P, _P, _I, _P]),
    "ec3r_vhash_insert_points": (_I, [_P, _P, _P, _I64, _P, _P]),
    "ec3r_vhash_stats_get": (_I, [_P, _P, _P]),
    "ec3r_vhash_count": (_I, [_P, _P, _P]),
    "ec3r_vhash_extract_workspace": (_SZ, [_P]),
    "ec3r_vhash_extract": (_I, [_P, _P, _P, _P, _P, _P, _I, _P, _SZ, _P]),
    "ec3r_vhash_extract_count": (_I64, [_P]),
    "ec3r_vhash_extract_partials": (_I, [_P, _I, _P, _P, _P, _P, _P, _SZ, _P]),
    "ec3r_vhash_merge_partials": (_I, [_P, _P, _P, _P, _I64, _P]),
    "ec3r_vhash_extract_partials_fixed": (_I, [_P, _I, _I64, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "ec3r_vhash_merge_partials_slabs": (_I, [_P, _P, _P, _P, _I, _I64, _P, _P]),
    "ec3r_vhash_stats_device": (_I, [_P, _P, _P]),
    "ec3r_match_workspace": (_SZ, [_P, _P, _I]),
    "ec3r_match_batched": (_I, [_P, _P, _P, _P, _I, _P, _P, _I, _I, _D, _D, _P, _P, _P, _SZ, _P]),
    "ec3r_match_batched_rows": (_I, [_P, _P, _P, _P, _I, _P, _P, _P, _I64, _I, _I, _D, _D, _P, _P, _P, _SZ, _P]),
    "ec3r_match_stats": (_I, [_P, _I64, _I64, _I, _P, _P, _P]),
    "ec3r_retrieval": (_I, [_P, _I, _I, _I, _I, _D, _D, _P, _P, _P, _P, _P, _P, _I64, _P, _I, _I, _P,
                            _SZ, _P]),
    "ec3r_retrieval_workspace": (_SZ, [_I, _I, _I64]),
    "ec3r_nn_workspace": (_SZ, [_I64, _I64]),
    "ec3r_nn_query": (_I, [_P, _I64, _P, _I64, _D, _P, _P, _P, _SZ, _P]),
    "ec3r_raycast": (_I, [_P, _P, _I64, _P, _I, _P, _P]),
    "ec3r_synthetic_decode": (_I, [_P, _I, _P, _I, _I, _I, _P, _D, _D, C.c_uint64, _P, _P, _P]),
    "ec3r_apply_window_offset": (_I, [_P, _I, _I, _P, _I, _P, _I64, _P, _P]),
    "ec3r_homography_workspace": (_SZ, [_I, _I]),
    "ec3r_homography_ransac_score": (_I, [_P, _P, _P, _I, _P, _I, _D, _P, _P, _P, _SZ, _P]),
    "ec3r_homography_ransac_refit": (_I, [_P, _P, _P, _I, _P, _I, _D, _P, _P, _P, _P, _SZ, _P]),
    "ec3r_ransac_draws_workspace": (_SZ, [_I]),
    "ec3r_ransac_draws": (_I, [_P, _I, _P, _I, _P, _P, _SZ, _P]),
    "ec3r_pnp_score": (_I, [_P, _P, _P, _P, _P, _P, _I, _D, _D, _P, _P, _P, _P]),
    "ec3r_local_candidates_workspace": (_SZ, [_I]),
    "ec3r_local_candidates": (_I, [_P, _I64, _P, _I, _P, _D, _P, _P, _P, _SZ, _P]),
    "ec3r_local_candidates_ex": (_I, [_P, _I64, _P, _I, _P, _D, _P, _P, _P, _I64, _P, _P, _SZ, _P]),
}

EXPORTED = tuple(_PROTOS)


class VHashStats(C.Structure):
    _fields_ = [("n_points_in", _I64), ("n_out_of_range", _I64), ("n_overflow", _I64),
                ("n_slow_path", _I64), ("n_blocks", _I64)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library and bind every prototype (no CUDA needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make` (or __graft_entry__.build()); "
            "the B200 path has no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    """The bound library, after checking that a CUDA device is present."""
    L = load()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_02080_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.ec3r_last_error().decode() if _lib is not None else ""
        names = {-1: "CUDA error", -2: "invalid argument", -3: "workspace too small", -4: "out of memory"}
        raise RuntimeError(f"{what} failed: {names.get(rc, rc)} {msg}")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    """Device (or host) address of a tensor / numpy array, None for None."""
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return t.ctypes.data


_ws_cache: dict = {}


def workspace(nbytes: int, device=None, tag: str = "default") -> torch.Tensor:
    """Reusable per-(device, tag) byte workspace from torch's caching allocator."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (dev, tag)
    buf = _ws_cache.get(key)
    nbytes = max(int(nbytes), 256)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    return buf


TIMED_KERNELS = ("mt_tc_kernel", "register_edges_kernel", "vh_insert_frames_kernel")


def timing_enable(on: bool = True) -> None:
    """Record CUDA events around the three hot kernels' launches (on their
    launching streams); read and clear with kernel_times()."""
    lib().ec3r_timing_enable(1 if on else 0)


def kernel_times() -> dict:
    """{kernel name: (total ms, launches)} since the last call."""
    L = lib()
    out = {}
    for k, name in enumerate(TIMED_KERNELS):
        ms, n = C.c_double(), C.c_int64()
        check(L.ec3r_timing_get(k, C.byref(ms), C.byref(n)), "ec3r_timing_get")
        out[name] = (ms.value, n.value)
    return out

