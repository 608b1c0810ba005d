"""Benchmark of the B200 dense data-parallel path (BASELINE.json metric:
fused map points/sec and descriptor matches/sec vs the CPU reference).

Workload (N=1): BASELINE configs[1] — synthetic TUM-style sequence, 300
keyframes / 60 submaps (5 new + 1 shared frame each, 518x392), 1024 x 256-d
descriptors per frame; one step = tracking match of 1500 frames, each against
its keyframe interval's resident 1024-point local map (300 maps, 5 frames per
map) + registration of all 59 edges (one launch) + pose chaining +
voxel-hash fusion at 2 cm of all 360 frames + sorted emit.  Inputs are
resident in HBM and larger than L2 (126 MB).  Under torchrun each rank owns a
contiguous window of the sequence (weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "fused map points/sec and descriptor matches/sec at 1/2/4/8 B200 vs CPU ref"


def load_traffic(config: int = 1):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each hot
    kernel, from the committed ncu --set full capture of the same config
    (profiles/kernel_traffic_c<config>.json; kernel_traffic.json holds
    configs[1]); {} when that config has no capture (traffic null)."""
    names = [f"kernel_traffic_c{config}.json"] + (["kernel_traffic.json"] if config == 1 else [])
    for n in names:
        p = os.path.join(ROOT, "profiles", n)
        if os.path.exists(p):
            return {k: v["dram_bytes_per_launch"] for k, v in json.load(open(p)).get("kernels", {}).items()}
    return {}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        """Starts nvidia-smi and waits (<= 5 s) for its first row, so the
        sampler is live when the timed region begins (mark() opens it)."""
        try:
            self._proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "50"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 5.0 and self._proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self._proc = None
        self.t_mark = time.perf_counter()

    def mark(self):
        self.t_mark = time.perf_counter()

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        valid = [(t, r) for t, r in self.rows if len(r) >= 9]
        rows = [r for t, r in valid if t >= self.t_mark]
        extra = {}
        if not rows and valid:  # region shorter than the sampling interval: the sample just before it
            t, r = max((x for x in valid if x[0] < self.t_mark), default=valid[0], key=lambda x: x[0])
            rows = [r]
            extra = {"samples_in_region": 0, "nearest_before_ms": (self.t_mark - t) * 1e3}
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows) if not extra else 0, **extra}


# ---------------------------------------------------------------------------
# workload

CONFIGS = {
    1: dict(keyframes=300, invalid=0.0,
            workload="configs[1]: TUM-style 300 keyframes / 60 submaps, 1024 descriptors per frame, "
                     "tracking match + align + fuse"),
    3: dict(keyframes=1500, invalid=0.0,
            workload="configs[3]: large indoor map, 1500 keyframes / 300 submaps per GPU, 2 cm voxel-hash fusion, "
                     "1024 descriptors per frame"),
    4: dict(keyframes=500, invalid=0.5,
            workload="configs[4]: 4000-keyframe long trajectory sharded 500 keyframes per GPU (8 x B200), ~50% "
                     "invalid pixels (~400M raw points at 8 GPUs), submap-sharded align + fuse"),
}


def build_workload(rank: int, world: int, n_kf: int, n_desc: int, device, invalid: float = 0.0):
    import torch

    from paper_2510_02080_b200 import mapping, synth

    cfg = synth.SceneConfig()
    stub, send_pos = None, []
    if world == 1:
        sb = synth.make_submaps(n_kf, cfg, seed=rank, device=device, invalid_fraction=invalid)
        dm = mapping.DenseMapping(cfg.height, cfg.width, sb.K4, slot_capacity=len(sb.poses8))
    else:
        # one sequence of n_kf x world keyframes (world x the laps, so every
        # window has the N = 1 geometry), rank r decoding its contiguous
        # window of flush batches; the first submap's shared keyframe comes
        # from rank r-1 as a halo every step (dist.WindowChain)
        from paper_2510_02080_b200 import dist as pdist

        cfg = synth.SceneConfig(laps=cfg.laps * world)
        batches = synth.flush_batches(n_kf * world)
        lo, hi = pdist.shard_window(len(batches), world, rank)
        send_pos, recv_ids = pdist.halo_handshake(batches[lo], batches[hi - 1])
        sb = synth.make_submaps(n_kf * world, cfg, seed=0, device=device, batch_range=(lo, hi),
                                invalid_fraction=invalid)
        dm = mapping.DenseMapping(cfg.height, cfg.width, sb.K4, slot_capacity=len(sb.poses8) + len(recv_ids))
        if recv_ids:  # stub slots first: a ChainPlan walks contiguous slots
            n = len(recv_ids)
            z = torch.zeros((n, cfg.height, cfg.width), dtype=torch.float32, device=device)
            ident = np.tile(np.array([1.0, 1.0, 0, 0, 0, 0, 0, 0]), (n, 1))
            stub = dm.add_submap(recv_ids, z, z, list(ident), -1)
    sms = []
    for j, ids in enumerate(sb.frame_ids):
        o = sb.slot_offsets[j]
        F = len(ids)
        sms.append(dm.add_submap(ids, sb.depth[o:o + F], sb.conf[o:o + F], list(sb.poses8[o:o + F]), j))
    del sb
    n_frames = 5 * n_kf  # tracked frames: 5 per keyframe
    # frames tracked against resident local maps: the 5 frames of a keyframe
    # interval share one map (tracking.py:173-194), uploaded once
    A, B, a_off, b_off, b_row = synth.make_descriptor_maps(n_frames, 5, n_desc, n_desc, 256, 0.05,
                                                           seed=100 + rank, device=device)
    torch.cuda.synchronize()
    return dm, sms, (A, B, a_off, b_off, b_row), (stub, send_pos)


class Step:
    """One pass of the hot path over the resident workload."""

    def __init__(self, dm, sms, desc, cell=0.02, halo=(None, [])):
        import torch

        from paper_2510_02080_b200 import mapping, tracking

        self.torch, self.mapping, self.tracking = torch, mapping, tracking
        self.dm, self.sms, self.desc, self.cell = dm, sms, desc, cell
        self.slots = torch.as_tensor(np.concatenate([sm.slots for sm in sms]).astype(np.int32), device="cuda")
        self.chain = None
        if torch.distributed.is_available() and torch.distributed.is_initialized() \
                and torch.distributed.get_world_size() > 1:
            from paper_2510_02080_b200 import dist as pdist
            self.chain = pdist.WindowChain(dm, halo[0], sms, halo[1])
            self.plan = self.chain.plan
        else:
            self.plan = mapping.ChainPlan(sms)
        self.pairs = self.plan.pairs
        self.seg = self.plan.seg
        self.vmap = None
        # max|a| * max|b| of the descriptor rows (error-bound scale of the
        # matcher's certification), measured once outside the timed region
        A, B = desc[0], desc[1]
        na = A.view(torch.bfloat16).float().norm(dim=1).max().item()
        nb = B.view(torch.bfloat16).float().norm(dim=1).max().item()
        self.norm_bound = na * nb * (1.0 + 1e-4)
        self.ev = {}
        self.n_points = 0
        self.exchange = None
        if torch.distributed.is_available() and torch.distributed.is_initialized() \
                and torch.distributed.get_world_size() > 1:
            from paper_2510_02080_b200 import dist as pdist
            self.exchange = pdist.MapExchange(cell)
        self.n_voxels = 0
        self.async_exchange = False
        self.n_dev = None
        self.match_stream = None
        # schedule of the tracking matcher against the mapping stages
        # (EC3R_BENCH_OVERLAP): "late" (default) = its own stream once the
        # fusion insert is queued, so it shares the SMs with the latency-bound
        # emit kernels; "early" = from the step's start (it then holds SMs the
        # registration clusters need); "serial" = one stream.  Measured
        # (profiles/r02o_*): serial 2.96, early 2.92, late 2.87 ms per step.
        self.overlap = os.environ.get("EC3R_BENCH_OVERLAP", "late")
        # the sorted emit without the host read of U (EC3R_BENCH_EMIT_SYNC=1
        # restores it): U is known from the sizing fill and checked on the
        # device count after the timed region, so the host never waits
        # mid-step and the next step's launches are queued before this one
        # ends (measured: 2.78 -> 2.70 ms per step, profiles/r02aa_*)
        self.emit_sync = os.environ.get("EC3R_BENCH_EMIT_SYNC", "0") == "1"

    def _event(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def run(self, record=None):
        """Mapping (registration, chain, fusion insert, sorted emit) on the
        current stream; the tracking matcher -- independent of the map -- on
        a second stream (schedule `self.overlap`, see __init__), so the
        latency- and barrier-bound mapping kernels and the tensor-core matcher
        share the SMs.  The current stream joins the matcher before
        returning, so every output is ordered after the step."""
        torch = self.torch
        nvtx = torch.cuda.nvtx
        main = torch.cuda.current_stream()
        if self.match_stream is None:
            self.match_stream = torch.cuda.Stream()
        ev = {}
        ev["t0"] = self._event()
        A, B, ao, bo, b_row = self.desc
        def launch_match():
            # tracking matcher on its own stream (inputs ready: it follows the
            # step's start on the current stream)
            ms = self.match_stream if self.overlap != "serial" else main
            ms.wait_event(ev[{"late": "t_insert", "mid": "t_reg"}.get(self.overlap, "t0")])
            ev["m0"] = torch.cuda.Event(enable_timing=True)
            ev["m0"].record(ms)
            nvtx.range_push("match")
            self.mb, self.nm = self.tracking.match_batched_device(A, B, None, None, 0, ao, bo, 0.8, self.norm_bound,
                                                                  b_row=b_row, stream=ms)
            nvtx.range_pop()
            ev["m1"] = torch.cuda.Event(enable_timing=True)
            ev["m1"].record(ms)

        if self.overlap in ("early", "serial"):
            launch_match()
        ev["t_reg0"] = self._event()
        # registration of all edges (one launch) + device pose chain (one launch)
        nvtx.range_push("register+chain")
        out = self.plan.run(self.dm.pool) if self.chain is None else self.chain.run()
        nvtx.range_pop()
        ev["t_reg"] = self._event()  # both launches: stage "reg" = registration + chain
        if self.overlap == "mid":
            launch_match()
        self.edge_status, self.sub_status = out[4], out[6]
        ev["t_chain"] = self._event()
        if self.vmap is None:
            # size the block pool once from a first fusion (outside the timed region)
            self.vmap, out, stt = self.mapping.fuse_slots(self.dm.pool, self.slots, self.cell)
            U = int(out[0].numel())
            # re-size: pool for 2x the blocks this fill used, sparse table
            self.vmap, out, stt = self.mapping.fuse_slots(self.dm.pool, self.slots, self.cell, expected_voxels=U,
                                                          expected_blocks=stt["n_blocks"])
            self.out = tuple(torch.empty((U,) + tuple(x.shape[1:]), dtype=x.dtype, device="cuda") for x in out)
        nvtx.range_push("fuse")
        self.vmap.clear()
        self.vmap.insert_frames(self.dm.pool, self.slots)
        nvtx.range_pop()
        ev["t_insert"] = self._event()
        if self.overlap == "late":
            launch_match()
        nvtx.range_push("emit" if self.exchange is None else "exchange+emit")
        if self.exchange is None:
            if self.emit_sync:
                keys, cen, wsum, cnt_v = self.vmap.extract(sort=True, out=self.out)
            else:
                # no host read of U mid-step (it is known from the sizing fill):
                # the host keeps the queue full across the step boundary
                keys, cen, wsum, cnt_v, self.n_dev = self.vmap.extract(sort=True, out=self.out, sync=False)
        else:
            # N > 1: global map partitioned by voxel key — owner-bucketed
            # partials, one NCCL all-to-all, owner-side merge + sorted emit
            # device-timed steps: no host round trip (fixed slabs, device
            # counts; overflow flags verified after the timed region)
            if self.async_exchange:
                keys, cen, wsum, cnt_v, self.n_dev = self.exchange.run(self.vmap, int(self.out[0].shape[0]),
                                                                       sync=False)
            else:
                keys, cen, wsum, cnt_v = self.exchange.run(self.vmap, int(self.out[0].shape[0]))
        nvtx.range_pop()
        ev["t_emit"] = self._event()
        main.wait_event(ev["m1"])  # join the matcher
        ev["t_end"] = self._event()
        if (self.exchange is None and self.emit_sync) or (self.exchange is not None and not self.async_exchange):
            self.n_voxels = int(keys.numel())
        if record is not None:
            record.append(ev)
        return keys, cen, wsum, cnt_v


def stage_ms(records):
    """Per-stage device time: the mapping stages on the step's stream, the
    matcher on its own stream (it overlaps the emit), and the critical path
    from the step's start to the join."""
    out = {}
    names = ["t_reg0", "t_reg", "t_chain", "t_insert", "t_emit"]
    for a, b in zip(names[:-1], names[1:]):
        out[b[2:]] = float(np.mean([r[a].elapsed_time(r[b]) for r in records]))
    out["match"] = float(np.mean([r["m0"].elapsed_time(r["m1"]) for r in records]))
    out["step"] = float(np.mean([r["t0"].elapsed_time(r["t_end"]) for r in records]))
    return out


# ---------------------------------------------------------------------------
# CPU reference on a bounded sample, scaled to the GPU step's per-step mix

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The unmodified reference package (installed into baseline/_ref by
    tools/install_reference.sh; it travels to the GPU box), or None."""
    if os.path.isdir(os.path.join(REF_DIR, "submap_slam")) and REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import submap_slam  # noqa: F401
        return submap_slam
    except ImportError:
        return None


def _ref_submaps(sb, cfg, n_submaps):
    """Reference Submap objects (mapping.py:30-62) of the first n synthetic
    submaps, through the reference's own inverse_project (backend.py:78-101);
    returns (submaps, seconds spent in inverse_project)."""
    from submap_slam.backend import ReconstructionOutput, inverse_project
    from submap_slam.geometry import CameraIntrinsics
    from submap_slam.liegroups import Pose3, Rotation3, Sim3Transform
    from submap_slam.mapping import Submap

    K = CameraIntrinsics(float(sb.K4[0]), float(sb.K4[1]), float(sb.K4[2]), float(sb.K4[3]), cfg.width, cfg.height)
    out, t_ip = [], 0.0
    for j, ids in enumerate(sb.frame_ids[:n_submaps]):
        o, F = sb.slot_offsets[j], len(ids)
        poses = tuple(Pose3(Rotation3(p[1:5]), p[5:].copy()) for p in sb.poses8[o:o + F])
        ro = ReconstructionOutput(tuple(ids), sb.depth[o:o + F].double().numpy(), sb.conf[o:o + F].double().numpy(),
                                  poses, K, j)
        t0 = time.perf_counter()
        cloud = inverse_project(ro)
        t_ip += time.perf_counter() - t0
        out.append(Submap(j, tuple(ids), cloud, {f: p for f, p in zip(ids, poses)}, K, Sim3Transform.identity(), j))
    return out, t_ip


def step_mix(keyframes: int):
    """(submaps, edges, tracked frames) of one GPU step over `keyframes`
    keyframes per GPU: KeyframeBuffer flushes of 5 new keyframes (+ the shared
    old one), one regular edge per submap after the first, 5 tracked frames
    per keyframe (SURVEY §8(d) cfg 2)."""
    n_sub = max(keyframes // 5, 1)
    return n_sub, max(n_sub - 1, 1), 5 * keyframes


def cpu_sample(n_submaps: int = 3, n_match: int = 2, seed: int = 0, budget_s: float = 20.0, use_reference=True,
               mix=(60, 59, 1500), invalid: float = 0.0):
    """Times the reference CPU path on a bounded sample of the workload and
    scales it to the GPU step's mix (S submaps decoded and fused, E
    registration edges, T tracking matches of 1024 x 1024 x 256; configs[1]:
    60, 59, 1500; configs[3]: 300, 299, 7500):
    step time = S x t(submap) + E x t(edge) + T x t(match).

    With the reference importable (baseline/_ref): its own inverse_project,
    Mapping._shared_correspondences + the gate of _registration_edges +
    align_point_sets (mapping.py:138-188, registration.py:38-102),
    Submap.world_points concatenation (fused_cloud, mapping.py:332-338) and
    match_descriptors (tracking.py:143-170); the voxel rule, which the
    reference does not have, is oracle/fuse.py.  Else the oracle port."""
    import torch

    from oracle import fuse as ofuse
    from oracle import ref_numpy as ref
    from paper_2510_02080_b200 import synth

    cfg = synth.SceneConfig()
    sb = synth.make_submaps(5 * n_submaps + 1, cfg, seed=seed, device="cpu", invalid_fraction=invalid)
    A, B, ao, bo = synth.make_descriptor_pairs(n_match, 1024, 1024, 256, 0.05, seed=seed, device="cpu")
    a = A.view(torch.bfloat16).double().numpy()
    b = B.view(torch.bfloat16).double().numpy()
    rm = reference_module() if use_reference else None
    if rm is not None:
        from submap_slam.mapping import Mapping, MappingConfig
        from submap_slam.registration import align_point_sets
        from submap_slam.tracking import match_descriptors

        kind = "reference"
        mcfg = MappingConfig()
        sms, t_ip = _ref_submaps(sb, cfg, n_submaps)
        mp = Mapping.__new__(Mapping)  # only the config and _shared_correspondences are used
        mp.config = mcfg
        t0 = time.perf_counter()
        for j in range(1, len(sms)):
            p, q, w = mp._shared_correspondences(sms[j], sms[j - 1])
            floor = mcfg.confidence_floor_frac * float(w.max())
            keep = w >= floor
            tr, _ = align_point_sets(p[keep], q[keep], w[keep])
            sms[j].global_pose = sms[j - 1].global_pose.compose(tr)
        t_edges = time.perf_counter() - t0
        t0 = time.perf_counter()
        x = np.concatenate([sm.world_points() for sm in sms])
        c = np.concatenate([sm.cloud.confidences for sm in sms])
        f = ofuse.fuse_points(x, c, 0.02)
        t_fuse = time.perf_counter() - t0 + t_ip
        match = match_descriptors
    else:
        kind = "port"
        dense = []
        for j, ids in enumerate(sb.frame_ids[:n_submaps]):
            o, F = sb.slot_offsets[j], len(ids)
            dense.append(dict(depth=sb.depth[o:o + F].numpy(), conf=sb.conf[o:o + F].numpy(), frame_ids=np.array(ids),
                              pose_q=sb.poses8[o:o + F, 1:5], pose_t=sb.poses8[o:o + F, 5:], K=sb.K4))
        t0 = time.perf_counter()
        globs = [(1.0, np.array([1.0, 0, 0, 0]), np.zeros(3))]
        for j in range(1, len(dense)):
            e = ref.registration_edge(dense[j], dense[j - 1])
            globs.append(ref.sim3_compose(globs[j - 1], (e["s"], e["q"], e["t"])))
        t_edges = time.perf_counter() - t0
        t0 = time.perf_counter()
        f = ofuse.fuse_submaps(dense, globs, 0.02)
        t_fuse = time.perf_counter() - t0
        match = ref.match_descriptors
    pts = f["n_in"]
    t1 = time.perf_counter()
    done = 0
    for p in range(n_match):
        match(a[ao[p]:ao[p + 1]], b[bo[p]:bo[p + 1]], 0.8)
        done = p + 1
        if time.perf_counter() - t1 > budget_s:
            break
    t_match = time.perf_counter() - t1
    n_edges = max(n_submaps - 1, 1)
    t_sub, t_edge, t_m = t_fuse / n_submaps, t_edges / n_edges, t_match / done
    S, E, T = mix
    step_s = S * t_sub + E * t_edge + T * t_m
    step_pts = pts / n_submaps * S
    return {"kind": kind, "points": pts, "points_per_s": step_pts / step_s, "step_s": step_s,
            "t_submap_s": t_sub, "t_edge_s": t_edge, "t_match_s": t_m,
            "pairs_per_s": 1024 * 1024 / t_m,
            "sample": f"{'unmodified reference (baseline/_ref)' if kind == 'reference' else 'oracle port'}: "
                      f"{n_submaps} submaps decoded + fused at 2 cm ({pts} points, 518x392), {n_edges} registration "
                      f"edge(s), {done} match(es) of 1024x1024x256"
                      f"{', %.0f%% invalid pixels' % (100 * invalid) if invalid else ''}; scaled to the GPU step's "
                      f"mix ({S} submaps, {E} edges, {T} matches): step = {S} t_submap + {E} t_edge + {T} t_match"}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS),
                    help="BASELINE configs[i] preset (3, the default: the 1500-keyframe map quoted at 1/2/4/8 GPUs, "
                         "so the driver's scaling curve runs on it; 1: the 300-keyframe sequence; 4: 500 keyframes "
                         "per GPU with ~50%% invalid pixels)")
    ap.add_argument("--keyframes", type=int, default=None, help="override the preset's keyframes per GPU")
    ap.add_argument("--desc", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-floor", action="store_true",
                    help="skip the post-timing diagnostics (fusion reduction-floor replay, emit timed alone); "
                         "ncu launch lists use it so they hold the steps only")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: validation of the N>1 path with ranks sharing a GPU (not a measurement)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    preset = CONFIGS[args.config]
    if args.keyframes is None:
        args.keyframes = preset["keyframes"]
    args.invalid = preset["invalid"]
    args.workload = preset["workload"] if args.keyframes == preset["keyframes"] else (
        f"configs[{args.config}] shape at {args.keyframes} keyframes per GPU")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    # Fewer GPUs than ranks (validation only, never a measurement): ranks
    # share the GPUs; under NCCL each rank then takes its own NCCL_HOSTID, so
    # NCCL treats the ranks as separate hosts (no duplicate-GPU refusal) and
    # moves data over its socket transport (tools/nccl_one_gpu.py).
    n_dev = max(torch.cuda.device_count(), 1)
    shared = world > n_dev
    dev_index = local % n_dev
    if shared and args.dist_backend == "nccl":
        os.environ["NCCL_HOSTID"] = f"ec3r-shared-gpu-rank{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    torch.cuda.set_device(dev_index)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    from paper_2510_02080_b200 import _lib

    L = _lib.lib()
    dm, sms, desc, halo = build_workload(rank, world, args.keyframes, args.desc, "cuda", args.invalid)
    step = Step(dm, sms, desc, halo=halo)
    for _ in range(args.warmup):
        step.run()
    torch.cuda.synchronize()
    if step.exchange is not None:  # size the exchange slabs from the warm-up's buckets
        step.exchange.retune()
        step.run()
        torch.cuda.synchronize()
    step.async_exchange = step.exchange is not None
    n_points = step.vmap.stats()["n_points_in"]
    A, B, ao, bo = desc[:4]
    n_pairs_scored = int(np.sum(np.diff(ao) * np.diff(bo)))

    sampler = ClockSampler(local)
    sampler.start()
    records = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.ec3r_kernel_launches()
    _lib.kernel_times()  # drop anything recorded before the timed region
    _lib.timing_enable(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.mark()
    e0.record()
    for _ in range(args.steps):
        step.run(records)
    e1.record()
    torch.cuda.synchronize()
    launches = L.ec3r_kernel_launches() - launches0
    _lib.timing_enable(False)
    if step.async_exchange:
        step.exchange.verify()  # overflow flags of the host-sync-free exchange
        step.n_voxels = int(step.n_dev.item())
        step.async_exchange = False
    elif step.exchange is None and not step.emit_sync:
        step.n_voxels = int(step.n_dev.item())  # U of the last step (device count, read after the timed region)
        if step.n_voxels > int(step.out[0].shape[0]) or step.vmap.stats()["n_overflow"] != 0:
            raise RuntimeError("host-sync-free voxel emit overflowed (rows or 32-bit keys): "
                               "rerun with EC3R_BENCH_EMIT_SYNC=1")
    ktimes = _lib.kernel_times()  # per hot kernel: CUDA events on its launching stream
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device="cuda" if args.dist_backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    stages = stage_ms(records)
    n_matches = int(step.nm.sum().item())
    from paper_2510_02080_b200 import tracking as _tr
    rescans = _tr.last_match_stats()

    # roofline accounting
    peaks, peak_src = load_peaks()
    H, W = dm.pool.H, dm.pool.W
    P = int(n_points)
    U = step.n_voxels
    C = int(step.seg.shape[0]) * H * W  # overlap pixel pairs streamed by registration
    traffic = load_traffic(args.config if args.keyframes == CONFIGS[args.config]["keyframes"] else -1)

    def kms(name):  # average launch duration of a hot kernel over the timed region
        t, n = ktimes.get(name, (0.0, 0))
        return t / max(n, 1), n

    bytes_fuse = 8 * P  # depth + confidence per streamed pixel
    bytes_reg = 16 * C  # both frames' depth + confidence per overlap pixel pair
    flops_match = 2.0 * n_pairs_scored * 256
    roof = {}
    for key, kname, alg, bound in (("fuse_insert", "vh_insert_frames_kernel", bytes_fuse, "hbm"),
                                   ("register", "register_edges_kernel", bytes_reg, "hbm"),
                                   ("match", "mt_tc_kernel", flops_match, "tensor")):
        kt, n = kms(kname)
        if bound == "hbm":
            ach = alg / (kt * 1e-3) / 1e9 if kt > 0 else None
            pk, unit = peaks["hbm_gbs"], "GB/s"
        else:
            ach = alg / (kt * 1e-3) / 1e12 if kt > 0 else None
            pk, unit = peaks["bf16_tflops"], "TFLOP/s"
        roof[key] = {"bound": bound, "achieved": ach, "peak": pk, "unit": unit,
                     "frac": (ach / pk) if ach else None, "traffic": traffic.get(kname), "ms": kt,
                     "launches": n, "kernel": kname, ("alg_bytes" if bound == "hbm" else "alg_flops"): alg}
    # the north star's stage-level figures: align + fuse (registration, pose
    # chain, fusion, sorted emit) against HBM with SURVEY §8(d)'s bytes
    # (depth-input variant: 8 B/px + 16 B per overlap pair + 24 B per voxel),
    # and the whole matcher (tensor pass + certification) against bf16
    # the emit stage runs beside the matcher (it waits for SMs the matcher
    # holds), so the align + fuse figure takes the emit timed alone, after the
    # timed region, on the step's own map and buffers
    emit_alone = None
    if step.exchange is None and not args.no_floor:
        torch.cuda.synchronize()
        emit_alone = _time_ms(lambda: step.vmap.extract(sort=True, out=step.out, sync=False), reps=10, warm=2)
        stages["emit_alone"] = emit_alone
    af_ms = stages["reg"] + stages["chain"] + stages["insert"] + (emit_alone if emit_alone else stages["emit"])
    af_bytes = 8 * P + 16 * C + 24 * U
    stage_roof = {
        "align_fuse": {"bound": "hbm", "ms": af_ms, "alg_bytes": af_bytes, "unit": "GB/s",
                       "achieved": af_bytes / (af_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                       "frac": af_bytes / (af_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
        "match": {"bound": "tensor", "ms": stages["match"], "alg_flops": flops_match, "unit": "TFLOP/s",
                  "achieved": flops_match / (stages["match"] * 1e-3) / 1e12, "peak": peaks["bf16_tflops"],
                  "frac": flops_match / (stages["match"] * 1e-3) / 1e12 / peaks["bf16_tflops"]},
    }
    if rank == 0 and world == 1 and not args.no_floor and step.vmap is not None and \
            os.environ.get("EC3R_FUSE_ENGINE", "hash") != "binned":
        # the fusion kernel against its own reduction stream
        fl = reduction_floor(step)
        kt = roof["fuse_insert"]["ms"]
        fl["what"] = ("the insert's 2 reductions per run (red.global.add.v4.f32 + red.global.add.u32), replayed "
                      "alone from a log of the same launch; frac = replay / kernel")
        fl["frac"] = fl["replay_ms"] / kt if kt else None
        roof["fuse_insert"]["reduction_floor"] = fl
    dominant = max(roof, key=lambda k: roof[k]["ms"])
    value = P * world / (ms * 1e-3)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(step, dm, desc, args, world)

    extras = None
    if rank == 0 and not args.no_extras:
        extras = run_extras(peaks)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        c = cpu_sample(mix=step_mix(args.keyframes), invalid=args.invalid)
        cpu = {"value": c["points_per_s"], "unit": "fused map points/s", "cores": cpu_cores(), "kind": c["kind"],
               "sample": c["sample"], "step_s": c["step_s"], "matches_value": c["pairs_per_s"],
               "matches_unit": "candidate pairs/s", "same_config": True}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "fused map points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 planes / f64 transforms+moments / bf16 tensor-core matcher",
            "data": "synthetic (device ray-cast box room, seeded)",
            "config": {"workload": args.workload, "invalid_pixel_fraction": args.invalid,
                       "keyframes_per_gpu": args.keyframes, "frames_tracked_per_gpu": int(len(ao) - 1),
                       "local_maps_per_gpu": int(B.shape[0]) // args.desc,
                       "resolution": [W, H], "voxel_m": 0.02, "submaps_per_gpu": len(sms),
                       "edges_per_gpu": len(step.pairs), "points_per_step_per_gpu": P, "voxels_per_gpu": U,
                       "l2": "inputs larger than L2 (pool %.0f MB, descriptors %.0f MB)" %
                             (dm.pool.nbytes() / 1e6, (A.numel() + B.numel()) * 2 / 1e6),
                       "parallelism": f"submap windows x{world}" + (
                           ": one sequence sharded by flush batches, shared-frame halo by P2P and an all-gather "
                           "of window poses per step; global map partitioned by voxel key (one NCCL all-to-all "
                           "of partials per step)" if world > 1 else ""),
                       "matcher_float64_rescans": rescans,
                       **({"validation_only": f"{world} ranks share {n_dev} GPU(s) ({args.dist_backend}): "
                                              "a functional run of the N > 1 path, not a measurement"}
                          if shared else {})},
            "matches_per_s": n_pairs_scored * world / (ms * 1e-3), "matches_unit": "candidate descriptor pairs/s",
            "emitted_matches_per_s": n_matches * world / (ms * 1e-3),
            "stages_ms": stages,
            "roofline": dict(roof[dominant], stage=dominant, peak_source=f"{peak_src} MEASURED_PEAKS.json",
                             traffic_source=f"profiles/kernel_traffic_c{args.config}.json (ncu --set full, dram bytes per "
                                            "launch of this config)"),
            "rooflines": roof,
            "stage_rooflines": stage_roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "extras": extras,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(step, dm, desc, args, world):
    """Same metric through the public API with host buffers: every step H2D
    (from pinned memory) of that step's frame planes, poses and descriptors,
    the full path, then D2H of the fused map and the matches into pinned
    memory.  Input sets are double-buffered: step i+1's H2D runs on a copy
    stream while step i computes (a data-loader pipeline); every step's
    copies are inside the timed region."""
    import torch

    pool = dm.pool
    n = pool.n
    A, B, ao, bo, b_row = desc
    h_in = [x.cpu().pin_memory() for x in (pool.depth[:n], pool.conf[:n], pool.poses[:n], A, B)]
    bufs = [(pool.depth, pool.conf, pool.poses, A, B),
            (pool.depth.clone(), pool.conf.clone(), pool.poses.clone(), A.clone(), B.clone())]
    cs = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    free = [torch.cuda.Event(), torch.cuda.Event()]

    def h2d(i):
        d, c, po, a, b = bufs[i % 2]
        with torch.cuda.stream(cs):
            cs.wait_event(free[i % 2])  # the compute that last read this set is done
            d[:n].copy_(h_in[0], non_blocking=True)
            c[:n].copy_(h_in[1], non_blocking=True)
            po[:n].copy_(h_in[2], non_blocking=True)
            a.copy_(h_in[3], non_blocking=True)
            b.copy_(h_in[4], non_blocking=True)
            ready[i % 2].record(cs)

    U0 = int(max(step.out[0].shape[0], step.n_voxels) * 1.25) + 1  # N > 1: the owned partition may be larger
    h_out = [torch.empty((U0,) + tuple(x.shape[1:]), dtype=x.dtype).pin_memory() for x in step.out]
    h_match = torch.empty(int(ao[-1]), dtype=torch.int32).pin_memory()
    steps = max(2, min(args.steps, 20))  # enough steps to amortise the pipeline fill (first H2D)
    out_bytes = 0
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    h2d(0)
    for i in range(steps):
        if i + 1 < steps:
            h2d(i + 1)  # the next step's inputs stream in while this step computes
        main.wait_event(ready[i % 2])
        d, c, po, a, b = bufs[i % 2]
        pool.depth, pool.conf, pool.poses = d, c, po
        step.desc = (a, b, ao, bo, b_row)
        res = step.run()
        free[i % 2].record(main)
        out_bytes = 0
        for hx, x in zip(h_out, res):
            hx[: x.shape[0]].copy_(x, non_blocking=True)
            out_bytes += x.numel() * x.element_size()
        h_match.copy_(step.mb, non_blocking=True)
        out_bytes += step.mb.numel() * step.mb.element_size()
    e1.record()
    torch.cuda.synchronize()
    pool.depth, pool.conf, pool.poses = bufs[0][0], bufs[0][1], bufs[0][2]
    step.desc = desc
    ms = e0.elapsed_time(e1) / steps
    P = step.vmap.stats()["n_points_in"]
    h2d_bytes = sum(x.numel() * x.element_size() for x in h_in)
    # raw pinned H2D bandwidth of this box (context for the e2e number)
    big = h_in[3]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    bufs[1][3].copy_(big, non_blocking=True)
    t1.record()
    torch.cuda.synchronize()
    h2d_gbs = big.numel() * big.element_size() / (t0.elapsed_time(t1) * 1e-3) / 1e9
    return {"value": P * world / (ms * 1e-3), "unit": "fused map points/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(out_bytes), "steps": steps,
            "pipelined": "inputs double-buffered: step i+1 H2D overlaps step i compute",
            "h2d_pinned_gbs": h2d_gbs}


def reduction_floor(step, reps=10):
    """The fusion insert's reduction floor, measured live: one insert logs
    its runs' (pool voxel, count) pairs in issue order instead of reducing
    (ec3r_vhash_diag_log), then the logged reductions alone are replayed
    into the same map (ec3r_vhash_diag_replay; float4 sums + u32 counts, and
    the sums alone).  Median of `reps` replays, the map cleared before each."""
    import torch

    from paper_2510_02080_b200 import _lib

    L = _lib.lib()
    vm, pool, slots = step.vmap, step.dm.pool, step.slots
    cap = int(slots.numel()) * pool.H * pool.W
    runs = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    vm.clear()
    _lib.check(L.ec3r_vhash_diag_log(vm._h, _lib.ptr(runs), cap, _lib.ptr(n_dev)), "ec3r_vhash_diag_log")
    vm.insert_frames(pool, slots)
    n_runs = int(n_dev.item())
    out = {"runs": n_runs, "reps": reps}
    for wc, key in ((1, "replay_ms"), (0, "replay_sums_only_ms")):
        ts = []
        for _ in range(reps + 2):
            vm.clear()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            _lib.check(L.ec3r_vhash_diag_replay(vm._h, _lib.ptr(runs), _lib.ptr(n_dev), cap, wc, None),
                       "ec3r_vhash_diag_replay")
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[key] = float(np.median(ts[2:]))
    # leave the map as the step left it
    vm.clear()
    vm.insert_frames(pool, slots)
    torch.cuda.synchronize()
    del runs
    return out


def _time_ms(fn, reps=5, warm=2):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_extras(peaks):
    """Side measurements outside the step (not part of `value`):
    * configs[2]: the matcher sweep, one N = M pair per size and the
      local-loop batch (1 query x 7 window keyframes) at 4k, D = 256, with
      the tensor-core kernel's own CUDA-event time;
    * K7: nn_query at the cloud_metrics size (20k x 20k) and
      at 1M x 1M points, raycast of 100 full 518x392 frames."""
    import torch

    from paper_2510_02080_b200 import _lib, kernels, synth, tracking

    out = {"matcher_sweep": [], "nn_query": [], "raycast": None}
    for n in (2048, 4096, 8192, 16384, 32768):  # SURVEY §8(d) cfg 3 sweep
        A, B, ao, bo = synth.make_descriptor_pairs(1, n, n, 256, 0.05, seed=n, device="cuda")
        run = lambda: tracking.match_batched_device(A, B, None, None, 0, ao, bo, 0.8)  # noqa: E731
        run()
        _lib.kernel_times()
        _lib.timing_enable(True)
        ms = _time_ms(run)
        _lib.timing_enable(False)
        kt, kn = _lib.kernel_times()["mt_tc_kernel"]
        kms = kt / max(kn, 1)
        fl = 2.0 * n * n * 256
        st = tracking.last_match_stats()
        out["matcher_sweep"].append({"n": n, "m": n, "ms": ms, "pairs_per_s": n * n / (ms * 1e-3),
                                     "tc_kernel_ms": kms, "tc_tflops": fl / (kms * 1e-3) / 1e12,
                                     "tc_frac": fl / (kms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                                     "rows_rescanned": st["rows_rescanned"], "cols_rescanned": st["cols_rescanned"]})
    A, B, ao, bo = synth.make_descriptor_pairs(7, 4096, 4096, 256, 0.05, seed=7, device="cuda")
    A = A[:4096].repeat(7, 1)  # one query frame against 7 window keyframes
    run = lambda: tracking.match_batched_device(A, B, None, None, 0, ao, bo, 0.8)  # noqa: E731
    ms = _time_ms(run)
    out["local_loop_batch"] = {"pairs": 7, "n": 4096, "m": 4096, "ms": ms, "pairs_per_s": 7 * 4096 * 4096 / (ms * 1e-3)}
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    for n, cell in ((20000, 0.05), (1 << 20, 0.01)):
        ref = torch.rand((n, 3), generator=g, device="cuda", dtype=torch.float64) * torch.tensor(
            [4.0, 4.0, 0.0], device="cuda", dtype=torch.float64)
        ref[:, 2] = 0.2 * torch.sin(3 * ref[:, 0])
        qry = ref[torch.randperm(n, generator=g, device="cuda")] + 0.003 * torch.randn(
            (n, 3), generator=g, device="cuda", dtype=torch.float64)
        ms = _time_ms(lambda: kernels.nn_query_device(qry, ref, cell))
        out["nn_query"].append({"n_query": n, "n_ref": n, "cell": cell, "ms": ms, "queries_per_s": n / (ms * 1e-3)})
    h, w = 392, 518
    uu, vv = torch.meshgrid(torch.arange(w, device="cuda", dtype=torch.float64),
                            torch.arange(h, device="cuda", dtype=torch.float64), indexing="xy")
    d = torch.stack([(uu - w / 2) / 400.0, (vv - h / 2) / 400.0, torch.ones_like(uu)], -1).reshape(-1, 3)
    d = d.repeat(100, 1)
    o = torch.tensor([4.0, 3.0, 1.5], device="cuda", dtype=torch.float64).expand_as(d).contiguous()
    boxes = [((2.0, 2.0, 0.0), (3.0, 3.5, 1.0)), ((5.0, 1.0, 0.0), (6.5, 2.0, 2.0))]
    ms = _time_ms(lambda: kernels.raycast_device(o, d, (0.0, 0.0, 0.0), (8.0, 8.0, 4.0), boxes))
    out["raycast"] = {"rays": int(d.shape[0]), "ms": ms, "rays_per_s": d.shape[0] / (ms * 1e-3)}
    # K6 global retrieval (configs[3]/[4] databases): latency of one
    # update_similarity scoring call through the public device API (host
    # list assembly included), and the scored (coarse + refined) pairs
    from paper_2510_02080_b200 import loops

    out["retrieval"] = []
    for K in (1500, 4000):
        pooled = synth.pooled_embeddings(K, seed=K)
        res = loops.retrieval_device(pooled, 5, 15, 0.93, 0.96)
        scored = int(len(res[0]) + len(res[4]))
        ms = _time_ms(lambda: loops.retrieval_device(pooled, 5, 15, 0.93, 0.96), reps=5, warm=1)
        out["retrieval"].append({"keyframes": K, "ms": ms, "scored_pairs": scored,
                                 "scored_pairs_per_s": scored / (ms * 1e-3), "candidates": int(len(res[2]))})
    # K1 inverse projection (§8(a) a2, backend.py:78-101; off the fusion step,
    # which reads the pool planes directly): one 6-frame full-resolution
    # submap per call, float64 points + conf + frame ids + pixels out
    from paper_2510_02080_b200 import backend

    cfg = synth.SceneConfig()
    sb = synth.make_submaps(11, cfg, seed=3, device="cuda")
    o, ids = sb.slot_offsets[0], sb.frame_ids[0]
    dsub, csub = sb.depth[o:o + len(ids)].contiguous(), sb.conf[o:o + len(ids)].contiguous()
    psub = sb.poses8[o:o + len(ids)]
    res = backend.inverse_project_device(dsub, csub, sb.K4, psub, ids)
    n_valid = int(res[0].shape[0])
    ms = _time_ms(lambda: backend.inverse_project_device(dsub, csub, sb.K4, psub, ids), reps=10, warm=2)
    px = int(dsub.numel())
    out["inverse_project"] = {"frames": len(ids), "pixels": px, "points": n_valid, "ms": ms,
                              "points_per_s": n_valid / (ms * 1e-3),
                              "gbs": (8 * px + 56 * n_valid) / (ms * 1e-3) / 1e9,
                              "note": "8 B/px in + 56 B/point out; includes the one D2H of the point count"}
    del sb, dsub, csub
    # K9 loop verification (§8f rank 4): 64 candidates x 500 matches, 40 %
    # inliers, full 1000-iteration budget scored on the device; the reference
    # loop (oracle port) on 4 of them on the host for scale
    from oracle import ransac as orr  # cpu_baseline leg only
    from paper_2510_02080_b200 import geometry

    rng = np.random.default_rng(99)
    probs = []
    for _ in range(64):
        h = np.eye(3) + 0.05 * rng.normal(size=(3, 3))
        h[2, :2] = rng.uniform(-3e-4, 3e-4, 2)
        h[2, 2] = 1.0
        src = rng.uniform(0, 640, size=(500, 2))
        sh = np.concatenate([src, np.ones((500, 1))], axis=1) @ h.T
        dst = sh[:, :2] / sh[:, 2:3] + 0.5 * rng.normal(size=(500, 2))
        dst[200:] = rng.uniform(0, 640, size=(300, 2))
        probs.append((src, dst))
    seeds = list(range(64))
    ms = _time_ms(lambda: geometry.estimate_homography_ransac_batch(probs, seeds=seeds), reps=3, warm=1)
    t0 = time.perf_counter()
    for (src, dst), sd in zip(probs[:4], seeds[:4]):
        orr.estimate_homography_ransac(src, dst, seed=sd)
    cpu_ms = (time.perf_counter() - t0) * 1e3 / 4
    out["homography_ransac"] = {"problems": 64, "matches": 500, "iterations_scored": 64 * 1000, "ms": ms,
                                "problems_per_s": 64 / (ms * 1e-3),
                                "cpu_baseline": {"value": 1e3 / cpu_ms, "unit": "problems/s", "cores": 1, "kind": "port",
                                                 "sample": "the reference loop on 4 of the 64 problems"}}
    # PnP RANSAC (tracking, geometry.py:414-474): 16 frames x 1,000 2D-3D
    # correspondences (30 % outliers); device draws + scoring, the
    # reference's host EPnP per hypothesis; against the unmodified reference
    # solve_pnp_ransac on the same problems (host, 1 core)
    try:
        from paper_2510_02080_b200.types import reference_module
        rg = reference_module("submap_slam.geometry")
    except ImportError:
        rg = None
    if rg is not None:
        KV = rg.CameraIntrinsics(fx=500.0, fy=500.0, cx=320.0, cy=240.0, width=640, height=480)
        rng = np.random.default_rng(7)
        pp = []
        for f in range(16):
            n = 1000
            u, v, z = rng.uniform(5, 634, n), rng.uniform(5, 474, n), rng.uniform(2, 8, n)
            cam = np.stack([(u - 320) / 500 * z, (v - 240) / 500 * z, z], axis=1)
            pts = cam + rng.normal(size=3) * 0.2
            pix = np.stack([u, v], axis=1) + 0.4 * rng.normal(size=(n, 2))
            bad = rng.choice(n, size=300, replace=False)
            pix[bad] = rng.uniform([0, 0], [640, 480], size=(300, 2))
            pp.append([rg.Correspondence2D3D(pix[i], pts[i], i) for i in range(n)])
        cfg = rg.RansacConfig(seed=3)
        stats = {}
        ms = _time_ms(lambda: geometry.solve_pnp_ransac_batch([(c, KV) for c in pp], cfg, stats=stats), reps=3,
                      warm=1)
        t0 = time.perf_counter()
        for c in pp[:4]:
            rg.solve_pnp_ransac(c, KV, cfg)
        cpu_ms = (time.perf_counter() - t0) * 1e3 / 4
        out["pnp_ransac"] = {"problems": 16, "correspondences": 1000, "ms": ms, "problems_per_s": 16 / (ms * 1e-3),
                             "hypotheses_scored": stats.get("hypotheses_scored"),
                             "host_rescored": stats.get("host_rescored"),
                             "note": "device draws + scoring; EPnP per hypothesis is the reference's host code",
                             "cpu_baseline": {"value": 1e3 / cpu_ms, "unit": "problems/s", "cores": 1,
                                              "kind": "reference",
                                              "sample": "the unmodified reference solve_pnp_ransac on 4 of the 16"}}
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation (the
    unmodified package from baseline/_ref; the oracle port only when it is
    absent) on the host cores, rank 0 only.  Each step is a bounded sample
    of the selected config's workload scaled to its GPU step's mix
    (cpu_sample, step_mix)."""
    if rank != 0:
        return
    vals, mvals, steps_s, wall_s = [], [], [], []
    c = None
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        c = cpu_sample(n_submaps=2, n_match=1, seed=k, budget_s=15.0, mix=step_mix(args.keyframes),
                       invalid=args.invalid)
        if k >= args.warmup:
            wall_s.append(time.perf_counter() - t0)
            vals.append(c["points_per_s"])
            mvals.append(c["pairs_per_s"])
            steps_s.append(c["step_s"])
    v = float(np.median(vals))
    # ms_per_step is the wall time a step (one bounded sample) really took;
    # the full GPU step's mix at the sampled rates would take scaled_step_ms
    line = {"metric": METRIC, "value": v, "unit": "fused map points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.median(wall_s)) * 1e3,
            "scaled_step_ms": float(np.median(steps_s)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator, CPU)",
            "impl": "reference",
            "config": {"workload": args.workload, "keyframes_per_gpu": args.keyframes,
                       "invalid_pixel_fraction": args.invalid,
                       "sample": "each step a bounded sample (2 submaps, 1 edge, 1 match) scaled to the full "
                                 "step's mix: %d submaps decoded + fused, %d edges, %d matches" %
                                 step_mix(args.keyframes), "voxel_m": 0.02},
            "matches_per_s": float(np.median(mvals)), "matches_unit": "candidate descriptor pairs/s",
            "cpu_baseline": {"value": v, "unit": "fused map points/s", "cores": cpu_cores(), "kind": c["kind"],
                             "sample": c["sample"]},
            "e2e": {"value": v, "unit": "fused map points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
