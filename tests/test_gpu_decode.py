"""§8(f) rank 3: the synthetic producer on the device (synth.DeviceDecoder
over ec3r_synthetic_decode) against the reference's SyntheticBackend.decode
(backend.py:228-281, render_depth scenesim.py:145-163) at 518 x 392 on the
reference's own world and trajectory (tests/golden/decode.npz, made by
make_golden.py from the unmodified reference):

  * noise-free decode: depth and confidence planes bit-exact (float32 of the
    reference's float64), gauge scale and relative poses exact;
  * noisy decode (sigma = 0.01): the same gauge and poses; the device noise
    is a Philox stream, so its xi = log(noisy / clean) / sigma is checked as
    a standard normal, and conf == 1 / (1 + |xi|), conf = 0 where depth <= 0.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2510_02080_b200.types import reference_module
    try:
        return dict(backend=reference_module("submap_slam.backend"), scenesim=reference_module("submap_slam.scenesim"))
    except ImportError:
        pytest.skip("the reference (baseline/_ref) is not installed")


def _backend(ref, sigma):
    rb, ss = ref["backend"], ref["scenesim"]
    world = ss.generate_world(ss.WorldConfig(room_size=(8.0, 8.0, 4.0), landmark_count=300), seed=0)
    traj = ss.generate_trajectory(ss.TrajectorySpec(kind="circle", frame_count=16, radius=2.0, step_bound=1.0), world,
                                  seed=0)
    cfg = rb.SyntheticBackendConfig(depth_resolution=(518, 392), focal=400.0, depth_noise_sigma=sigma)
    return rb.SyntheticBackend(world, traj, cfg, seed=100)


def _emb(ref, ids):
    return [ref["backend"].KeyframeEmbedding(i, np.zeros((1, 1))) for i in ids]


def test_device_decode_noise_free_bit_exact(golden, ref):
    from paper_2510_02080_b200 import synth
    g = golden("decode")
    be = _backend(ref, 0.0)
    np.testing.assert_array_equal(np.stack([p.rotation.q for p in be.trajectory]), g["traj_q"])
    dec = synth.DeviceDecoder(be)
    for call in range(2):
        ids = tuple(int(x) for x in g[f"clean{call}_ids"])
        out = dec.decode(_emb(ref, ids))
        assert out.call_index == call and out.frame_ids == ids
        assert be.injected_gauges[-1].scale == float(g[f"clean{call}_scale"])
        np.testing.assert_array_equal(out.depths.cpu().numpy(), g[f"clean{call}_depth"])
        np.testing.assert_array_equal(out.confidences.cpu().numpy(), g[f"clean{call}_conf"])
        np.testing.assert_array_equal(np.stack([p.rotation.q for p in out.poses]), g[f"clean{call}_pose_q"])
        np.testing.assert_array_equal(np.stack([p.translation for p in out.poses]), g[f"clean{call}_pose_t"])
        assert (out.depths > 0).float().mean().item() > 0.9


def test_device_decode_noise_statistics(golden, ref):
    from paper_2510_02080_b200 import synth
    g = golden("decode")
    clean = synth.DeviceDecoder(_backend(ref, 0.0))
    be = _backend(ref, 0.01)
    noisy = synth.DeviceDecoder(be)
    for call in range(2):
        ids = tuple(int(x) for x in g[f"noisy{call}_ids"])
        a = clean.decode(_emb(ref, ids))
        b = noisy.decode(_emb(ref, ids))
        assert be.injected_gauges[-1].scale == float(g[f"noisy{call}_scale"])
        np.testing.assert_array_equal(np.stack([p.translation for p in b.poses]), g[f"noisy{call}_pose_t"])
        d0, d1, c1 = a.depths.double(), b.depths.double(), b.confidences.double()
        hit = d0 > 0
        assert torch.equal(hit, d1 > 0) and torch.equal(c1 > 0, hit)
        xi = torch.log(d1[hit] / d0[hit]) / 0.01
        assert abs(xi.mean().item()) < 0.01 and abs(xi.std().item() - 1.0) < 0.01
        assert (c1[hit] - 1.0 / (1.0 + xi.abs())).abs().max().item() < 1e-4
    assert not torch.equal(b.depths, noisy.decode(_emb(ref, ids)).depths)  # next decode call: a new stream
