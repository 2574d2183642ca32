"""GPU: the blend's two record-staging engines (vrs_set_staging_mode) --
block threads (LDG + STS) and the Tensor Memory Accelerator (cp.async.bulk
into shared memory, mbarrier completion) -- give bit-identical frames and
counters, and the TMA path meets the oracle bars on its own."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg
from helpers import identity_camera
from test_gpu_parity import _quest_workload, assert_images_close, assert_lists_equal, render_both

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vrs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    import paper_2505_10144_b200 as p
    return p


def _frame(vrs, scene, cams, fov, T, masks, mode, projection=0, max_pairs=1 << 22):
    W, H = max(c.width for c in cams), max(c.height for c in cams)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=len(cams), max_pairs=max_pairs, max_width=W, max_height=H,
                     assign_tile=T, projection=projection)
    r.upload(scene)
    for slot, m in (masks or {}).items():
        r.set_mask(slot, m)
    r.vrs_set_instrumentation(counters=1)
    r.vrs_set_staging_mode(mode)
    rgba, depth = r.render(cams, fov)
    torch.cuda.synchronize()
    out = (rgba.cpu().numpy().copy(), depth.cpu().numpy().copy(), r.stats())
    r.close()
    return out


def test_tma_staging_oracle_parity_foveated_masked_stereo(vrs, oracle_mod):
    scene = sg.vr_room(7, 20000, sh_degree=3)
    W, H = 320, 256
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
            for e, x in enumerate((-0.0315, 0.0315))]
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10)] * 2
    masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)}
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, masks=masks, staging=1)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    st, ost = r.stats(), o.stats()
    for k in ("evaluations", "contributions", "overflow_samples", "terminated_samples"):
        assert st[k] == ost[k], k


@pytest.mark.parametrize("projection", [0, 1])
def test_tma_staging_c1_seeds(vrs, oracle_mod, projection):
    for seed in range(3):
        scene = sg.random_scene(seed, n=1000)
        r, o, g, oi = render_both(vrs, oracle_mod, scene, [identity_camera(128, 128, 64.0)], T=16,
                                  projection=projection, staging=1)
        assert_lists_equal(r, o)
        assert_images_close(g, oi)


def test_tma_and_thread_staging_bit_identical_c2(vrs):
    """Config C2 at full size in bench.py's launch configuration: both staging
    engines produce byte-identical frames and identical counters."""
    scene, cams, fov, mk = _quest_workload(2, 500_000, 1.0, True, 32, True)
    a = _frame(vrs, scene, cams, fov, 32, mk, 0, max_pairs=6 << 20)
    b = _frame(vrs, scene, cams, fov, 32, mk, 1, max_pairs=6 << 20)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for k in ("pairs", "evaluations", "contributions", "overflow_samples", "terminated_samples"):
        assert a[2][k] == b[2][k], k


def test_staging_mode_rejects_unknown(vrs):
    r = vrs.Renderer(max_gaussians=10, max_views=1, max_pairs=1 << 10, max_width=32, max_height=32)
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_set_staging_mode(7)
    r.close()
