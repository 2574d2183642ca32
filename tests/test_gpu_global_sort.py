"""GPU parity of the N3 global-sort baselines (vrs_set_sort_mode; SURVEY §8f
N3): Mini-Splatting (z) and (Dist) -- one key depth per
Gaussian, tile lists blended in list order with no per-sample window --
against the oracle's sort_mode 1 / 2 (pinned in test_oracle_pins_r2.py by the
tile-free render in the global order and the popping invariants).  Bars as for
the method: pair lists, ranges and counters bit-exact, RGB 2e-3, depth 1e-4."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg
from helpers import identity_camera
from test_gpu_parity import _quest_workload, assert_images_close, assert_lists_equal

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


def render_mode(vrs, oracle_mod, scene, cams, foveas, T, mode, masks=None, projection=0, max_pairs=1 << 22,
                oracle_pixels=None):
    W, H = max(c.width for c in cams), max(c.height for c in cams)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=len(cams), max_pairs=max_pairs, max_width=W, max_height=H,
                     assign_tile=T, projection=projection)
    r.upload(scene)
    o = oracle_mod.Oracle(scene)
    for slot, m in (masks or {}).items():
        r.set_mask(slot, m)
        o.set_mask(slot, m)
    r.vrs_set_instrumentation(counters=1)
    r.vrs_set_sort_mode(mode)
    rgba, depth = r.render(cams, foveas)
    torch.cuda.synchronize()
    g = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), cams)
    o.prepare(cams, foveas, assign_tile=T, projection=projection, sort_mode=mode)
    return r, o, g


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("projection", [0, 1])
def test_global_sort_c1_seeds(vrs, oracle_mod, mode, projection):
    for seed in range(4):
        scene = sg.random_scene(seed, n=1000)
        r, o, g = render_mode(vrs, oracle_mod, scene, [identity_camera(128, 128, 64.0)], None, 16, mode,
                              projection=projection)
        assert_lists_equal(r, o)
        assert_images_close(g, o.render())
        st, ost = r.stats(), o.stats()
        for k in ("evaluations", "contributions", "overflow_samples", "terminated_samples"):
            assert st[k] == ost[k], k
        assert st["overflow_samples"] == 0


@pytest.mark.parametrize("mode", [1, 2])
def test_global_sort_foveated_masked_stereo(vrs, oracle_mod, mode):
    scene = sg.vr_room(7, 20000, sh_degree=3)
    W, H = 320, 256
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
            for e, x in enumerate((-0.0315, 0.0315))]
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10)] * 2
    masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)}
    r, o, g = render_mode(vrs, oracle_mod, scene, cams, fov, 32, mode, masks=masks)
    assert_lists_equal(r, o)
    assert_images_close(g, o.render())


@pytest.mark.parametrize("mode", [1, 2])
def test_global_sort_c2_full_size(vrs, oracle_mod, mode):
    """C2 at full size: pair lists bit-exact, EVERY pixel of both eyes within tolerance."""
    scene, cams, fov, mk = _quest_workload(2, 500_000, 1.0, True, 32, True)
    r, o, g = render_mode(vrs, oracle_mod, scene, cams, fov, 32, mode, masks=mk, max_pairs=6 << 20)
    assert_lists_equal(r, o)
    assert_images_close(g, o.render())


def test_global_sort_differs_from_stopthepop(vrs):
    """The baselines are a different method: on a scene with overlapping
    Gaussians the frames differ from the StopThePop frame (and from each other)."""
    scene = sg.vr_room(7, 20000, sh_degree=0)
    cam = sg.look_camera((0, 0, 0), 0.4, 0.0, 0.0, f=200.0, width=256, height=256)
    outs = []
    for mode in (0, 1, 2):
        r = vrs.Renderer(max_gaussians=scene.n, max_views=1, max_pairs=1 << 22, max_width=256, max_height=256)
        r.upload(scene)
        r.vrs_set_sort_mode(mode)
        rgba, _ = r.render([cam])
        outs.append(rgba.cpu().numpy())
        r.close()
    assert np.abs(outs[0] - outs[1]).max() > 1e-3 and np.abs(outs[0] - outs[2]).max() > 1e-3
    assert np.abs(outs[1] - outs[2]).max() > 1e-3


def test_global_sort_mode_validation(vrs):
    r = vrs.Renderer(max_gaussians=10, max_views=1, max_pairs=1 << 10, max_width=32, max_height=32)
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_set_sort_mode(3)
    r.vrs_set_resort_mode(1)
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_set_sort_mode(1)  # no per-sample resort in a global sort
    r.vrs_set_resort_mode(0)
    r.vrs_set_sort_mode(2)
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_set_resort_mode(1)
    r.close()
