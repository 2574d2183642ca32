"""GPU parity of the N2 hierarchical resort mode (vrs_set_resort_mode(1):
K_B = 8 block queue per 4x4 sample block, K_G = 4 queue per 2x2 group,
K_P = 8 per-sample window) against
the oracle's resort=1 mode (pinned by tests/test_hier_pins.py).  Bars as in
test_gpu_parity.py: pair lists bit-exact (unchanged by the mode), RGB/A
within 2e-3, depth within 1e-4 relative, workload counters equal (they count
exact decisions: memberships, releases, window overflows, T < 1e-4 stops)."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RGB_TOL = 2e-3
DEPTH_REL = 1e-4
KB = KP = 8
KG = 4
COUNTERS = ("pairs", "samples", "evaluations", "contributions", "overflow_samples", "terminated_samples")


@pytest.fixture(scope="module")
def vrs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    import paper_2505_10144_b200 as p
    return p


def _render(vrs, oracle_mod, scene, cams, fov=None, T=16, masks=None, max_pairs=1 << 22, oracle_full=True,
            no_cull=False):
    W, H = max(c.width for c in cams), max(c.height for c in cams)
    r = vrs.Renderer(max_gaussians=max(scene.n, 1), max_views=len(cams), max_pairs=max_pairs, max_width=W,
                     max_height=H, assign_tile=T)
    r.upload(scene)
    r.vrs_set_resort_mode(1, KB, KP)
    o = oracle_mod.Oracle(scene)
    for slot, m in (masks or {}).items():
        r.set_mask(slot, m)
        o.set_mask(slot, m)
    r.vrs_set_instrumentation(counters=1, no_cull=no_cull)
    rgba, depth = r.render(cams, fov)
    torch.cuda.synchronize()
    g = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), cams)
    o.prepare(cams, fov, assign_tile=T, window_k=KP, resort=1, block_queue=KB, group_queue=KG)
    oi = o.render() if oracle_full else None
    return r, o, g, oi


def _close(g, oi):
    for (gi, gd), (oo, od) in zip(g, oi):
        d = np.abs(gi - oo)
        assert d.max() <= RGB_TOL, f"max |dRGBA| {d.max()} at {np.unravel_index(d.argmax(), d.shape)}"
        dd = np.abs(gd - od) - DEPTH_REL * np.abs(od)
        assert dd.max() <= 1e-6, f"depth excess {dd.max()} at {np.unravel_index(dd.argmax(), dd.shape)}"


def _counters(r, o):
    st, ost = r.stats(), o.stats()
    for k in COUNTERS:
        assert st[k] == ost[k], (k, st[k], ost[k])


@pytest.mark.parametrize("seed", [0, 1, 2, 5])
def test_hier_c1_parity(vrs, oracle_mod, seed):
    scene = sg.random_scene(seed, n=1000, sh_degree=0)
    cam = sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)
    r, o, g, oi = _render(vrs, oracle_mod, scene, [cam])
    _close(g, oi)
    _counters(r, o)


def _stereo(W, H, masks=False):
    f = sg.focal_for_hfov(W, 110.0)
    return [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e if masks else -1)
            for e, x in enumerate((-0.0315, 0.0315))]


def test_hier_foveated_masked_stereo_parity(vrs, oracle_mod):
    """HighRes, Hybrid and LowRes (4x4 groups = 8x8 px blocks) items, masks, stereo."""
    W, H = 320, 256
    scene = sg.vr_room(7, 20000, sh_degree=3)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10)] * 2
    masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)}
    r, o, g, oi = _render(vrs, oracle_mod, scene, _stereo(W, H, True), fov, T=32, masks=masks)
    _close(g, oi)
    _counters(r, o)


@pytest.mark.parametrize("W,H,T", [(131, 97, 16), (203, 150, 32), (66, 34, 32)])
def test_hier_odd_sizes_and_edges(vrs, oracle_mod, W, H, T):
    """Image borders cut 4x4 blocks: out-of-image samples take no part."""
    scene = sg.vr_room(11, 8000, sh_degree=1)
    fov = [sg.Fovea((W / 2, H / 2), (W / 5 + 1, H / 5 + 1), 0.2)] * 2 if T == 32 else None
    r, o, g, oi = _render(vrs, oracle_mod, scene, _stereo(W, H), fov, T=T)
    _close(g, oi)
    _counters(r, o)


def test_hier_dense_overflow_parity(vrs, oracle_mod):
    """Deep per-ray overlap: queues and windows overflow constantly."""
    W, H = 192, 160
    scene = sg.vr_room(13, 60000, scale_mul=1.6, sh_degree=0)
    r, o, g, oi = _render(vrs, oracle_mod, scene, _stereo(W, H), None, T=16)
    _close(g, oi)
    _counters(r, o)
    assert r.stats()["overflow_samples"] > 1000


def test_hier_warp_culling_never_changes_results(vrs, oracle_mod):
    W, H = 256, 192
    scene = sg.vr_room(17, 20000, sh_degree=2)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    outs = []
    for nc in (False, True):
        r, _, g, _ = _render(vrs, oracle_mod, scene, _stereo(W, H), fov, T=32, oracle_full=False, no_cull=nc)
        outs.append(g)
    for (a, da), (b, db) in zip(*outs):
        assert np.array_equal(a, b) and np.array_equal(da, db)


def test_hier_c2_full_size_parity(vrs, oracle_mod):
    """Config C2 at full size in the hierarchical mode: EVERY output pixel of
    both eyes within tolerance, workload counters equal."""
    scene = sg.vr_room(2, 500_000, scale_mul=1.0, sh_degree=3)
    cams = sg.stereo_pair(masks=True)
    fov = [sg.quest_fovea()] * 2
    mk = {0: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H), 1: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H)}
    r, o, g, oi = _render(vrs, oracle_mod, scene, cams, fov, T=32, masks=mk, max_pairs=6 << 20)
    _close(g, oi)
    st, ost = r.stats(), o.stats()
    for k in ("pairs", "samples", "contributions", "terminated_samples"):
        assert st[k] == ost[k], (k, st[k], ost[k])


def test_hier_mode_arguments(vrs):
    r = vrs.Renderer(max_gaussians=16, max_views=1, max_pairs=1024, max_width=64, max_height=64, assign_tile=16)
    for bad in ((2, 0, 0), (1, 4, 8), (1, 8, 16), (0, 0, 8)):
        with pytest.raises(vrs.vrs.VrsError):
            r.vrs_set_resort_mode(*bad)
    r.vrs_set_resort_mode(1, 0, 0)
    r.vrs_set_resort_mode(0, 0, 16)
    e = vrs.Renderer(max_gaussians=16, max_views=1, max_pairs=1024, max_width=64, max_height=64, assign_tile=16,
                     projection=1)
    with pytest.raises(vrs.vrs.VrsError):
        e.vrs_set_resort_mode(1)
