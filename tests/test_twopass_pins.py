"""Pins of the two-pass foveated baseline oracle (oracle/twopass.py; SURVEY
§8f N1, PAPER App. A).  CPU only.

Each pin checks the oracle against something other than itself: ray
equality from first principles (crop_frustum S:401-409), the sample
positions of the half-resolution pass, brute-force 2x2 OR, exactness of
bilinear interpolation on linear data, the ramp's closed form at known
points, coverage of the positive-weight region, and the SPEC example "centre
covering the whole image equals the full render".
"""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg
from helpers import identity_camera

from oracle import twopass as tpo


def _ray(cam, px, py):
    """World-independent camera-frame ray of continuous pixel position (px, py)."""
    return ((px - np.float64(cam.cx)) / np.float64(cam.fx), (py - np.float64(cam.cy)) / np.float64(cam.fy))


def test_crop_camera_casts_parent_rays():
    """crop pixel (a, b) casts the parent's ray of pixel (i0 + a, j0 + b)."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        W, H = int(rng.integers(16, 400)), int(rng.integers(16, 400))
        cam = identity_camera(W, H, float(rng.uniform(20, 500)))  # principal point W/2, H/2
        i0, j0 = int(rng.integers(0, W - 1)), int(rng.integers(0, H - 1))
        i1, j1 = int(rng.integers(i0 + 1, W + 1)), int(rng.integers(j0 + 1, H + 1))
        c1 = tpo.crop_camera(cam, (i0, j0, i1, j1))
        assert (c1.width, c1.height) == (i1 - i0, j1 - j0)
        a = rng.integers(0, c1.width, 100)
        b = rng.integers(0, c1.height, 100)
        rc = _ray(c1, a + 0.5, b + 0.5)
        rp = _ray(cam, i0 + a + 0.5, j0 + b + 0.5)
        assert np.array_equal(rc[0], rp[0]) and np.array_equal(rc[1], rp[1])
    full = tpo.crop_camera(identity_camera(64, 48, 40), (0, 0, 64, 48))  # rect = image -> same camera
    assert (full.cx, full.cy, full.width, full.height) == (32.0, 24.0, 64, 48)


def test_half_camera_samples_group_centres():
    """Pass 2 pixel (a, b) looks along the parent's ray through (2a + 1, 2b + 1)."""
    for W, H in ((64, 48), (65, 47), (2064, 2208)):
        cam = identity_camera(W, H, float(np.float32(722.64)))  # an f32 focal, as the ABI carries it
        c2 = tpo.half_camera(cam)
        assert (c2.width, c2.height) == ((W + 1) // 2, (H + 1) // 2)
        a, b = np.arange(c2.width), np.arange(c2.height)
        np.testing.assert_allclose(_ray(c2, a + 0.5, 0)[0], _ray(cam, 2 * a + 1.0, 0)[0], rtol=0, atol=1e-12)
        np.testing.assert_allclose(_ray(c2, 0, b + 0.5)[1], _ray(cam, 0, 2 * b + 1.0)[1], rtol=0, atol=1e-12)


def test_half_mask_is_2x2_or():
    rng = np.random.default_rng(1)
    for H, W in ((7, 9), (8, 8), (1, 5), (33, 2)):
        m = (rng.random((H, W)) < 0.2).astype(np.uint8)
        h = tpo.half_mask(m)
        ref = np.zeros(((H + 1) // 2, (W + 1) // 2), np.uint8)
        for j in range(H):
            for i in range(W):
                if m[j, i]:
                    ref[j // 2, i // 2] = 1
        assert np.array_equal(h, ref)


def test_bilinear_upsample_exact_on_linear_data():
    """A pass-2 image sampled from a linear function at the pass-2 sample
    positions (2a+1, 2b+1) upsamples to that function at every full-res pixel
    centre away from the clamped border; constants stay constant everywhere."""
    W, H = 37, 22
    W2, H2 = (W + 1) // 2, (H + 1) // 2
    xs, ys = 2 * np.arange(W2) + 1.0, 2 * np.arange(H2) + 1.0
    f = lambda x, y: 0.25 * x - 1.5 * y + 3.0
    img2 = f(xs[None, :], ys[:, None])
    up = tpo.bilinear_up(img2, W, H)
    px, py = np.arange(W) + 0.5, np.arange(H) + 0.5
    ref = f(px[None, :], py[:, None])
    inner = (slice(1, H - 2), slice(1, W - 2))
    np.testing.assert_allclose(up[inner], ref[inner], rtol=0, atol=1e-12)
    assert up[0, 0] == img2[0, 0]  # clamped corner
    c = tpo.bilinear_up(np.full((H2, W2, 4), 0.3), W, H)
    np.testing.assert_allclose(c, 0.3, rtol=0, atol=1e-15)


def test_fovea_weight_closed_form():
    """1 inside the full-rate rectangle, 0 beyond ramp * extent, linear in between."""
    fov = sg.Fovea((100.0, 80.0), (40.0, 20.0), 0.1)  # ramp widths 8 px (x), 4 px (y)
    w = lambda x, y: float(tpo.fovea_weight(fov, np.float64(x), np.float64(y)))
    assert w(100, 80) == 1.0 and w(139.9, 99.9) == 1.0
    assert w(144, 80) == pytest.approx(0.5) and w(100, 102) == pytest.approx(0.5)
    assert w(148.01, 80) == 0.0 and w(100, 104.01) == 0.0
    assert w(144, 102) == pytest.approx(0.5)  # separable max, not product


def test_pass1_rect_covers_every_positive_weight():
    rng = np.random.default_rng(2)
    for _ in range(30):
        W, H = int(rng.integers(8, 300)), int(rng.integers(8, 300))
        fov = sg.Fovea((float(rng.uniform(-20, W + 20)), float(rng.uniform(-20, H + 20))),
                       (float(rng.uniform(1, W)), float(rng.uniform(1, H))), float(rng.choice([0.0, 0.1, 0.25])))
        cam = identity_camera(W, H, 100.0)
        i0, j0, i1, j1 = tpo.pass1_rect(cam, fov)
        assert 0 <= i0 < i1 <= W and 0 <= j0 < j1 <= H
        py, px = np.mgrid[0:H, 0:W]
        pos = tpo.fovea_weight(fov, px + 0.5, py + 0.5) > 0
        inside = (px >= i0) & (px < i1) & (py >= j0) & (py < j1)
        assert not (pos & ~inside).any()


def test_two_pass_full_coverage_equals_full_render(oracle_mod):
    """a centre covering the whole image gives the full-resolution
    render (pass 2 has weight 0 everywhere)."""
    scene = sg.vr_room(11, 3000, sh_degree=1)
    W, H = 96, 64
    cam = sg.look_camera((0.0, 0.0, 0.0), f=60.0, width=W, height=H)
    fov = sg.Fovea((W / 2, H / 2), (W, H), 0.0)
    out, _ = tpo.render_two_pass(oracle_mod, scene, [cam], [fov], assign_tile=16)
    ref = oracle_mod.Oracle(scene).prepare([cam], assign_tile=16).render()[0]
    assert np.array_equal(out[0][0], ref[0].astype(np.float64))
    assert np.array_equal(out[0][1], ref[1].astype(np.float64))


def test_two_pass_quality_close_to_single_pass(oracle_mod):
    """SPEC S:398 (derived): against the full-resolution render, the two-pass
    baseline's PSNR is within 1 dB of (or above) the single-pass method's,
    while it preprocesses strictly more (view, Gaussian) pairs."""
    # a 256x192 window at the C2 focal length (722.64 px), so splats have their
    # C2 pixel sizes: at sub-pixel sizes pass 2's 0.3 px^2 dilation at half
    # resolution (a property of rendering at that resolution, L5) dominates
    scene = sg.vr_room(12, 100000, sh_degree=1)
    W, H = 256, 192
    cam = sg.look_camera((0.0, 0.0, 0.0), f=722.64, width=W, height=H)
    fov = sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)
    full = oracle_mod.Oracle(scene).prepare([cam], assign_tile=32).render()[0][0][..., :3].astype(np.float64)
    o1 = oracle_mod.Oracle(scene).prepare([cam], [fov], assign_tile=32)
    single = o1.render()[0][0][..., :3].astype(np.float64)
    two, o2 = tpo.render_two_pass(oracle_mod, scene, [cam], [fov], assign_tile=32)
    psnr = lambda a: 10 * np.log10(1.0 / max(np.mean((a - full) ** 2), 1e-20))
    assert psnr(two[0][0][..., :3]) >= psnr(single) - 1.0
    assert o2.stats()["visible_splats"] > o1.stats()["visible_splats"]
