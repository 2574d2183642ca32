"""GPU: the VRS_OUT_RGBA16F_D32F output format (RGBA IEEE binary16 + depth
float, 12 B per pixel, the half-float swap-chain format) is the F32 frame
rounded to binary16 bit for bit on every path, and stays within the
north_star tolerances (|dRGB| <= 2e-3, |dDepth| <= 1e-4 relative) against the
oracle on every pixel: rounding moves a value by at most 2^-11 |v| (half an
ulp), i.e. <= 2e-3 for |v| <= 4."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RGB_TOL = 2e-3
DEPTH_REL = 1e-4


@pytest.fixture(scope="module")
def vrs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    import paper_2505_10144_b200 as p
    return p


def _half_bits(a32):
    """binary32 -> binary16, round to nearest even (numpy's cast, the kernels' __floats2half2_rn)"""
    return a32.astype(np.float32).astype(np.float16).view(np.uint16)


def _stereo(W=320, H=256, n=20000):
    scene = sg.vr_room(7, n, sh_degree=3)
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
            for e, x in enumerate((-0.0315, 0.0315))]
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10)] * 2
    return scene, cams, fov


@pytest.mark.parametrize("mode", ["single", "two_pass", "hier", "host"])
def test_rgba16f_is_the_rounded_f32_frame(vrs, mode):
    scene, cams, fov = _stereo()
    W, H = cams[0].width, cams[0].height
    r = vrs.Renderer(max_gaussians=scene.n, max_views=4, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    for e in range(2):
        r.set_mask(e, sg.ellipse_mask(W, H))
    if mode == "hier":
        r.vrs_set_resort_mode(1)
    fn = r.render_two_pass if mode == "two_pass" else r.render

    def run():
        if mode == "host":
            a, d = r.vrs_render_views_host(cams, fov)
            return np.asarray(a).copy(), np.asarray(d).copy()
        a, d = fn(cams, fov)
        torch.cuda.synchronize()
        return a.cpu().numpy(), d.cpu().numpy()

    a32, d32 = run()
    r.vrs_set_output_format(2)
    a16, dd = run()
    assert a16.dtype == np.float16 and dd.dtype == np.float32 and a16.shape == a32.shape
    assert np.array_equal(a16.view(np.uint16), _half_bits(a32))
    assert np.array_equal(dd.view(np.uint32), d32.view(np.uint32))
    assert (np.abs(a16.astype(np.float64) - a32) <= 2.0 ** -11 * np.abs(a32) + 2.0 ** -25).all()


def test_rgba16f_within_tolerance_of_the_oracle(vrs, oracle_mod):
    """Every pixel of a foveated, masked stereo frame in the half-float
    format against the oracle's frame (no clamping: HDR values stay)."""
    scene, cams, fov = _stereo()
    W, H = cams[0].width, cams[0].height
    masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)}
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    o = oracle_mod.Oracle(scene)
    for s, m in masks.items():
        r.set_mask(s, m)
        o.set_mask(s, m)
    r.vrs_set_output_format(2)
    a16, dd = r.render(cams, fov)
    torch.cuda.synchronize()
    a = a16.cpu().numpy().astype(np.float64)
    d = dd.cpu().numpy().astype(np.float64)
    o.prepare(cams, fov, assign_tile=32)
    off = 0
    for (oimg, odep), c in zip(o.render(), cams):
        px = c.width * c.height
        g = a[off:off + px].reshape(c.height, c.width, 4)
        gd = d[off:off + px].reshape(c.height, c.width)
        off += px
        assert np.abs(g - oimg).max() <= RGB_TOL
        assert (np.abs(gd - odep) - DEPTH_REL * np.abs(odep)).max() <= 1e-6


def test_rgba16f_c2_full_size(vrs):
    """Config C2 at full size (bench.py's e2e headline format): the half-float
    frame is the F32 frame rounded to binary16 bit for bit, every RGBA value
    within 2^-11 |v| (<= 2e-3) of it (the F32 frame is checked against the
    oracle on every pixel by test_c2_full_size_parity)."""
    scene = sg.vr_room(2, 500_000, scale_mul=1.0, sh_degree=3)
    cams = sg.stereo_pair(masks=True)
    fov = [sg.quest_fovea()] * 2
    W, H = cams[0].width, cams[0].height
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=6 << 20, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    for e in range(2):
        r.set_mask(e, sg.ellipse_mask(W, H))
    a32, d32 = r.render(cams, fov)
    torch.cuda.synchronize()
    a32, d32 = a32.cpu().numpy(), d32.cpu().numpy()
    r.vrs_set_output_format(2)
    a16, dd = r.render(cams, fov)
    torch.cuda.synchronize()
    h = a16.cpu().numpy()
    assert np.array_equal(h.view(np.uint16), _half_bits(a32))
    assert np.array_equal(dd.cpu().numpy().view(np.uint32), d32.view(np.uint32))
    assert np.abs(h.astype(np.float64) - a32).max() <= RGB_TOL


def test_unknown_output_format_rejected(vrs):
    r = vrs.Renderer(max_gaussians=16, max_views=1, max_pairs=1 << 10, max_width=16, max_height=16,
                     assign_tile=16)
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_set_output_format(3)
    r.vrs_set_output_format(2)
    r.vrs_set_output_format(0)
