"""GPU parity of the N4 backward (vrs_backward) against the PyTorch fp64
gradient oracle (oracle/grad.py over the C++ oracle's blend orders, pinned
by tests/test_grad_pins.py).  Gradients are tolerance quantities: per
parameter group, max |g_gpu - g_ref| <= 2e-3 * max |g_ref| (fp32 atomics and
fp32 chain rule against fp64 autograd)."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
grad = pytest.importorskip("oracle.grad")

REL = 2e-3


@pytest.fixture(scope="module")
def vrs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    import paper_2505_10144_b200 as p
    return p


def _check(vrs, oracle_mod, scene, cams, T=16, seed=0):
    W, H = max(c.width for c in cams), max(c.height for c in cams)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=len(cams), max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=T)
    r.upload(scene)
    rgba, depth = r.render(cams)
    rng = np.random.default_rng(seed)
    gr = [rng.normal(size=(c.height, c.width, 4)) for c in cams]
    gd = [rng.normal(size=(c.height, c.width)) * 0.1 for c in cams]
    g_rgba = torch.tensor(np.concatenate([x.reshape(-1, 4) for x in gr]), dtype=torch.float32, device="cuda")
    g_depth = torch.tensor(np.concatenate([x.reshape(-1) for x in gd]), dtype=torch.float32, device="cuda")
    out = r.vrs_backward(rgba, depth, g_rgba, g_depth)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene).prepare(cams, assign_tile=T)
    orders = [o.blend_orders(v) for v in range(len(cams))]
    ref, _ = grad.gradients(scene, cams, orders, gr, gd)
    for k in ("means", "quats", "log_scales", "logits", "sh"):
        a = out[k].cpu().numpy().astype(np.float64).reshape(ref[k].shape)
        scale = np.abs(ref[k]).max()
        err = np.abs(a - ref[k]).max()
        assert err <= REL * scale + 1e-7, (k, err, scale)
    r.close()


@pytest.mark.parametrize("seed,deg", [(0, 0), (1, 1), (2, 3)])
def test_backward_c1_like(vrs, oracle_mod, seed, deg):
    scene = sg.random_scene(seed, n=300, sh_degree=deg)
    cams = [sg.look_camera((0, 0, 0), f=40.0, width=64, height=48)]
    _check(vrs, oracle_mod, scene, cams, seed=seed)


def test_backward_stereo_vr_room_t32(vrs, oracle_mod):
    """Two views sharing Gaussians (gradients summed over views), 32x32 assignment tiles."""
    W, H = 96, 80
    scene = sg.vr_room(9, 3000, scale_mul=1.0, sh_degree=2)
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H) for x in (-0.0315, 0.0315)]
    _check(vrs, oracle_mod, scene, cams, T=32, seed=3)


def test_backward_rejects_foveated_frames(vrs):
    W, H = 64, 64
    scene = sg.vr_room(9, 500, sh_degree=0)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=1, max_pairs=1 << 20, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    cam = sg.look_camera((0, 0, 0), f=40.0, width=W, height=H)
    rgba, depth = r.render([cam], [sg.Fovea((32, 32), (16, 16), 0.1)])
    z = torch.zeros_like(rgba), torch.zeros_like(depth)
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_backward(rgba, depth, *z)


@pytest.mark.parametrize("which", ["rgb_only", "alpha_only", "depth_only"])
def test_backward_single_output_losses(vrs, oracle_mod, which):
    """Each output channel group on its own (the colour, transmittance and
    depth chains are separate code paths of k_blend_bwd)."""
    scene = sg.random_scene(7, n=300, sh_degree=1)
    cam = sg.look_camera((0, 0, 0), f=40.0, width=64, height=48)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=1, max_pairs=1 << 20, max_width=64, max_height=48,
                     assign_tile=16)
    r.upload(scene)
    rgba, depth = r.render([cam])
    rng = np.random.default_rng(11)
    gr = rng.normal(size=(48, 64, 4))
    gd = rng.normal(size=(48, 64)) * 0.1
    if which == "rgb_only":
        gr[..., 3] = 0.0
        gd[:] = 0.0
    elif which == "alpha_only":
        gr[..., :3] = 0.0
        gd[:] = 0.0
    else:
        gr[:] = 0.0
    out = r.vrs_backward(rgba, depth, torch.tensor(gr.reshape(-1, 4), dtype=torch.float32, device="cuda"),
                         torch.tensor(gd.reshape(-1), dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene).prepare([cam], assign_tile=16)
    ref, _ = grad.gradients(scene, [cam], [o.blend_orders(0)], [gr], [gd])
    for k in ("means", "quats", "log_scales", "logits", "sh"):
        a = out[k].cpu().numpy().astype(np.float64).reshape(ref[k].shape)
        scale = np.abs(ref[k]).max()
        assert np.abs(a - ref[k]).max() <= REL * scale + 1e-7, (which, k)


def test_backward_rejects_other_modes(vrs):
    W, H = 64, 64
    scene = sg.vr_room(9, 500, sh_degree=0)
    cam = sg.look_camera((0, 0, 0), f=40.0, width=W, height=H)
    for setup in ("ewa", "hier", "packed"):
        r = vrs.Renderer(max_gaussians=scene.n, max_views=1, max_pairs=1 << 20, max_width=W, max_height=H,
                         assign_tile=16, projection=1 if setup == "ewa" else 0)
        r.upload(scene)
        if setup == "hier":
            r.vrs_set_resort_mode(1)
        if setup == "packed":
            r.vrs_set_output_format(1)
        rgba, depth = r.render([cam])
        f32 = (torch.zeros((W * H, 4), device="cuda"), torch.zeros(W * H, device="cuda"))
        with pytest.raises(vrs.vrs.VrsError):
            r.vrs_backward(*f32, *f32)
        r.close()
    # the two-pass baseline's frame state is its internal 2n-view frame
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 20, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    r.render_two_pass([cam], [sg.Fovea((32, 32), (16, 16), 0.1)])
    f32 = (torch.zeros((W * H, 4), device="cuda"), torch.zeros(W * H, device="cuda"))
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_backward(*f32, *f32)
    # a new upload invalidates the last frame (its records refer to the old scene)
    r2 = vrs.Renderer(max_gaussians=scene.n, max_views=1, max_pairs=1 << 20, max_width=W, max_height=H,
                      assign_tile=16)
    r2.upload(scene)
    rgba, depth = r2.render([cam])
    r2.upload(sg.vr_room(10, 300, sh_degree=0))
    with pytest.raises(vrs.vrs.VrsError):
        r2.vrs_backward(rgba, depth, *f32)
    r.close()
    r2.close()
