"""Full-size parity of the paths round 1 checked only at small sizes
(VERDICT r1 "weak #3"), in bench.py's launch configurations:

* N1 two-pass baseline on the full C6 frame (C2 scene, 2x2064x2208,
  foveated, masks): the 4-view pass frame's sorted pair list and ranges
  bit-exact, EVERY output pixel within the tolerances;
* Optimal Projection at 160 deg (C5's widest point) on the full frame:
  lists bit-exact, every pixel;
* N2 hierarchical mode (C8) on the full C2 frame: pair list and ranges
  bit-exact (the pixel comparison is test_gpu_hier's sampled C2 test);
* N4 backward on a 512x512 stereo frame against the fp64 autograd oracle
  (built block by block: oracle.grad.gradients_blocked)."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg
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


def test_two_pass_c6_full_size(vrs, oracle_mod):
    from oracle import twopass as tpo
    scene, cams, fov, mk = _quest_workload(2, 500_000, 1.0, True, 32, True)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=4, max_pairs=16 << 20, max_width=sg.QUEST_W,
                     max_height=sg.QUEST_H, assign_tile=32)
    r.upload(scene)
    for s_, m in mk.items():
        r.set_mask(s_, m)
    rgba, depth = r.render_two_pass(cams, fov)
    torch.cuda.synchronize()
    g = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), cams)
    out, o = tpo.render_two_pass(oracle_mod, scene, cams, fov, masks=mk, assign_tile=32)
    k, v = r.vrs_debug_pairs(True)
    ok, ov = o.pairs(True)
    assert len(k) > 1_000_000
    assert np.array_equal(k, ok) and np.array_equal(v, ov)
    assert np.array_equal(r.vrs_debug_ranges(), o.ranges())
    assert_images_close(g, [(c.astype(np.float32), d.astype(np.float32)) for c, d in out])


def test_op_160_full_size(vrs, oracle_mod):
    scene = sg.vr_room(2, 500_000, scale_mul=1.0, sh_degree=3)
    cams = sg.stereo_pair(hfov_deg=160.0, masks=False)
    fov = [sg.quest_fovea()] * 2
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, max_pairs=8 << 20, projection=0)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)


def test_hier_c8_full_size_lists(vrs, oracle_mod):
    scene, cams, fov, mk = _quest_workload(2, 500_000, 1.0, True, 32, True)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=8 << 20, max_width=sg.QUEST_W,
                     max_height=sg.QUEST_H, assign_tile=32)
    r.upload(scene)
    for s_, m in mk.items():
        r.set_mask(s_, m)
    r.vrs_set_resort_mode(1)
    r.render(cams, fov)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene)
    for s_, m in mk.items():
        o.set_mask(s_, m)
    o.prepare(cams, fov, assign_tile=32, resort=1, block_queue=8, group_queue=4)
    assert_lists_equal(r, o)


def test_backward_512_stereo(vrs, oracle_mod):
    from oracle import grad
    W = H = 512
    scene = sg.vr_room(9, 20000, scale_mul=1.0, sh_degree=3)
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H) for x in (-0.0315, 0.0315)]
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=16)
    r.upload(scene)
    rgba, depth = r.render(cams)
    rng = np.random.default_rng(7)
    gr = [rng.normal(size=(H, W, 4)) for _ in cams]
    gd = [rng.normal(size=(H, W)) * 0.1 for _ in cams]
    g_rgba = torch.tensor(np.concatenate([x.reshape(-1, 4) for x in gr]), dtype=torch.float32, device="cuda")
    g_depth = torch.tensor(np.concatenate([x.reshape(-1) for x in gd]), dtype=torch.float32, device="cuda")
    out = r.vrs_backward(rgba, depth, g_rgba, g_depth)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene).prepare(cams, assign_tile=16)
    orders = [o.blend_orders(v) for v in range(2)]
    assert sum(int(c.sum()) for c, _ in orders) > 1_000_000  # a real frame's worth of blends (1.49 M)
    ref = grad.gradients_blocked(scene, cams, orders, gr, gd, rows=32)
    for k in ("means", "quats", "log_scales", "logits", "sh"):
        a = out[k].cpu().numpy().astype(np.float64).reshape(ref[k].shape)
        scale = np.abs(ref[k]).max()
        assert np.abs(a - ref[k]).max() <= 2e-3 * scale + 1e-7, k
    r.close()


def test_backward_c9_full_frame_banded_loss(vrs, oracle_mod):
    """N4 in config C9's launch configuration: the C2 scene, non-foveated stereo
    2x2064x2208 (9.1 M pixels, T_a = 16), full-frame forward and backward on the
    GPU; the loss weights three 32-row bands per eye (zero elsewhere), so the fp64
    oracle only back-propagates those rows -- the GPU still runs every pixel."""
    from oracle import grad
    scene = sg.vr_room(2, 500_000, scale_mul=1.0, sh_degree=3)
    cams = sg.stereo_pair(masks=False)
    W, H = cams[0].width, cams[0].height
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=16 << 20, max_width=W, max_height=H,
                     assign_tile=16)
    r.upload(scene)
    rgba, depth = r.render(cams)
    rng = np.random.default_rng(9)
    gr, gd = [], []
    for e in range(2):
        a = np.zeros((H, W, 4))
        b = np.zeros((H, W))
        for y0 in (96 + 32 * e, 1088, 2016 - 32 * e):
            a[y0:y0 + 32] = rng.normal(size=(32, W, 4))
            b[y0:y0 + 32] = rng.normal(size=(32, W)) * 0.1
        gr.append(a)
        gd.append(b)
    g_rgba = torch.tensor(np.concatenate([x.reshape(-1, 4) for x in gr]), dtype=torch.float32, device="cuda")
    g_depth = torch.tensor(np.concatenate([x.reshape(-1) for x in gd]), dtype=torch.float32, device="cuda")
    out = r.vrs_backward(rgba, depth, g_rgba, g_depth)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene).prepare(cams, assign_tile=16)
    orders = [o.blend_orders(v) for v in range(2)]
    ref = grad.gradients_blocked(scene, cams, orders, gr, gd, rows=32)
    for k in ("means", "quats", "log_scales", "logits", "sh"):
        a = out[k].cpu().numpy().astype(np.float64).reshape(ref[k].shape)
        scale = np.abs(ref[k]).max()
        assert scale > 0
        assert np.abs(a - ref[k]).max() <= 2e-3 * scale + 1e-7, k
    r.close()
