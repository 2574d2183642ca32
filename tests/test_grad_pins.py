"""Pins of the N4 gradient oracle (oracle/grad.py, plain PyTorch fp64):

G1  its forward equals the pinned C++ oracle's render (fp64 vs the binary32
    contract: |dRGBA| <= 2e-5, |dDepth| <= 1e-4 relative) on the blend orders
    the C++ oracle decided;
G2  its gradient equals central finite differences of that forward (fixed
    orders), per parameter group, along random directions;
G3  closed forms for one isotropic Gaussian on the optical axis:
    RGB = alpha (0.5 + C0 dc), A = alpha, alpha = sigma exp(-q/2),
    q = |D|^2 / (f^2 s^2 / z^2 + 0.3) -> dR/d dc = alpha C0,
    dA/d logit = sigma (1 - sigma) exp(-q/2), dA/d log s = alpha q (1 - 0.3/(f^2 s^2/z^2 + 0.3)).
CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import scenegen as sg
from helpers import C0, identity_camera, scene_from

grad = pytest.importorskip("oracle.grad")


def _setup(oracle_mod, seed, n=300, deg=2, W=64, H=48, f=40.0, stereo=False):
    sc = sg.random_scene(seed, n=n, sh_degree=deg)
    if stereo:
        cams = [sg.look_camera((x, 0, 0), 0.05, -0.03, 0.0, f=f, width=W, height=H) for x in (-0.03, 0.03)]
    else:
        cams = [sg.look_camera((0, 0, 0), f=f, width=W, height=H)]
    o = oracle_mod.Oracle(sc).prepare(cams, assign_tile=16)
    return sc, cams, o


@pytest.mark.parametrize("seed,deg,stereo", [(0, 0, False), (1, 1, False), (2, 2, True), (3, 3, False)])
def test_g1_forward_matches_cpp_oracle(oracle_mod, seed, deg, stereo):
    sc, cams, o = _setup(oracle_mod, seed, deg=deg, stereo=stereo)
    ref = o.render()
    orders = [o.blend_orders(v) for v in range(len(cams))]
    outs = grad.render_fixed_order(grad.to_params(sc, False), cams, orders, sc.sh_degree)
    for (a, d), (ti, td) in zip(ref, outs):
        assert np.abs(ti.numpy() - a).max() <= 2e-5
        assert (np.abs(td.numpy() - d) - 1e-4 * np.abs(d)).max() <= 1e-6


@pytest.mark.parametrize("seed", [4, 5])
def test_g2_autograd_is_the_derivative(oracle_mod, seed):
    sc, cams, o = _setup(oracle_mod, seed, n=120, deg=2, W=48, H=40, stereo=True)
    orders = [o.blend_orders(v) for v in range(len(cams))]
    rng = np.random.default_rng(seed)
    gr = [rng.normal(size=(c.height, c.width, 4)) for c in cams]
    gd = [rng.normal(size=(c.height, c.width)) * 0.1 for c in cams]
    g, _ = grad.gradients(sc, cams, orders, gr, gd)

    def loss(p):
        outs = grad.render_fixed_order(p, cams, orders, sc.sh_degree)
        return sum(float((a * torch.as_tensor(x)).sum() + (d * torch.as_tensor(y)).sum())
                   for (a, d), x, y in zip(outs, gr, gd))

    base = grad.to_params(sc, False)
    for k in ("means", "quats", "log_scales", "logits", "sh"):
        dirn = rng.normal(size=base[k].shape)
        h = 1e-6
        pp = {kk: v.clone() for kk, v in base.items()}
        pm = {kk: v.clone() for kk, v in base.items()}
        pp[k] = pp[k] + h * torch.as_tensor(dirn)
        pm[k] = pm[k] - h * torch.as_tensor(dirn)
        fd = (loss(pp) - loss(pm)) / (2 * h)
        an = float((g[k] * dirn).sum())
        assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)), (k, fd, an)


def test_g3_on_axis_closed_forms(oracle_mod):
    z, s, sigma, dc, f = 4.0, 0.15, 0.5, 0.7, 50.0
    sc = scene_from([[0, 0, z]], s, opacities=sigma, dc=[dc, dc, dc])
    W = H = 32
    cam = identity_camera(W, H, f)
    o = oracle_mod.Oracle(sc).prepare([cam], assign_tile=16)
    orders = [o.blend_orders(0)]
    i, j = 19, 14  # pixel centre offset D = (3.5, -1.5) px from (16, 16)
    D2 = (i + 0.5 - 16) ** 2 + (j + 0.5 - 16) ** 2
    den = f * f * s * s / (z * z) + 0.3
    q = D2 / den
    a = sigma * math.exp(-q / 2)
    gr = np.zeros((H, W, 4))
    gr[j, i, 0] = 1.0
    g, outs = grad.gradients(sc, [cam], orders, [gr], [np.zeros((H, W))])
    # (scene parameters are stored in float32: agreement to ~1e-7 relative)
    assert abs(outs[0][0][j, i, 0] - a * (0.5 + C0 * dc)) < 1e-6 * a
    assert abs(g["sh"][0, 0, 0] - a * C0) < 1e-6 * a
    gr[j, i, 0] = 0.0
    gr[j, i, 3] = 1.0
    g, _ = grad.gradients(sc, [cam], orders, [gr], [np.zeros((H, W))])
    assert abs(g["logits"][0] - sigma * (1 - sigma) * math.exp(-q / 2)) < 1e-6 * a
    # dA/d log s_k summed over the three axes (isotropic): da/dq * dq/d(log s) with s^2 in den
    dq_dlogs = -q * (2 * f * f * s * s / (z * z)) / den
    assert abs(g["log_scales"][0].sum() - (-a / 2) * dq_dlogs) < 1e-6 * a


def test_blocked_gradients_equal_whole_frame(oracle_mod):
    """gradients_blocked (row blocks, for large frames) = gradients (one graph)."""
    import scenegen as sg
    from oracle import grad
    scene = sg.random_scene(3, n=120, sh_degree=1)
    cam = sg.look_camera((0, 0, 0), f=40.0, width=48, height=40)
    o = oracle_mod.Oracle(scene).prepare([cam], assign_tile=16)
    orders = [o.blend_orders(0)]
    rng = np.random.default_rng(2)
    gr = [rng.normal(size=(40, 48, 4))]
    gd = [rng.normal(size=(40, 48)) * 0.1]
    ref, _ = grad.gradients(scene, [cam], orders, gr, gd)
    got = grad.gradients_blocked(scene, [cam], orders, gr, gd, rows=7)
    for k in ref:
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-9, atol=1e-12)
