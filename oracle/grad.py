"""N4 ORACLE (test infrastructure only, not product code): gradients of the
training-mode render (non-foveated, full-rate, K = 16 window, Optimal
Projection) with respect to the raw 3DGS parameters, in plain PyTorch fp64 on
the CPU ("the method's training side ... gradient-checked
against finite differences on synthetic scenes"; the paper fine-tunes
StopThePop + Optimal Projection models).

The forward re-states the C++ oracle's math (oracle.cpp) in
fp64 torch ops: activation (L1: exp / sigmoid / normalised quaternion,
Sigma = R S S^T R^T, Eq.1), Optimal Projection (O2-O5: tangent basis,
Sigma_2 = E^T Sigma_c E / r^2 + pixel-mapped 0.3 px^2 dilation, C = Sigma_2^-1),
per-sample q = [e1.d, e2.d] C [e1.d, e2.d]^T / (u.d)^2, alpha = min(0.99,
sigma exp(-q/2)), tau = max(d^T b / d^T A d, near) (O10, R4), the
SH colour + 0.5 clamped at 0 (O5), and front-to-back compositing (Eq.2 with
product transmittance, L2; depth L13) -- over the blend order the C++ oracle
decided (``Oracle.blend_orders``).  The order and the set of blended
Gaussians are held fixed (they are piecewise constant in the parameters), so
the render is a smooth function there and autograd gives its gradient.  The
clamps (alpha <= 0.99, tau >= near, colour >= 0) contribute zero derivative
where they bind.

Loss convention (the backward contract): L = sum over pixels of
g_rgba . RGBA + g_depth * Depth, i.e. the incoming gradient images.
"""
from __future__ import annotations

import numpy as np
import torch

C0 = 0.28209479177387814
C1 = 0.4886025119029199
C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
      1.445305721320277, -0.5900435899266435)


def sh_basis(d, deg):
    """Real SH basis of the 3DGS convention ([ext] constants) at unit dirs d (n, 3)."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    out = [torch.full_like(x, C0)]
    if deg > 0:
        out += [-C1 * y, C1 * z, -C1 * x]
    if deg > 1:
        xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
        out += [C2[0] * xy, C2[1] * yz, C2[2] * (2 * zz - xx - yy), C2[3] * xz, C2[4] * (xx - yy)]
        if deg > 2:
            out += [C3[0] * y * (3 * xx - yy), C3[1] * xy * z, C3[2] * y * (4 * zz - xx - yy),
                    C3[3] * z * (2 * zz - 3 * xx - 3 * yy), C3[4] * x * (4 * zz - xx - yy), C3[5] * z * (xx - yy),
                    C3[6] * x * (xx - 3 * yy)]
    return torch.stack(out, 1)  # (n, k)


def activate(means, quats, log_scales, logits):
    """L1: normalised quaternion -> R, Sigma = R S^2 R^T, Sigma^-1 = R S^-2 R^T, sigma = sigmoid."""
    q = quats / quats.norm(dim=1, keepdim=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = torch.stack([torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1),
                     torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1),
                     torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)], 1)
    s2 = torch.exp(2.0 * log_scales)
    cov = R @ torch.diag_embed(s2) @ R.transpose(1, 2)
    icov = R @ torch.diag_embed(1.0 / s2) @ R.transpose(1, 2)
    return means, cov, icov, torch.sigmoid(logits)


def render_fixed_order(params, cams, orders, sh_degree, near=0.2, background=(0.0, 0.0, 0.0)):
    """fp64 render of non-foveated views over fixed per-pixel blend orders.
    params: dict of fp64 tensors means (n,3), quats (n,4), log_scales (n,3),
    logits (n,), sh (n,k,3); orders[v] = (counts (H,W), seq).  Returns a list
    of (rgba (H,W,4), depth (H,W))."""
    mu, cov, icov, sig = activate(params["means"], params["quats"], params["log_scales"], params["logits"])
    bg = torch.tensor(background, dtype=torch.float64)
    outs = []
    for cam, order in zip(cams, orders):
        # order = (counts (H, W), seq) for a whole view, or (counts, seq, y0) for the row block
        # [y0, y0 + H) of it (the gradient of a sum over pixels can be taken block by block)
        counts, seq = order[0], order[1]
        y0 = order[2] if len(order) > 2 else 0
        H, W = counts.shape
        Wm = torch.tensor(np.asarray(cam.R_wc, np.float64).reshape(3, 3))
        o = torch.tensor(np.asarray(cam.position, np.float64))
        g = torch.as_tensor(seq.astype(np.int64))
        pix = torch.as_tensor(np.repeat(np.arange(H * W), counts.reshape(-1)))
        jj, ii = pix // W + y0, pix % W
        x = ((ii.double() + 0.5) - cam.cx) / cam.fx
        y = ((jj.double() + 0.5) - cam.cy) / cam.fy
        # O1-O5 for the blended Gaussians (per entry; the same Gaussian repeats)
        v = mu[g] - o
        muc = v @ Wm.T
        r = muc.norm(dim=1)
        u = muc / r[:, None]
        h = torch.sqrt(u[:, 2] ** 2 + u[:, 0] ** 2)
        e1 = torch.stack([u[:, 2] / h, torch.zeros_like(h), -u[:, 0] / h], 1)
        e2 = torch.stack([u[:, 1] * e1[:, 2], u[:, 2] * e1[:, 0] - u[:, 0] * e1[:, 2], -u[:, 1] * e1[:, 0]], 1)
        Sc = Wm @ cov[g] @ Wm.T
        r2 = r * r
        s00 = torch.einsum("ni,nij,nj->n", e1, Sc, e1) / r2
        s01 = torch.einsum("ni,nij,nj->n", e1, Sc, e2) / r2
        s11 = torch.einsum("ni,nij,nj->n", e2, Sc, e2) / r2
        jx, jy = u[:, 2] / cam.fx, u[:, 2] / cam.fy  # O4: +0.3 px^2 mapped to the chart (L5)
        J00, J01, J10, J11 = e1[:, 0] * jx, e1[:, 1] * jy, e2[:, 0] * jx, e2[:, 1] * jy
        s00 = s00 + 0.3 * (J00 * J00 + J01 * J01)
        s01 = s01 + 0.3 * (J00 * J10 + J01 * J11)
        s11 = s11 + 0.3 * (J10 * J10 + J11 * J11)
        det = s00 * s11 - s01 * s01
        c00, c01, c11 = s11 / det, -s01 / det, s00 / det
        A = Wm @ icov[g] @ Wm.T
        b = torch.einsum("nij,nj->ni", A, muc)
        dirs = v / v.norm(dim=1, keepdim=True)
        rgb = torch.clamp(torch.einsum("nk,nkc->nc", sh_basis(dirs, sh_degree), params["sh"][g]) + 0.5, min=0.0)
        # O10 per sample
        d = torch.stack([x, y, torch.ones_like(x)], 1)
        s = (u * d).sum(1)
        ex, ey = (e1 * d).sum(1), (e2 * d).sum(1)
        num = c00 * ex * ex + 2.0 * c01 * ex * ey + c11 * ey * ey
        q = num / (s * s)
        alpha = torch.clamp(sig[g] * torch.exp(-0.5 * q), max=0.99)
        den = torch.einsum("ni,nij,nj->n", d, A, d)
        tau = torch.clamp((d * b).sum(1) / den, min=near)
        # O11 front to back in the given order: T_k = prod_{j<k} (1 - alpha_j) per pixel
        la = torch.log1p(-alpha)
        csum = torch.cumsum(la, 0)
        starts = np.concatenate([[0], np.cumsum(counts.reshape(-1))[:-1]])
        seg_off = torch.as_tensor(np.repeat(starts, counts.reshape(-1)))
        base = torch.where(seg_off > 0, csum[(seg_off - 1).clamp(min=0)], torch.zeros_like(csum))
        T = torch.exp(csum - la - base)
        wgt = alpha * T
        dn = d.norm(dim=1)
        npx = H * W
        Cc = torch.zeros(npx, 3, dtype=torch.float64).index_add(0, pix, rgb * wgt[:, None])
        Dd = torch.zeros(npx, dtype=torch.float64).index_add(0, pix, tau * dn * wgt)
        logT = torch.zeros(npx, dtype=torch.float64).index_add(0, pix, la)
        Tf = torch.exp(logT)
        rgba = torch.cat([Cc + Tf[:, None] * bg, (1.0 - Tf)[:, None]], 1)
        outs.append((rgba.reshape(H, W, 4), Dd.reshape(H, W)))
    return outs


def to_params(scene, requires_grad=True):
    p = {"means": scene.means, "quats": scene.quats, "log_scales": scene.log_scales, "logits": scene.logits,
         "sh": scene.sh}
    return {k: torch.tensor(np.asarray(v, np.float64), requires_grad=requires_grad) for k, v in p.items()}


def gradients_blocked(scene, cams, orders, g_rgba, g_depth, rows=64, near=0.2):
    """gradients() for large frames: L is a sum over pixels and every pixel's
    blend order is contiguous in seq, so the autograd graph is built and
    back-propagated one block of `rows` image rows at a time (leaf gradients
    accumulate); returns the gradient dict only."""
    p = to_params(scene)
    for cam, (counts, seq), gr, gd in zip(cams, orders, g_rgba, g_depth):
        H, W = counts.shape
        off = np.concatenate([[0], np.cumsum(counts.reshape(-1))])
        for y0 in range(0, H, rows):
            y1 = min(H, y0 + rows)
            if not (np.any(gr[y0:y1]) or np.any(gd[y0:y1])):
                continue  # no loss on these rows: no gradient from them
            sub = (counts[y0:y1], seq[off[y0 * W]:off[y1 * W]], y0)
            (rgba, dep), = render_fixed_order(p, [cam], [sub], scene.sh_degree, near)
            L = (rgba * torch.as_tensor(np.asarray(gr[y0:y1], np.float64))).sum() + \
                (dep * torch.as_tensor(np.asarray(gd[y0:y1], np.float64))).sum()
            L.backward()
    return {k: v.grad.numpy() for k, v in p.items()}


def gradients(scene, cams, orders, g_rgba, g_depth, near=0.2):
    """dL/d(raw parameters) for L = sum g_rgba . RGBA + g_depth . Depth (per view lists of images)."""
    p = to_params(scene)
    outs = render_fixed_order(p, cams, orders, scene.sh_degree, near)
    L = sum((rgba * torch.as_tensor(np.asarray(gr, np.float64))).sum() +
            (dep * torch.as_tensor(np.asarray(gd, np.float64))).sum()
            for (rgba, dep), gr, gd in zip(outs, g_rgba, g_depth))
    L.backward()
    return {k: v.grad.numpy() for k, v in p.items()}, [(a.detach().numpy(), d.detach().numpy()) for a, d in outs]
