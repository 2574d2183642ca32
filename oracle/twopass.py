"""ORACLE (test infrastructure, NOT product code) of the two-pass foveated
baseline, SURVEY §8f N1 / PAPER App. A, SPEC
``render_foveated_two_pass`` / ``crop_frustum``.

Written from the paper and DESIGN.md's N1 readings, independently of the
CUDA library: the two passes are ordinary renders of the C++ oracle
(``Oracle.prepare/render``); the pass geometry, the 2x2-OR mask reduction,
the bilinear upsample and the blend are plain numpy in float64.

* Pass-1 rectangle (N1-R1): the pixels whose fovea blend weight can be
  non-zero -- half-extents radius*(1 + 2*ramp) around the centre (the weight
  ramps to 0 over ramp * full extent) -- plus one pixel of margin,
  clipped to the view.  Pass 1 renders it through the cropped camera of
  ``crop_camera`` (principal point shifted by the integer origin).
* Pass 2 (N1-R2): the whole view at half resolution, focal lengths and
  principal point halved, ceil(W/2) x ceil(H/2) pixels, honouring the
  visibility mask reduced by 2x2 OR ("also considering the visibility
  mask").
* Upsample (N1-R3): bilinear, pixel-centre aligned (full-resolution pixel i
  reads pass-2 coordinate (i - 0.5)/2), edge clamped: the NPP resize
  convention the paper uses.
* Blend (N1-R4): w * P1 + (1 - w) * up(P2) for RGBA and depth, w the same
  continuous fovea weight as the single-pass hybrid ramp ("the
  size of the center and transitional region ... identical to Ours").
"""
from __future__ import annotations

import math
from dataclasses import replace

import numpy as np


def pass1_rect(cam, fov):
    """(i0, j0, i1, j1): pixels with a possibly non-zero blend weight, +1 px, clipped."""
    gx, gy = float(np.float32(fov.center[0])), float(np.float32(fov.center[1]))
    ex = float(np.float32(fov.radius[0])) * (1.0 + 2.0 * float(np.float32(fov.ramp)))
    ey = float(np.float32(fov.radius[1])) * (1.0 + 2.0 * float(np.float32(fov.ramp)))
    i0 = int(min(max(0.0, math.floor(gx - ex) - 1.0), cam.width - 1.0))
    j0 = int(min(max(0.0, math.floor(gy - ey) - 1.0), cam.height - 1.0))
    i1 = int(max(min(float(cam.width), math.ceil(gx + ex) + 1.0), i0 + 1.0))
    j1 = int(max(min(float(cam.height), math.ceil(gy + ey) + 1.0), j0 + 1.0))
    return i0, j0, i1, j1


def crop_camera(cam, rect):
    """S:401-409 crop_frustum: pixel (a, b) of the result casts the parent's ray of
    pixel (i0 + a, j0 + b) (the principal point moves by the integer origin)."""
    i0, j0, i1, j1 = rect
    return replace(cam, cx=float(np.float32(cam.cx) - np.float32(i0)), cy=float(np.float32(cam.cy) - np.float32(j0)),
                   width=i1 - i0, height=j1 - j0, mask_slot=-1)


def half_camera(cam, mask_slot=-1):
    """Half resolution: pixel (a, b) centre = parent position (2a + 1, 2b + 1)."""
    h = np.float32(0.5)
    return replace(cam, fx=float(np.float32(cam.fx) * h), fy=float(np.float32(cam.fy) * h),
                   cx=float(np.float32(cam.cx) * h), cy=float(np.float32(cam.cy) * h),
                   width=(cam.width + 1) // 2, height=(cam.height + 1) // 2, mask_slot=mask_slot)


def half_mask(mask):
    """Visibility at half resolution: a pixel is visible iff any of its (up to) 2x2 pixels is."""
    m = np.asarray(mask, np.uint8)
    H, W = m.shape
    H2, W2 = (H + 1) // 2, (W + 1) // 2
    out = np.zeros((H2, W2), np.uint8)
    for b in range(2):
        for a in range(2):
            sub = m[b::2, a::2]
            out[:sub.shape[0], :sub.shape[1]] |= sub
    return (out != 0).astype(np.uint8)


def fovea_weight(fov, px, py):
    """weight 1 inside the full-rate rectangle, ramping linearly to 0 over
    ramp * (full-rate extent) outside it (separable max of the two ramps)."""
    gx, gy = float(fov.center[0]), float(fov.center[1])
    rx, ry, ramp = float(fov.radius[0]), float(fov.radius[1]), float(fov.ramp)
    ax = np.maximum(np.abs(px - gx) - rx, 0.0)
    ay = np.maximum(np.abs(py - gy) - ry, 0.0)
    dxn, dyn = ramp * 2.0 * rx, ramp * 2.0 * ry
    wx = ax / dxn if dxn > 0 else (ax > 0).astype(np.float64)
    wy = ay / dyn if dyn > 0 else (ay > 0).astype(np.float64)
    return np.clip(1.0 - np.maximum(wx, wy), 0.0, 1.0)


def bilinear_up(img2, W, H):
    """Upsample a (H2, W2, C) pass-2 image to (H, W, C): pixel i reads
    coordinate (i - 0.5)/2, bilinear weights, edge clamping."""
    img2 = np.asarray(img2, np.float64)
    H2, W2 = img2.shape[:2]
    u = (np.arange(W) - 0.5) / 2.0
    v = (np.arange(H) - 0.5) / 2.0
    fu, fv = np.floor(u), np.floor(v)
    ax, ay = u - fu, v - fv
    xa = np.clip(fu.astype(np.int64), 0, W2 - 1)
    xb = np.clip(fu.astype(np.int64) + 1, 0, W2 - 1)
    ya = np.clip(fv.astype(np.int64), 0, H2 - 1)
    yb = np.clip(fv.astype(np.int64) + 1, 0, H2 - 1)
    ax = ax[None, :, None] if img2.ndim == 3 else ax[None, :]
    ay = ay[:, None, None] if img2.ndim == 3 else ay[:, None]
    r0, r1 = img2[ya], img2[yb]
    top = (1 - ax) * r0[:, xa] + ax * r0[:, xb]
    bot = (1 - ax) * r1[:, xa] + ax * r1[:, xb]
    return (1 - ay) * top + ay * bot


def combine(p1, p2, rect, fov, W, H):
    """Final view: up(P2) everywhere, blended with P1 by w inside the pass-1 rectangle."""
    (c1, d1), (c2, d2) = p1, p2
    col = bilinear_up(c2, W, H)
    dep = bilinear_up(d2, W, H)
    i0, j0, i1, j1 = rect
    py, px = np.mgrid[j0:j1, i0:i1]
    w = fovea_weight(fov, px + 0.5, py + 0.5)
    col[j0:j1, i0:i1] = w[..., None] * np.asarray(c1, np.float64) + (1 - w[..., None]) * col[j0:j1, i0:i1]
    dep[j0:j1, i0:i1] = w * np.asarray(d1, np.float64) + (1 - w) * dep[j0:j1, i0:i1]
    return col, dep


def pass_cameras(cams, foveas, half_slot=lambda s: s):
    """Pass-1 cameras, pass-2 cameras and the pass-1 rectangles of a frame."""
    rects = [pass1_rect(c, f) for c, f in zip(cams, foveas)]
    c1 = [crop_camera(c, r) for c, r in zip(cams, rects)]
    c2 = [half_camera(c, half_slot(c.mask_slot) if c.mask_slot >= 0 else -1) for c in cams]
    return c1, c2, rects


def render_two_pass(oracle_mod, scene, cams, foveas, masks=None, assign_tile=16, threads=0, background=(0, 0, 0)):
    """Oracle two-pass frame: list of (rgba (H, W, 4), depth (H, W)) float64 per view,
    plus the oracle object of the 2n-view pass frame (for counters)."""
    masks = masks or {}
    o = oracle_mod.Oracle(scene)
    for slot, m in masks.items():
        o.set_mask(slot, half_mask(m))  # pass 2 is the only masked pass
    c1, c2, rects = pass_cameras(cams, foveas)
    o.prepare(c1 + c2, None, assign_tile=assign_tile, threads=threads, background=background)
    imgs = o.render()
    n = len(cams)
    out = [combine(imgs[i], imgs[n + i], rects[i], foveas[i], cams[i].width, cams[i].height) for i in range(n)]
    return out, o
