"""Evaluation protocols around the render path (host-side numpy; no method
arithmetic).  SURVEY §8f N3: the paper's large-FOV protocol (App. D,
P:835-843; SPEC ``large_fov_protocol`` / ``psnr``)."""
from __future__ import annotations

import math
from dataclasses import replace

import numpy as np


def psnr(a, b, max_val: float = 1.0) -> float:
    """10 log10(MAX^2 / MSE) over all channels; +inf for identical images."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"DimensionMismatch {a.shape} vs {b.shape}")
    mse = float(np.mean((a - b) ** 2)) if a.size else 0.0
    return math.inf if mse == 0.0 else 10.0 * math.log10(max_val * max_val / mse)


def wide_camera(cam, factor: int = 3):
    """App. D: same pixel focal length, factor x resolution, principal point moved
    by the original size, so the centre crop [W, 2W) x [H, 2H) casts the original
    rays pixel for pixel (no interpolation)."""
    k = factor // 2
    return replace(cam, cx=float(cam.cx + k * cam.width), cy=float(cam.cy + k * cam.height),
                   width=factor * cam.width, height=factor * cam.height, mask_slot=-1)


def centre_crop(img, cam, factor: int = 3):
    k = factor // 2
    return img[k * cam.height:(k + 1) * cam.height, k * cam.width:(k + 1) * cam.width]
