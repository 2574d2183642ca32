"""Shared test helpers (input construction only; no method arithmetic)."""
from __future__ import annotations

import math

import numpy as np

import scenegen as sg


def scene_from(means, scales, quats=None, opacities=None, dc=None, sh_degree=0):
    """Build a RawScene from activated-style parameters (log/logit applied here)."""
    means = np.asarray(means, np.float64).reshape(-1, 3)
    n = means.shape[0]
    scales = np.broadcast_to(np.asarray(scales, np.float64), (n, 3))
    quats = np.broadcast_to(np.asarray([1.0, 0, 0, 0] if quats is None else quats, np.float64), (n, 4))
    op = np.broadcast_to(np.asarray(0.8 if opacities is None else opacities, np.float64), (n,))
    k = (sh_degree + 1) ** 2
    sh = np.zeros((n, k, 3))
    if dc is not None:
        sh[:, 0, :] = np.broadcast_to(np.asarray(dc, np.float64), (n, 3))
    return sg.RawScene(means.astype(np.float32).copy(), quats.astype(np.float32).copy(),
                       np.log(scales).astype(np.float32).copy(),
                       np.log(op / (1.0 - op)).astype(np.float32).copy(), sh.astype(np.float32), sh_degree)


def identity_camera(width, height, f, cx=None, cy=None, position=(0.0, 0.0, 0.0), mask_slot=-1):
    return sg.Camera(np.eye(3, dtype=np.float32), np.asarray(position, np.float32), float(f), float(f),
                     float(width / 2 if cx is None else cx), float(height / 2 if cy is None else cy),
                     int(width), int(height), mask_slot)


def quat_to_R(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def rot_to_quat(R):
    from scenegen.scenes import _mat_to_quat
    return _mat_to_quat(np.asarray(R, np.float64)[None])[0]


C0 = 0.28209479177387814


def tiny_set(seed):
    """Brute-force pin set (seeds 100-199, N in {1,2,8,32,64}, 32^2/64^2)."""
    n = [1, 2, 8, 32, 64][seed % 5]
    res = 32 if (seed // 5) % 2 == 0 else 64
    scene = sg.random_scene(seed, n=n, sh_degree=0)
    cam = identity_camera(res, res, res / 2.0)
    return scene, cam


def lowres_compose(samples_low, cls, T, W, H):
    """Independent numpy restatement of P:438 (NN upsample + renormalised 3x3
    (1,2,1)^2 blur restricted to LowRes-class in-image pixels).  samples_low
    is indexed [j//2, i//2]."""
    jj, ii = np.mgrid[0:H, 0:W]
    nn = samples_low[jj // 2, ii // 2]
    pcls = cls[jj // T, ii // T]
    low = (pcls == 1)
    acc = np.zeros(nn.shape, np.float64)
    wsum = np.zeros((H, W), np.float64)
    for dj in (-1, 0, 1):
        for di in (-1, 0, 1):
            w = (2 - abs(di)) * (2 - abs(dj))
            src_j, src_i = jj + dj, ii + di
            ok = (src_j >= 0) & (src_j < H) & (src_i >= 0) & (src_i < W)
            sj, si = np.clip(src_j, 0, H - 1), np.clip(src_i, 0, W - 1)
            ok &= low[sj, si]
            acc += np.where(ok[..., None], w * nn[sj, si], 0.0)
            wsum += np.where(ok, w, 0.0)
    return acc / np.maximum(wsum, 1e-30)[..., None], low
