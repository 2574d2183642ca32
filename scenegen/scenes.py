"""Seeded synthetic scenes, cameras, masks and fovea settings.

Test/bench input infrastructure only (no arithmetic of the rendering method).
Recipes follow SURVEY.md §8(d) "Synthetic inputs" and "vr_room attribute
distributions"; they are restated in DESIGN.md §"Input recipe".

Raw attributes use the de-facto 3DGS storage convention that the C ABI
ingests: means (n,3) f32, quaternions (n,4) f32 in
(w,x,y,z) order, log-scales (n,3) f32, opacity logits (n,) f32 and SH
coefficients (n,(deg+1)^2,3) f32, coefficient-major RGB.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rng import Stream


@dataclass
class RawScene:
    means: np.ndarray
    quats: np.ndarray
    log_scales: np.ndarray
    logits: np.ndarray
    sh: np.ndarray
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx) -> "RawScene":
        return RawScene(self.means[idx].copy(), self.quats[idx].copy(), self.log_scales[idx].copy(),
                        self.logits[idx].copy(), self.sh[idx].copy(), self.sh_degree)


@dataclass
class Camera:
    """Pinhole camera, OpenCV axes (x right, y down, z forward).

    R_wc: world->camera rotation (row-major 3x3); position: eye centre o.
    Pixel (i, j) has its centre at (i + 0.5, j + 0.5).
    """
    R_wc: np.ndarray
    position: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    mask_slot: int = -1


@dataclass
class Fovea:
    """Full-rate rectangle centre +- radius (px half-extents); ramp = padding
    width as a fraction of the full-rate extent."""
    center: tuple
    radius: tuple
    ramp: float = 0.10
    enabled: int = 1


# ----------------------------------------------------------------------------- helpers

def _uniform_quats(s: Stream, n: int) -> np.ndarray:
    """Uniform random unit quaternions (Shoemake), (w,x,y,z)."""
    u1, u2, u3 = s.uniform(n), s.uniform(n), s.uniform(n)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    return np.stack([b * np.cos(2 * np.pi * u3), a * np.sin(2 * np.pi * u2),
                     a * np.cos(2 * np.pi * u2), b * np.sin(2 * np.pi * u3)], axis=1)


def _uniform_dirs(s: Stream, n: int) -> np.ndarray:
    z = s.uniform(n, -1.0, 1.0)
    phi = s.uniform(n, 0.0, 2 * np.pi)
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def _mat_to_quat(R: np.ndarray) -> np.ndarray:
    """Rotation matrices (n,3,3) -> unit quaternions (w,x,y,z) (input generation only)."""
    n = R.shape[0]
    q = np.zeros((n, 4))
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    m0 = tr > 0
    m1 = (~m0) & (R[:, 0, 0] >= R[:, 1, 1]) & (R[:, 0, 0] >= R[:, 2, 2])
    m2 = (~m0) & (~m1) & (R[:, 1, 1] >= R[:, 2, 2])
    m3 = (~m0) & (~m1) & (~m2)
    if m0.any():
        S = np.sqrt(tr[m0] + 1.0) * 2
        r = R[m0]
        q[m0] = np.stack([0.25 * S, (r[:, 2, 1] - r[:, 1, 2]) / S, (r[:, 0, 2] - r[:, 2, 0]) / S,
                          (r[:, 1, 0] - r[:, 0, 1]) / S], 1)
    if m1.any():
        r = R[m1]
        S = np.sqrt(1.0 + r[:, 0, 0] - r[:, 1, 1] - r[:, 2, 2]) * 2
        q[m1] = np.stack([(r[:, 2, 1] - r[:, 1, 2]) / S, 0.25 * S, (r[:, 0, 1] + r[:, 1, 0]) / S,
                          (r[:, 0, 2] + r[:, 2, 0]) / S], 1)
    if m2.any():
        r = R[m2]
        S = np.sqrt(1.0 + r[:, 1, 1] - r[:, 0, 0] - r[:, 2, 2]) * 2
        q[m2] = np.stack([(r[:, 0, 2] - r[:, 2, 0]) / S, (r[:, 0, 1] + r[:, 1, 0]) / S, 0.25 * S,
                          (r[:, 1, 2] + r[:, 2, 1]) / S], 1)
    if m3.any():
        r = R[m3]
        S = np.sqrt(1.0 + r[:, 2, 2] - r[:, 0, 0] - r[:, 1, 1]) * 2
        q[m3] = np.stack([(r[:, 1, 0] - r[:, 0, 1]) / S, (r[:, 0, 2] + r[:, 2, 0]) / S,
                          (r[:, 1, 2] + r[:, 2, 1]) / S, 0.25 * S], 1)
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _normal_aligned_quats(s: Stream, normals: np.ndarray) -> np.ndarray:
    """Frames whose 3rd axis is the surface normal, in-plane angle U(0, 2pi)."""
    n = normals.shape[0]
    helper = np.where(np.abs(normals[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]))
    t1 = np.cross(helper, normals)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(normals, t1)
    th = s.uniform(n, 0.0, 2 * np.pi)[:, None]
    a1 = np.cos(th) * t1 + np.sin(th) * t2
    a2 = np.cross(normals, a1)
    R = np.stack([a1, a2, normals], axis=2)  # columns = principal axes
    return _mat_to_quat(R)


def _logit(p: np.ndarray) -> np.ndarray:
    return np.log(p / (1.0 - p))


def _sh(s: Stream, n: int, degree: int, dc_std: float, hi_std: float) -> np.ndarray:
    k = (degree + 1) ** 2
    sh = np.zeros((n, k, 3))
    sh[:, 0, :] = s.normal(n * 3, 0.0, dc_std).reshape(n, 3)
    for l in range(1, degree + 1):
        for m in range(l * l, (l + 1) * (l + 1)):
            sh[:, m, :] = s.normal(n * 3, 0.0, hi_std / l).reshape(n, 3)
    return sh


def _pack(means, quats, log_scales, opac, sh, degree) -> RawScene:
    return RawScene(np.ascontiguousarray(means, np.float32), np.ascontiguousarray(quats, np.float32),
                    np.ascontiguousarray(log_scales, np.float32),
                    np.ascontiguousarray(_logit(opac), np.float32), np.ascontiguousarray(sh, np.float32),
                    degree)


# ----------------------------------------------------------------------------- scenes

def random_scene(seed: int, n: int = 1000, sh_degree: int = 0, z_range=(2.0, 8.0), xy_frac=0.9,
                 log_scale_range=(math.log(0.02), math.log(0.3)), opacity_range=(0.05, 0.99)) -> RawScene:
    """Config C1: mu z~U(2,8), x,y~U(-0.9,0.9)*z; scales
    exp(U(ln .02, ln .3)) per axis; uniform quaternion; sigma~U(.05,.99); DC~N(0,1)."""
    s = Stream(seed, 1)
    z = s.uniform(n, *z_range)
    x = s.uniform(n, -xy_frac, xy_frac) * z
    y = s.uniform(n, -xy_frac, xy_frac) * z
    means = np.stack([x, y, z], 1)
    log_scales = s.uniform(n * 3, *log_scale_range).reshape(n, 3)
    quats = _uniform_quats(s, n)
    opac = s.uniform(n, *opacity_range)
    sh = _sh(s, n, sh_degree, 1.0, 0.1)
    return _pack(means, quats, log_scales, opac, sh, sh_degree)


def vr_room(seed: int, n: int, scale_mul: float = 1.0, sh_degree: int = 3) -> RawScene:
    """The "vr_room" scene of SURVEY §8(d): 80% surface shell at 6 m, 17% object
    clusters (64 clusters, r~U(1.5,4.5)), 3% far dome at 30 m.  Means with
    |mu|<1 m are resampled.  Opacity 55% U(.7,.99) / 45% U(.02,.7); SH DC~N(0,.8),
    band l>=1 ~ N(0, .08/l).  ``scale_mul`` rescales every scale (C3: sqrt(1/6),
    C4: 0.707)."""
    s = Stream(seed, 2)
    n_shell = int(round(0.80 * n))
    n_obj = int(round(0.17 * n))
    n_dome = n - n_shell - n_obj
    ln_mul = math.log(scale_mul)

    # surface shell
    dirs = _uniform_dirs(s, n_shell)
    rad = 6.0 + s.normal(n_shell, 0.0, 0.02)
    m_shell = dirs * rad[:, None]
    q_shell = _normal_aligned_quats(s, dirs)
    tang = s.normal(n_shell * 2, math.log(0.04), 0.35).reshape(n_shell, 2)
    ls_shell = np.concatenate([tang, (math.log(0.15) + tang.min(axis=1))[:, None]], 1)

    # object clusters
    n_cl = 64
    c_dir = _uniform_dirs(s, n_cl)
    c_r = s.uniform(n_cl, 1.5, 4.5)
    centres = c_dir * c_r[:, None]
    spread = s.uniform(n_cl, 0.1, 0.4)
    cid = s.integers(n_obj, 0, n_cl)
    m_obj = centres[cid] + s.normal(n_obj * 3).reshape(n_obj, 3) * spread[cid][:, None]
    for _ in range(64):
        bad = np.nonzero(np.linalg.norm(m_obj, axis=1) < 1.0)[0]
        if bad.size == 0:
            break
        m_obj[bad] = centres[cid[bad]] + s.normal(bad.size * 3).reshape(bad.size, 3) * spread[cid[bad]][:, None]
    q_obj = _uniform_quats(s, n_obj)
    ls_obj = s.normal(n_obj * 3, math.log(0.015), 0.4).reshape(n_obj, 3)

    # far dome
    ddirs = _uniform_dirs(s, n_dome)
    m_dome = ddirs * 30.0
    q_dome = _normal_aligned_quats(s, ddirs)
    dt = s.normal(n_dome * 2, math.log(0.5), 0.3).reshape(n_dome, 2)
    ls_dome = np.concatenate([dt, (math.log(0.2) + dt.min(axis=1))[:, None]], 1)

    means = np.concatenate([m_shell, m_obj, m_dome])
    quats = np.concatenate([q_shell, q_obj, q_dome])
    log_scales = np.concatenate([ls_shell, ls_obj, ls_dome]) + ln_mul
    # interleave components deterministically so that any prefix/shard is representative
    perm = np.argsort(s.u64(n), kind="stable")
    means, quats, log_scales = means[perm], quats[perm], log_scales[perm]
    hi = s.uniform(n) < 0.55
    opac = np.where(hi, s.uniform(n, 0.7, 0.99), s.uniform(n, 0.02, 0.7))
    sh = _sh(s, n, sh_degree, 0.8, 0.08)
    return _pack(means, quats, log_scales, opac, sh, sh_degree)


# ----------------------------------------------------------------------------- cameras

def look_camera(position, yaw=0.0, pitch=0.0, roll=0.0, *, f, width, height, cx=None, cy=None,
                mask_slot=-1) -> Camera:
    """Camera at ``position`` looking along +z rotated by yaw (about y), pitch
    (about x), roll (about z); angles in radians.  R_wc = (Ry Rx Rz)^T."""
    cyw, syw = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cr, sr = math.cos(roll), math.sin(roll)
    Ry = np.array([[cyw, 0, syw], [0, 1, 0], [-syw, 0, cyw]])
    Rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    Rz = np.array([[cr, -sr, 0], [sr, cr, 0], [0, 0, 1]])
    R_cw = Ry @ Rx @ Rz
    return Camera(np.ascontiguousarray(R_cw.T, np.float32), np.asarray(position, np.float32), float(f), float(f),
                  float(width / 2 if cx is None else cx), float(height / 2 if cy is None else cy), int(width),
                  int(height), mask_slot)


def focal_for_hfov(width: int, hfov_deg: float) -> float:
    """horizontal symmetric FoV, square pixels: f = (W/2)/tan(hfov/2)."""
    return (width / 2.0) / math.tan(math.radians(hfov_deg) / 2.0)


QUEST_W, QUEST_H = 2064, 2208
IPD = 0.063


def stereo_pair(head=(0.0, 0.0, 0.0), yaw=0.0, pitch=0.0, roll=0.0, *, width=QUEST_W, height=QUEST_H,
                hfov_deg=110.0, masks=True):
    """Config C2 eyes: x = -+IPD/2 in the head frame, looking +z, f = 1032/tan(55 deg)."""
    f = focal_for_hfov(width, hfov_deg)
    cams = []
    cyw, syw = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cr, sr = math.cos(roll), math.sin(roll)
    Ry = np.array([[cyw, 0, syw], [0, 1, 0], [-syw, 0, cyw]])
    Rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    Rz = np.array([[cr, -sr, 0], [sr, cr, 0], [0, 0, 1]])
    R_cw = Ry @ Rx @ Rz
    for e, off in enumerate((-IPD / 2, IPD / 2)):
        pos = np.asarray(head, np.float64) + R_cw @ np.array([off, 0.0, 0.0])
        cams.append(Camera(np.ascontiguousarray(R_cw.T, np.float32), pos.astype(np.float32), f, f, width / 2.0,
                           height / 2.0, width, height, e if masks else -1))
    return cams


def trajectory_pose(t: int):
    """Config C4 head pose t in 0..359."""
    yaw = math.radians(60.0) * math.sin(2 * math.pi * t / 360)
    pitch = math.radians(15.0) * math.sin(4 * math.pi * t / 360)
    roll = math.radians(3.0) * math.sin(6 * math.pi * t / 360)
    head = (0.05 * math.sin(2 * math.pi * t / 120), 0.02 * math.sin(2 * math.pi * t / 90),
            0.05 * math.sin(2 * math.pi * t / 180))
    return head, yaw, pitch, roll


def ellipse_mask(width: int, height: int, s: float = 1.0859) -> np.ndarray:
    """Synthetic HMD visibility mask: centred ellipse with
    semi-axes s*(W/2, H/2), evaluated at pixel centres; uint8 (1 = visible)."""
    x = (np.arange(width) + 0.5 - width / 2.0) / (s * width / 2.0)
    y = (np.arange(height) + 0.5 - height / 2.0) / (s * height / 2.0)
    return ((x[None, :] ** 2 + y[:, None] ** 2) <= 1.0).astype(np.uint8)


def quest_fovea(width=QUEST_W, height=QUEST_H, ramp=0.10) -> Fovea:
    """P:461 "half the rendered image size, with 10% padding": radius = (W/4, H/4)."""
    return Fovea((width / 2.0, height / 2.0), (width / 4.0, height / 4.0), ramp, 1)
