"""ctypes front end of the C++ ORACLE (test infrastructure, NOT product code).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It never touches the
CUDA library and the CUDA library never touches it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
SPLAT_FLOATS = 48
NSTATS = 12
STAT_NAMES = ["pairs", "samples", "evaluations", "contributions", "overflow_samples", "terminated_samples",
              "tiles_high", "tiles_low", "tiles_hybrid", "tiles_invisible", "work_items", "visible_splats"]
# splat record field slices (oracle.cpp orc_get_splats)
SPLAT_FIELDS = {"valid": slice(0, 1), "muc": slice(1, 4), "u": slice(4, 7), "e1": slice(7, 10),
                "e2": slice(10, 13), "S2": slice(13, 16), "C": slice(16, 19), "eps": slice(19, 20),
                "m2": slice(20, 22), "Cp": slice(22, 25), "A": slice(25, 31), "bv": slice(31, 34), "rgb": slice(34, 37), "sigma": slice(37, 38),
                "qcut": slice(38, 39), "rect": slice(39, 43), "bbox": slice(43, 47), "count": slice(47, 48)}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = (f"g++ -O2 -ffp-contract=off -fno-fast-math -std=c++17 -shared -fPIC -pthread "
               f"-o {_LIB}.tmp {src} && mv {_LIB}.tmp {_LIB}")
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
    return _LIB


class _View(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("o", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("mask_slot", C.c_int32), ("fovea_enabled", C.c_int32), ("fovea_center", C.c_float * 2),
                ("fovea_radius", C.c_float * 2), ("fovea_ramp", C.c_float)]


class _Params(C.Structure):
    _fields_ = [("assign_tile", C.c_int32), ("window_k", C.c_int32), ("near_plane", C.c_float),
                ("background", C.c_float * 3), ("threads", C.c_int32), ("projection", C.c_int32),
                ("resort", C.c_int32), ("block_queue", C.c_int32), ("group_queue", C.c_int32),
                ("sort_mode", C.c_int32), ("tau_unclamped", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.orc_create.restype = vp
        L.orc_create.argtypes = [i64, i32, vp, vp, vp, vp, vp, C.POINTER(C.c_int64)]
        L.orc_destroy.argtypes = [vp]
        L.orc_num_gaussians.restype = i64
        L.orc_num_gaussians.argtypes = [vp]
        L.orc_get_activated.argtypes = [vp, vp, vp, vp, vp, vp]
        L.orc_set_mask.argtypes = [vp, i32, i32, i32, vp]
        L.orc_prepare.argtypes = [vp, i32, vp, vp]
        L.orc_num_pairs.restype = i64
        L.orc_num_pairs.argtypes = [vp]
        L.orc_get_counts.argtypes = [vp, vp]
        L.orc_get_pairs.argtypes = [vp, i32, vp, vp]
        L.orc_num_tiles.restype = i64
        L.orc_num_tiles.argtypes = [vp]
        L.orc_get_ranges.argtypes = [vp, vp]
        L.orc_get_tile_info.argtypes = [vp, i32, vp, vp]
        L.orc_get_splats.argtypes = [vp, i32, vp]
        L.orc_render.argtypes = [vp, vp, vp]
        L.orc_render_pixels.argtypes = [vp, i64, vp, vp, vp]
        L.orc_get_stats.argtypes = [vp, vp]
        L.orc_render_bruteforce.argtypes = [vp, i32, vp, vp]
        L.orc_tile_test.argtypes = [vp, i32, i64, i32, i32, i32, i32, vp]
        L.orc_sat.argtypes = [i32, i32, vp, vp]
        L.orc_sat_count.restype = i64
        L.orc_sat_count.argtypes = [i32, vp, i32, i32, i32, i32]
        L.orc_eq4_edge.restype = C.c_float
        L.orc_eq4_edge.argtypes = [vp, vp, vp, vp]
        L.orc_sample_depth.restype = C.c_float
        L.orc_sample_depth.argtypes = [vp, i32, i64, C.c_float, C.c_float]
        L.orc_hier_core.argtypes = [i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_sample_alpha_tau.argtypes = [i64, vp, vp, vp, vp, vp, C.c_float, vp, vp]
        L.orc_blend_orders.restype = i64
        L.orc_blend_orders.argtypes = [vp, i32, vp, vp, i64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def make_view(cam, fovea=None) -> _View:
    v = _View()
    v.R[:] = [float(x) for x in np.asarray(cam.R_wc, np.float32).reshape(9)]
    v.o[:] = [float(x) for x in np.asarray(cam.position, np.float32).reshape(3)]
    v.fx, v.fy, v.cx, v.cy = cam.fx, cam.fy, cam.cx, cam.cy
    v.width, v.height, v.mask_slot = cam.width, cam.height, cam.mask_slot
    if fovea is not None and fovea.enabled:
        v.fovea_enabled = 1
        v.fovea_center[:] = list(fovea.center)
        v.fovea_radius[:] = list(fovea.radius)
        v.fovea_ramp = fovea.ramp
    return v


class Oracle:
    """One scene + one prepared frame (views)."""

    def __init__(self, scene):
        L = lib()
        n = scene.n
        self._keep = [np.ascontiguousarray(a, np.float32) for a in
                      (scene.means, scene.quats, scene.log_scales, scene.logits, scene.sh)]
        rej = C.c_int64(0)
        self.h = L.orc_create(n, scene.sh_degree, *[_p(a) for a in self._keep], C.byref(rej))
        if not self.h:
            raise ValueError("orc_create failed")
        self.n_rejected = rej.value
        self.n = L.orc_num_gaussians(self.h)
        self.views = []

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def activated(self):
        n = self.n
        mu, cov, icov = np.zeros((n, 3), np.float32), np.zeros((n, 6), np.float32), np.zeros((n, 6), np.float32)
        sg, qc = np.zeros(n, np.float32), np.zeros(n, np.float32)
        lib().orc_get_activated(self.h, _p(mu), _p(cov), _p(icov), _p(sg), _p(qc))
        return dict(mu=mu, cov=cov, icov=icov, sigma=sg, qcut=qc)

    def set_mask(self, slot: int, mask):
        if mask is None:
            lib().orc_set_mask(self.h, slot, 0, 0, None)
        else:
            m = np.ascontiguousarray(mask, np.uint8)
            self._mask_keep = getattr(self, "_mask_keep", {})
            self._mask_keep[slot] = m
            lib().orc_set_mask(self.h, slot, m.shape[1], m.shape[0], _p(m))

    def prepare(self, cams, foveas=None, assign_tile=16, window_k=16, near=0.2, background=(0, 0, 0),
                threads=0, projection=0, resort=0, block_queue=8, group_queue=0, sort_mode=0, tau_unclamped=0):
        foveas = foveas if foveas is not None else [None] * len(cams)
        arr = (_View * len(cams))(*[make_view(c, f) for c, f in zip(cams, foveas)])
        p = _Params()
        p.assign_tile, p.window_k, p.near_plane = assign_tile, window_k, near
        p.background[:] = list(background)
        p.threads = threads
        p.projection = projection
        p.resort, p.block_queue, p.group_queue = resort, block_queue, group_queue
        p.sort_mode, p.tau_unclamped = sort_mode, tau_unclamped
        rc = lib().orc_prepare(self.h, len(cams), C.cast(arr, C.c_void_p), C.cast(C.pointer(p), C.c_void_p))
        if rc != 0:
            raise ValueError(f"orc_prepare rc={rc}")
        self.views = list(cams)
        self.assign_tile = assign_tile
        return self

    # ---- artefacts
    def num_pairs(self):
        return lib().orc_num_pairs(self.h)

    def counts(self):
        out = np.zeros(len(self.views) * self.n, np.uint32)
        lib().orc_get_counts(self.h, _p(out))
        return out

    def pairs(self, sorted_=True):
        P = self.num_pairs()
        k, v = np.zeros(P, np.uint64), np.zeros(P, np.uint32)
        lib().orc_get_pairs(self.h, 1 if sorted_ else 0, _p(k), _p(v))
        return k, v

    def ranges(self):
        out = np.zeros((lib().orc_num_tiles(self.h), 2), np.uint32)
        lib().orc_get_ranges(self.h, _p(out))
        return out

    def tile_info(self, view):
        cam = self.views[view]
        T = self.assign_tile
        tw, th = (cam.width + T - 1) // T, (cam.height + T - 1) // T
        cls, vis = np.zeros(tw * th, np.int32), np.zeros(tw * th, np.int32)
        lib().orc_get_tile_info(self.h, view, _p(cls), _p(vis))
        return cls.reshape(th, tw), vis.reshape(th, tw)

    def splats(self, view):
        out = np.zeros((self.n, SPLAT_FLOATS), np.float32)
        lib().orc_get_splats(self.h, view, _p(out))
        return out

    def render(self):
        tot = sum(c.width * c.height for c in self.views)
        rgba, depth = np.zeros((tot, 4), np.float32), np.zeros(tot, np.float32)
        lib().orc_render(self.h, _p(rgba), _p(depth))
        outs, off = [], 0
        for c in self.views:
            k = c.width * c.height
            outs.append((rgba[off:off + k].reshape(c.height, c.width, 4), depth[off:off + k].reshape(c.height, c.width)))
            off += k
        return outs

    def render_pixels(self, vxy):
        vxy = np.ascontiguousarray(vxy, np.int32)
        n = vxy.shape[0]
        rgba, depth = np.zeros((n, 4), np.float32), np.zeros(n, np.float32)
        lib().orc_render_pixels(self.h, n, _p(vxy), _p(rgba), _p(depth))
        return rgba, depth

    def stats(self):
        out = np.zeros(NSTATS, np.int64)
        lib().orc_get_stats(self.h, _p(out))
        return dict(zip(STAT_NAMES, out.tolist()))

    def bruteforce(self, view):
        c = self.views[view]
        rgba, depth = np.zeros((c.height, c.width, 4), np.float32), np.zeros((c.height, c.width), np.float32)
        lib().orc_render_bruteforce(self.h, view, _p(rgba), _p(depth))
        return rgba, depth

    def tile_test(self, view, g, x0, y0, x1, y1):
        out = np.zeros(6, np.float32)
        lib().orc_tile_test(self.h, view, g, x0, y0, x1, y1, _p(out))
        return dict(keep=out[0], qmin=out[1], t=out[2], dhat=out[3:6].copy())

    def blend_orders(self, view):
        """Per pixel of a non-foveated view: the Gaussians it blended, front to back (O10-O11).
        Returns (counts (H, W) int32, seq uint32) with seq the concatenated per-pixel lists (row-major)."""
        c = self.views[view]
        counts = np.zeros(c.width * c.height, np.int32)
        tot = lib().orc_blend_orders(self.h, view, _p(counts), None, 0)
        if tot < 0:
            raise ValueError("blend orders need a non-foveated view")
        seq = np.zeros(max(tot, 1), np.uint32)
        lib().orc_blend_orders(self.h, view, _p(counts), _p(seq), tot)
        return counts.reshape(c.height, c.width), seq[:tot]

    def sample_depth(self, view, g, x, y):
        return lib().orc_sample_depth(self.h, view, g, x, y)


def sat(bits: np.ndarray) -> np.ndarray:
    th, tw = bits.shape
    b = np.ascontiguousarray(bits, np.uint8)
    out = np.zeros((th + 1) * (tw + 1), np.uint32)
    lib().orc_sat(tw, th, _p(b), _p(out))
    return out.reshape(th + 1, tw + 1)


def sat_count(satt: np.ndarray, x0, y0, x1, y1) -> int:
    s = np.ascontiguousarray(satt, np.uint32)
    return lib().orc_sat_count(s.shape[1] - 1, _p(s), x0, y0, x1, y1)


def eq4_edge(Cc, p, d):
    Cc, p, d = (np.ascontiguousarray(a, np.float32) for a in (Cc, p, d))
    xh = np.zeros(2, np.float32)
    q = lib().orc_eq4_edge(_p(Cc), _p(p), _p(d), _p(xh))
    return q, xh


def sample_alpha_tau(num, ss, den, dtb, sigma, near=0.2):
    """Pin hook: the contract's per-sample alpha and tau (DESIGN R9) on float32 arrays."""
    a = [np.ascontiguousarray(np.broadcast_to(np.asarray(x, np.float32), np.shape(num))) for x in
         (num, ss, den, dtb, sigma)]
    n = a[0].size
    alpha, tau = np.zeros(n, np.float32), np.zeros(n, np.float32)
    lib().orc_sample_alpha_tau(n, *[_p(x) for x in a], near, _p(alpha), _p(tau))
    return alpha.reshape(np.shape(num)), tau.reshape(np.shape(num))


def hier_core(tau_b, g, member, tau, alpha, rgb, kb, kp, kg=0, tau_g=None):
    """Pin H3 hook: the N2 queue cascade on a given block stream (n entries;
    tau/alpha are n x 16, tau_g n x 4 (default: tau_b for every group)).
    Returns (out 16 x (r, g, b, a, depth), stats 16 x (evals, contribs, overflow, term))."""
    n = len(tau_b)
    if tau_g is None:
        tau_g = np.repeat(np.asarray(tau_b, np.float32)[:, None], 4, 1)
    a = [np.ascontiguousarray(x, t) for x, t in ((tau_b, np.float32), (tau_g, np.float32), (g, np.uint32),
                                                 (member, np.uint32), (tau, np.float32), (alpha, np.float32),
                                                 (rgb, np.float32))]
    out, st = np.zeros((16, 5), np.float64), np.zeros((16, 4), np.int64)
    lib().orc_hier_core(n, kb, kg, kp, *[_p(x) for x in a], _p(out), _p(st))
    return out, st
