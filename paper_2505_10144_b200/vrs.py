"""ctypes binding of include/vrs.h (same names as the C ABI).

Marshalling only: host structs are built from Python objects, device buffers
are torch CUDA tensors passed by ``data_ptr()``, streams are torch streams.
There is no CPU or PyTorch fallback: if ``libvrs.so`` cannot be loaded the
import raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VRS_LIB") or os.path.join(_HERE, "libvrs.so")  # VRS_LIB: tuning variants

VRS_OK, VRS_E_INVALID_ARG, VRS_E_INGEST, VRS_E_CUDA, VRS_E_OOM, VRS_E_CAPACITY, VRS_E_STATE = range(7)
VRS_MAX_VIEWS = 8
VRS_STAGING_THREADS, VRS_STAGING_TMA = 0, 1
VRS_SORT_STOPTHEPOP, VRS_SORT_Z, VRS_SORT_DIST = 0, 1, 2
EXPORTS = ["vrs_abi_version", "vrs_create", "vrs_destroy", "vrs_last_error", "vrs_upload_gaussians",
           "vrs_scene_blob_bytes", "vrs_export_scene", "vrs_import_scene",
           "vrs_set_visibility_mask", "vrs_render_views", "vrs_render_views_host", "vrs_set_instrumentation",
           "vrs_set_resort_mode", "vrs_set_sort_mode", "vrs_set_staging_mode", "vrs_set_output_format", "vrs_backward",
           "vrs_render_views_two_pass", "vrs_get_frame_stats", "vrs_debug_counts", "vrs_debug_pairs", "vrs_debug_ranges", "vrs_debug_splats",
           "vrs_debug_tile_info", "vrs_debug_set_sort_smem_cap", "vrs_sort_pairs", "vrs_exclusive_scan"]


class VrsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"vrs status {status}: {msg}")
        self.status = status


class vrs_config(C.Structure):
    _fields_ = [("device", C.c_int32), ("max_views", C.c_int32), ("max_gaussians", C.c_int64),
                ("max_pairs", C.c_int64), ("max_width", C.c_int32), ("max_height", C.c_int32),
                ("window_k", C.c_int32), ("assign_tile", C.c_int32), ("projection", C.c_int32),
                ("near_plane", C.c_float), ("background", C.c_float * 3)]


class vrs_camera(C.Structure):
    _fields_ = [("R_wc", C.c_float * 9), ("position", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("mask_slot", C.c_int32)]


class vrs_fovea(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("center", C.c_float * 2), ("radius", C.c_float * 2), ("ramp", C.c_float)]


class vrs_frame_stats(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("samples", C.c_int64), ("evaluations", C.c_int64),
                ("contributions", C.c_int64), ("overflow_samples", C.c_int64), ("terminated_samples", C.c_int64),
                ("tiles_by_class", C.c_int32 * 4), ("work_items", C.c_int64), ("visible_splats", C.c_int64),
                ("stage_ms", C.c_float * 8), ("candidates", C.c_int64), ("frustum_gaussians", C.c_int64),
                ("tile_tests", C.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("tiles_by_class", "stage_ms")}
        d["tiles_by_class"] = list(self.tiles_by_class)
        d["stage_ms"] = list(self.stage_ms)
        return d


_lib = None


# element types of (rgba, depth) per output format (VRS_OUT_F32, VRS_OUT_RGBA8_D16F, VRS_OUT_RGBA16F_D32F)
_FMT_NUMPY = {0: (np.float32, np.float32), 1: (np.uint8, np.float16), 2: (np.float16, np.float32)}


def _torch_types(fmt):
    import torch
    return {0: (torch.float32, torch.float32), 1: (torch.uint8, torch.float16), 2: (torch.float16, torch.float32)}[fmt]


def lib():
    """Load libvrs.so (raises if missing: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "vrs_abi_version": (i32, []),
            "vrs_create": (i32, [C.POINTER(vrs_config), C.POINTER(vp)]),
            "vrs_destroy": (None, [vp]),
            "vrs_last_error": (C.c_char_p, [vp]),
            "vrs_upload_gaussians": (i32, [vp, i64, i32, vp, vp, vp, vp, vp, C.POINTER(C.c_int64)]),
            "vrs_scene_blob_bytes": (i64, [i64, i32]),
            "vrs_export_scene": (i32, [vp, vp, i64, C.POINTER(C.c_int64), C.POINTER(C.c_int32), vp]),
            "vrs_import_scene": (i32, [vp, i64, i32, vp, i64, vp]),
            "vrs_set_visibility_mask": (i32, [vp, i32, i32, i32, vp]),
            "vrs_render_views": (i32, [vp, i32, vp, vp, vp, vp, vp]),
            "vrs_render_views_host": (i32, [vp, i32, vp, vp, vp, vp, vp]),
            "vrs_render_views_two_pass": (i32, [vp, i32, vp, vp, vp, vp, vp]),
            "vrs_set_instrumentation": (i32, [vp, i32, i32]),
            "vrs_set_resort_mode": (i32, [vp, i32, i32, i32]),
            "vrs_set_staging_mode": (i32, [vp, i32]),
            "vrs_set_sort_mode": (i32, [vp, i32]),
            "vrs_set_output_format": (i32, [vp, i32]),
            "vrs_backward": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "vrs_get_frame_stats": (i32, [vp, C.POINTER(vrs_frame_stats)]),
            "vrs_debug_counts": (i32, [vp, vp, i64, C.POINTER(C.c_int64)]),
            "vrs_debug_pairs": (i32, [vp, i32, vp, vp, i64, C.POINTER(C.c_int64)]),
            "vrs_debug_ranges": (i32, [vp, vp, i64, C.POINTER(C.c_int64)]),
            "vrs_debug_splats": (i32, [vp, i32, vp, i64]),
            "vrs_debug_tile_info": (i32, [vp, i32, vp, vp, i64]),
            "vrs_debug_set_sort_smem_cap": (i32, [vp, i32]),
            "vrs_sort_pairs": (i32, [vp, vp, vp, i64, i32, vp]),
            "vrs_exclusive_scan": (i32, [vp, vp, vp, vp, i64, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _np_ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def make_camera(cam) -> vrs_camera:
    c = vrs_camera()
    c.R_wc[:] = [float(x) for x in np.asarray(cam.R_wc, np.float32).reshape(9)]
    c.position[:] = [float(x) for x in np.asarray(cam.position, np.float32).reshape(3)]
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height, c.mask_slot = cam.width, cam.height, cam.mask_slot
    return c


def make_fovea(f) -> vrs_fovea:
    v = vrs_fovea()
    if f is not None and f.enabled:
        v.enabled = 1
        v.center[:] = list(f.center)
        v.radius[:] = list(f.radius)
        v.ramp = f.ramp
    return v


class Renderer:
    """One vrs_context (one device).  Thin object wrapper over the C ABI."""

    def __init__(self, max_gaussians, max_views=2, max_pairs=1 << 22, max_width=2064, max_height=2208,
                 assign_tile=16, device=0, near_plane=0.2, background=(0.0, 0.0, 0.0), window_k=16, projection=0):
        L = lib()
        cfg = vrs_config()
        cfg.device, cfg.max_views, cfg.max_gaussians, cfg.max_pairs = device, max_views, max_gaussians, max_pairs
        cfg.max_width, cfg.max_height, cfg.window_k, cfg.assign_tile = max_width, max_height, window_k, assign_tile
        cfg.projection, cfg.near_plane = projection, near_plane
        cfg.background[:] = list(background)
        h = C.c_void_p()
        st = L.vrs_create(C.byref(cfg), C.byref(h))
        if st != VRS_OK:
            raise VrsError(st, "vrs_create failed")
        self.h = h
        self.cfg = cfg
        self.device = device
        self.n = 0
        self._views = None

    def close(self):
        if getattr(self, "h", None):
            lib().vrs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != VRS_OK:
            msg = lib().vrs_last_error(self.h)
            raise VrsError(st, msg.decode() if msg else "")

    # ---- C ABI wrappers
    def vrs_upload_gaussians(self, scene):
        arrs = [np.ascontiguousarray(a, np.float32) for a in
                (scene.means, scene.quats, scene.log_scales, scene.logits, scene.sh)]
        rej = C.c_int64(0)
        self._check(lib().vrs_upload_gaussians(self.h, scene.n, scene.sh_degree, *[_np_ptr(a) for a in arrs],
                                               C.byref(rej)))
        self.n = scene.n - rej.value
        self.sh_degree = scene.sh_degree
        return rej.value

    upload = vrs_upload_gaussians

    def _stream_ptr(self, stream):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    def vrs_export_scene(self, stream=None):
        """The activated scene as one DEVICE blob (uint8 tensor on this renderer's device),
        enqueued on `stream` (default: torch's current stream).  Returns (blob, n, sh_degree)."""
        import torch
        n, deg = self.n, self.sh_degree
        nbytes = lib().vrs_scene_blob_bytes(n, deg)
        blob = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", self.device))
        n_out, d_out = C.c_int64(0), C.c_int32(0)
        self._check(lib().vrs_export_scene(self.h, C.c_void_p(blob.data_ptr()), nbytes, C.byref(n_out),
                                           C.byref(d_out), C.c_void_p(self._stream_ptr(stream))))
        return blob, n_out.value, d_out.value

    def vrs_import_scene(self, n, sh_degree, blob, stream=None):
        """Adopt a scene blob exported by another renderer (DEVICE uint8 tensor on this device)."""
        if not blob.is_cuda or blob.device.index != self.device or blob.dtype.itemsize != 1:
            raise ValueError(f"blob must be a byte tensor on cuda:{self.device}")
        self._check(lib().vrs_import_scene(self.h, int(n), int(sh_degree), C.c_void_p(blob.data_ptr()), blob.numel(),
                                           C.c_void_p(self._stream_ptr(stream))))
        self.n, self.sh_degree = int(n), int(sh_degree)

    def vrs_set_visibility_mask(self, slot, mask):
        if mask is None:
            self._check(lib().vrs_set_visibility_mask(self.h, slot, 0, 0, None))
        else:
            m = np.ascontiguousarray(mask, np.uint8)
            self._check(lib().vrs_set_visibility_mask(self.h, slot, m.shape[1], m.shape[0], _np_ptr(m)))

    set_mask = vrs_set_visibility_mask

    def vrs_backward(self, rgba, depth, grad_rgba, grad_depth, stream=None):
        """N4: gradients of L = sum grad_rgba . RGBA + grad_depth . Depth of the last (non-foveated)
        frame w.r.t. the uploaded raw parameters.  All tensors on the device; returns a dict of
        float32 device tensors means (n,3), quats (n,4), log_scales (n,3), logits (n,), sh (n,k,3)."""
        import torch
        dev = torch.device("cuda", self.device)
        n, k = self.n, (self.sh_degree + 1) ** 2
        out = {"means": torch.empty((n, 3), device=dev), "quats": torch.empty((n, 4), device=dev),
               "log_scales": torch.empty((n, 3), device=dev), "logits": torch.empty((max(n, 1),), device=dev)[:n],
               "sh": torch.empty((n, k, 3), device=dev)}
        for t in (rgba, depth, grad_rgba, grad_depth):
            if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                raise ValueError("backward tensors must be contiguous float32 CUDA tensors")
            if t.device.index != self.device:
                raise ValueError(f"backward tensors must live on cuda:{self.device}, got {t.device}")
        if self._views is not None:  # (after a two-pass frame the C ABI rejects the call itself)
            px = sum(c.width * c.height for c in self._views)
            self._check_buffers(px, rgba, depth, fmt=0)
            self._check_buffers(px, grad_rgba, grad_depth, fmt=0)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._check(lib().vrs_backward(self.h, *[C.c_void_p(t.data_ptr()) for t in (rgba, depth, grad_rgba, grad_depth)],
                                       *[C.c_void_p(out[f].data_ptr()) for f in ("means", "quats", "log_scales",
                                                                                  "logits", "sh")],
                                       C.c_void_p(sp)))
        return out

    def vrs_set_output_format(self, fmt):
        """VRS_OUT_F32 (0): float RGBA + float depth; VRS_OUT_RGBA8_D16F (1): uint8 RGBA + binary16
        depth; VRS_OUT_RGBA16F_D32F (2): binary16 RGBA + float depth."""
        self._check(lib().vrs_set_output_format(self.h, int(fmt)))
        self.out_fmt = int(fmt)

    def vrs_set_resort_mode(self, mode, block_queue=0, pixel_window=0):
        """0 = per-sample window K = 16; 1 = hierarchical (K_B = 8 block queue, K_P = 8 window)."""
        self._check(lib().vrs_set_resort_mode(self.h, int(mode), int(block_queue), int(pixel_window)))

    def vrs_set_sort_mode(self, mode):
        """VRS_SORT_STOPTHEPOP (0, default), VRS_SORT_Z (1) or VRS_SORT_DIST (2): the N3 global-sort baselines."""
        self._check(lib().vrs_set_sort_mode(self.h, int(mode)))

    def vrs_set_staging_mode(self, mode):
        """VRS_STAGING_THREADS (0, default): thread loads; VRS_STAGING_TMA (1): TMA bulk copies."""
        self._check(lib().vrs_set_staging_mode(self.h, int(mode)))

    def vrs_set_instrumentation(self, counters=0, timing=0, no_cull=0):
        self._check(lib().vrs_set_instrumentation(self.h, int(counters) | (int(no_cull) << 8), int(timing)))

    def _check_buffers(self, px, rgba, depth, fmt=None, host=False):
        """Validate caller buffers before they reach the C ABI: element counts for px
        pixels, dtypes of the output format, contiguity, and (device buffers) the
        context's device -- a mismatched buffer raises here instead of becoming an
        out-of-bounds device access."""
        import torch
        fmt = getattr(self, "out_fmt", 0) if fmt is None else fmt
        want_r, want_d = _torch_types(fmt)
        np_r, np_d = _FMT_NUMPY[fmt]
        for t, n, wt, wn, name in ((rgba, 4 * px, want_r, np_r, "rgba"), (depth, px, want_d, np_d, "depth")):
            if isinstance(t, np.ndarray):
                if not host:
                    raise ValueError(f"{name}: a device tensor is required")
                if t.dtype != wn or t.size != n or not t.flags["C_CONTIGUOUS"]:
                    raise ValueError(f"{name}: need {n} contiguous {np.dtype(wn).name}, got {t.size} {t.dtype}")
                continue
            if t.dtype != wt or t.numel() != n or not t.is_contiguous():
                raise ValueError(f"{name}: need {n} contiguous {wt}, got {t.numel()} {t.dtype}")
            if host:
                if t.is_cuda:
                    raise ValueError(f"{name}: a host buffer is required")
            elif not t.is_cuda or t.device.index != self.device:
                raise ValueError(f"{name}: must live on cuda:{self.device}, got {t.device}")

    def _views_structs(self, cams, foveas):
        carr = (vrs_camera * len(cams))(*[make_camera(c) for c in cams])
        farr = None
        if foveas is not None:
            farr = (vrs_fovea * len(cams))(*[make_fovea(f) for f in foveas])
        return carr, farr

    def alloc_outputs(self, cams, pinned_host=False):
        """Output tensors for the context's format: (px, 4) float32 + (px,) float32, (px, 4)
        uint8 + (px,) float16 for VRS_OUT_RGBA8_D16F, (px, 4) float16 + (px,) float32 for
        VRS_OUT_RGBA16F_D32F; on the device, or pinned host."""
        import torch
        px = sum(c.width * c.height for c in cams)
        rt, dt = _torch_types(getattr(self, "out_fmt", 0))
        if pinned_host:
            return (torch.empty((px, 4), dtype=rt).pin_memory(), torch.empty(px, dtype=dt).pin_memory())
        dev = torch.device("cuda", self.device)
        return torch.empty((px, 4), dtype=rt, device=dev), torch.empty(px, dtype=dt, device=dev)

    def vrs_render_views(self, cams, foveas=None, rgba=None, depth=None, stream=None):
        """Render into DEVICE torch tensors (allocated if None) on `stream`
        (default: torch's current stream).  Returns (rgba, depth) flat tensors."""
        import torch
        if rgba is None or depth is None:
            rgba, depth = self.alloc_outputs(cams)
        self._check_buffers(sum(c.width * c.height for c in cams), rgba, depth)
        carr, farr = self._views_structs(cams, foveas)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._check(lib().vrs_render_views(self.h, len(cams), C.cast(carr, C.c_void_p),
                                           C.cast(farr, C.c_void_p) if farr is not None else None,
                                           C.c_void_p(rgba.data_ptr()), C.c_void_p(depth.data_ptr()),
                                           C.c_void_p(sp)))
        self._views = list(cams)
        return rgba, depth

    render = vrs_render_views

    def vrs_render_views_two_pass(self, cams, foveas, rgba=None, depth=None, stream=None):
        """Two-pass foveated baseline (App. A) into DEVICE tensors; same output layout as render()."""
        import torch
        if rgba is None or depth is None:
            rgba, depth = self.alloc_outputs(cams)
        self._check_buffers(sum(c.width * c.height for c in cams), rgba, depth)
        carr, farr = self._views_structs(cams, foveas)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._check(lib().vrs_render_views_two_pass(self.h, len(cams), C.cast(carr, C.c_void_p),
                                                    C.cast(farr, C.c_void_p) if farr is not None else None,
                                                    C.c_void_p(rgba.data_ptr()), C.c_void_p(depth.data_ptr()),
                                                    C.c_void_p(sp)))
        self._views = None  # the last frame holds the 2n pass views
        return rgba, depth

    render_two_pass = vrs_render_views_two_pass

    def vrs_render_views_host(self, cams, foveas=None, rgba_host=None, depth_host=None, stream=None):
        """End-to-end path: outputs land in HOST buffers (numpy or pinned torch tensors)."""
        px = sum(c.width * c.height for c in cams)
        if rgba_host is None:
            nr, nd = _FMT_NUMPY[getattr(self, "out_fmt", 0)]
            rgba_host = np.empty((px, 4), nr)
            depth_host = np.empty(px, nd)
        self._check_buffers(px, rgba_host, depth_host, host=True)
        rp = rgba_host.data_ptr() if hasattr(rgba_host, "data_ptr") else rgba_host.ctypes.data
        dp = depth_host.data_ptr() if hasattr(depth_host, "data_ptr") else depth_host.ctypes.data
        carr, farr = self._views_structs(cams, foveas)
        sp = 0
        if stream is not None:
            sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._check(lib().vrs_render_views_host(self.h, len(cams), C.cast(carr, C.c_void_p),
                                                C.cast(farr, C.c_void_p) if farr is not None else None,
                                                C.c_void_p(rp), C.c_void_p(dp), C.c_void_p(sp)))
        self._views = list(cams)
        return rgba_host, depth_host

    render_host = vrs_render_views_host

    def vrs_get_frame_stats(self):
        s = vrs_frame_stats()
        self._check(lib().vrs_get_frame_stats(self.h, C.byref(s)))
        return s.as_dict()

    stats = vrs_get_frame_stats

    # ---- parity hooks
    def vrs_debug_counts(self):
        n = C.c_int64(0)
        cap = VRS_MAX_VIEWS * max(self.n, 1)
        out = np.zeros(cap, np.uint32)
        self._check(lib().vrs_debug_counts(self.h, _np_ptr(out), cap, C.byref(n)))
        return out[:n.value]

    def vrs_debug_pairs(self, sorted_=True):
        s = self.vrs_get_frame_stats()
        cap = max(int(s["pairs"]), 1)
        k, v = np.zeros(cap, np.uint64), np.zeros(cap, np.uint32)
        n = C.c_int64(0)
        self._check(lib().vrs_debug_pairs(self.h, 1 if sorted_ else 0, _np_ptr(k), _np_ptr(v), cap, C.byref(n)))
        return k[:n.value], v[:n.value]

    def vrs_debug_ranges(self):
        cap = 2 * (1 << 20)
        out = np.zeros(cap, np.uint32)
        n = C.c_int64(0)
        self._check(lib().vrs_debug_ranges(self.h, _np_ptr(out), cap, C.byref(n)))
        return out[:2 * n.value].reshape(-1, 2)

    def vrs_debug_splats(self, view):
        out = np.zeros((max(self.n, 1), 48), np.float32)
        self._check(lib().vrs_debug_splats(self.h, view, _np_ptr(out), out.size))
        return out[:self.n]

    def vrs_debug_tile_info(self, view, tile):
        c = self._views[view]
        tw, th = (c.width + tile - 1) // tile, (c.height + tile - 1) // tile
        cls, vis = np.zeros(tw * th, np.int32), np.zeros(tw * th, np.int32)
        self._check(lib().vrs_debug_tile_info(self.h, view, _np_ptr(cls), _np_ptr(vis), tw * th))
        return cls.reshape(th, tw), vis.reshape(th, tw)

    def vrs_debug_set_sort_smem_cap(self, cap):
        self._check(lib().vrs_debug_set_sort_smem_cap(self.h, int(cap)))

    # ---- primitives
    def vrs_sort_pairs(self, keys, vals, key_bits=64, stream=None):
        """In-place stable radix sort of DEVICE torch tensors (int64 keys viewed as u64, int32 vals)."""
        import torch
        stream = stream or torch.cuda.current_stream(self.device)
        self._check(lib().vrs_sort_pairs(self.h, C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()),
                                         keys.numel(), key_bits, C.c_void_p(stream.cuda_stream)))

    def vrs_exclusive_scan(self, inp, out, total, stream=None):
        import torch
        stream = stream or torch.cuda.current_stream(self.device)
        self._check(lib().vrs_exclusive_scan(self.h, C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr()),
                                             C.c_void_p(total.data_ptr()), inp.numel(),
                                             C.c_void_p(stream.cuda_stream)))


def split_views(flat_rgba, flat_depth, cams):
    """Split flat (views concatenated) outputs into per-view (H, W, 4) / (H, W)."""
    outs, off = [], 0
    for c in cams:
        k = c.width * c.height
        outs.append((flat_rgba[off:off + k].reshape(c.height, c.width, 4), flat_depth[off:off + k].reshape(c.height, c.width)))
        off += k
    return outs
