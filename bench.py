#!/usr/bin/env python
"""bench.py — stereo frames/s of the VRSplat render path on B200.

Default workload (BASELINE.json metric, config C2): 500k-Gaussian "vr_room"
scene (SH degree 3), stereo 2 x 2064 x 2208 at 110 deg FoV, single-pass
foveated (fovea = half the image, 10% ramp), synthetic ellipse visibility
masks, one sort and one blend launch per stereo frame.  One step = one full
stereo frame through every stage (preprocess, scan, duplicate, onesweep
sort, ranges, blend, compose).

Timing: W untimed warm-up frames; then K frames, each bracketed by CUDA
events on the render stream, with an L2 flush (a 256 MB write) between frames
outside the events; barrier + synchronize around the timed region; the
max over ranks is reported.  N > 1 (torchrun): rank 0 builds the scene and
NCCL-broadcasts the raw arrays (the only data-path collective); every rank
renders its own stereo frames (weak scaling over views).

``--impl reference`` times the C++ oracle (the only reference this paper
has: no code was published) on the box's host cores on a bounded sample of
the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import math
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# frames in flight on the end-to-end path (device/pinned output buffers rotating between render and D2H)
E2E_DEPTH = int(os.environ.get("VRS_E2E_DEPTH", "2"))
sys.path.insert(0, ROOT)

import scenegen as sg  # noqa: E402

CONFIGS = {
    # name: (n_gaussians, scale_mul, sh_degree, foveated, assign_tile, masks)
    "c2": dict(n=500_000, scale_mul=1.0, sh=3, fovea=True, T=32, masks=True, seed=2,
               desc="500k vr_room SH3, stereo 2x2064x2208, 110deg, single-pass foveated, ellipse masks"),
    "c3": dict(n=3_000_000, scale_mul=(1 / 6) ** 0.5, sh=3, fovea=False, T=16, masks=False, seed=3,
               desc="3M vr_room SH3 (scales x0.408), stereo 2x2064x2208, 110deg, no foveation"),
    "c1": dict(n=1000, scale_mul=None, sh=0, fovea=False, T=16, masks=False, seed=0,
               desc="1000 random Gaussians SH0, one 128x128 view, 90deg, 16x16 tiles"),
    "c4": dict(n=1_000_000, scale_mul=0.707, sh=3, fovea=True, T=32, masks=True, seed=4, trajectory=True,
               desc="1M vr_room SH3 (scales x0.707), 360-pose head trajectory = 720 views, stereo pairs "
                    "sharded by rank, foveated"),
    "c5": dict(n=500_000, scale_mul=1.0, sh=3, fovea=True, T=32, masks=False, seed=2,
               desc="C2 scene, FoV sweep 90-160 deg, Optimal Projection vs EWA baseline"),
    "c7": dict(n=500_000, scale_mul=1.0, sh=3, fovea=False, T=16, masks=False, seed=2,
               desc="large-FOV protocol (App. D) on the C2 scene: per eye, crop [W,2W)x[H,2H) of the 3W x 3H "
                    "render at the same pixel focal length vs the W x H render, Optimal Projection vs EWA"),
    "c8": dict(n=500_000, scale_mul=1.0, sh=3, fovea=True, T=32, masks=True, seed=2, resort=1,
               desc="C2 workload with the hierarchical resort mode (SURVEY N2): K_B = 8 queue per 4x4 sample "
                    "block, K_G = 4 queue per 2x2 group, K_P = 8 per-sample window; vs_flat compares with the "
                    "K = 16 frame"),
    "c9": dict(n=500_000, scale_mul=1.0, sh=3, fovea=False, T=16, masks=False, seed=2,
               desc="training step (SURVEY N4): C2 scene, stereo 2x2064x2208 non-foveated (T_a = 16), forward "
                    "render + vrs_backward of synthetic gradient images to all raw parameters"),
    "c10": dict(n=500_000, scale_mul=1.0, sh=3, fovea=True, T=32, masks=True, seed=2,
                desc="C2 workload with the paper's global-sort baselines (SURVEY N3, P:456): Mini-Splatting (z) "
                     "and (Dist) orders blended in list order, vs OP + StopThePop; pairs and blend ms per order"),
    "c6": dict(n=500_000, scale_mul=1.0, sh=3, fovea=True, T=32, masks=True, seed=2, two_pass=True,
               desc="C2 workload rendered with the paper's two-pass foveated baseline (App. A): full-res "
                    "centre crop + half-res masked periphery, bilinear upsample + blend (SURVEY N1)"),
}
METRIC = "stereo frames/sec (2x2064x2208, foveated) at 500k Gaussians; ms/stage"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="vrs", choices=["vrs", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--projection", type=int, default=0, help="0 = Optimal Projection, 1 = EWA baseline")
    ap.add_argument("--staging", default="threads", choices=["threads", "tma"],
                    help="blend record staging: block threads (default) or the TMA bulk-copy engine")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--quiet", action="store_true")
    return ap.parse_args()


def step_cams(cfg_name, cams, step, rank=0, world=1):
    """Cameras of timed step ``step``: fixed for C1/C2/C3; for C4 the rank's
    contiguous shard of the 360-pose trajectory (a stereo pair never split),
    visited cyclically."""
    if not CONFIGS[cfg_name].get("trajectory"):
        return cams
    from paper_2505_10144_b200.parallel import shard_range
    a, b = shard_range(360, world, rank)
    t = a + (step % max(1, b - a))
    head, yaw, pitch, roll = sg.trajectory_pose(t)
    return sg.stereo_pair(head, yaw, pitch, roll, masks=True)


def make_workload(cfg_name):
    c = CONFIGS[cfg_name]
    if cfg_name == "c1":
        scene = sg.random_scene(c["seed"], n=c["n"], sh_degree=0)
        cams = [sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)]
        return scene, cams, None, {}
    scene = sg.vr_room(c["seed"], c["n"], scale_mul=c["scale_mul"], sh_degree=c["sh"])
    cams = sg.stereo_pair(masks=c["masks"])
    fov = [sg.quest_fovea()] * 2 if c["fovea"] else None
    masks = {0: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H), 1: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H)} if c["masks"] else {}
    return scene, cams, fov, masks


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    HW_SLOWDOWN, SW_THERMAL, HW_THERMAL, SW_POWER = 0x8, 0x20, 0x40, 0x4

    def __init__(self, index=0, period=0.005):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = {self.HW_SLOWDOWN: "hw_slowdown", self.HW_THERMAL: "hw_thermal_slowdown",
                 self.SW_THERMAL: "sw_thermal_slowdown", self.SW_POWER: "sw_power_cap"}
        reasons = sorted({n for _, r in self.rows for bit, n in names.items() if r & bit})
        return {"sm_mhz": statistics.median([r[0] for r in self.rows]), "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 5 ms period"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def stage_roofline(counters, stage_ms, n, n_views, peaks):
    """HBM roofline of the memory-side stages (SURVEY §8d "Roofline per stage"):
    algorithmic bytes per unit x the frame's units, over the stage's event time,
    against the measured copy bandwidth and the nominal 8 TB/s.  Units: N
    Gaussians, G1 Gaussians in >= 1 view's frustum cone, V visible (view,
    Gaussian), P pairs.  preprocess = 16 B/Gaussian (mu + q_cut) + 244 B per G1
    (Sigma_w, Sigma_w^-1, sigma, SH3) + 112 B record per V + 4 B count per
    (view, Gaussian); duplicate = 64 B read per V + 12 B written per pair; sort
    (+ ranges) = 24 B per pair (one read + one write of key and value) + 8 B per
    pair and per tile for the ranges."""
    hbm = float(peaks.get("hbm_gbs", 6549.0))
    N, G1 = float(n), float(counters.get("frustum_gaussians", 0))
    V, P = float(counters.get("visible_splats", 0)), float(counters.get("pairs", 0))
    tiles = float(sum(counters.get("tiles_by_class", [0, 0, 0, 0])))
    rows = {
        "preprocess": (16 * N + 244 * G1 + 112 * V + 4 * N * n_views, stage_ms[0] + stage_ms[1],
                       "k_cull + k_preprocess (k_color on the side stream)"),
        "duplicate": (64 * V + 12 * P, stage_ms[2], "k_tiletest_direct"),
        "sort": (24 * P + 8 * P + 8 * tiles, stage_ms[3] + stage_ms[4], "k_tile_scan + k_ovf_bucket + k_tile_sort"),
    }
    out = {}
    for k, (b, ms, kern) in rows.items():
        gbs = b / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        out[k] = {"kernels": kern, "bound": "hbm", "algorithmic_bytes": b, "ms": ms, "achieved_gbs": gbs,
                  "frac": gbs / hbm, "frac_8tbs": gbs / 8000.0}
    out["units"] = {"N": N, "G1": G1, "V": V, "P": P, "candidates": counters.get("candidates"),
                    "tile_tests": counters.get("tile_tests")}
    out["peak_gbs"] = hbm
    return out


def cpu_baseline(scene, cams, fov, masks, T, budget_s=15.0, threads=0):
    """The oracle as it stands on the host cores, on a bounded sample:
    full per-Gaussian stage + instantiation + sort + ranges for both eyes, then
    a random sample of output pixels; frames/s extrapolated to the full frame.
    threads = 0: all cores."""
    import oracle
    ncores = threads or os.cpu_count() or 1
    o = oracle.Oracle(scene)
    for k, m in masks.items():
        o.set_mask(k, m)
    t0 = time.perf_counter()
    o.prepare(cams, fov, assign_tile=T, threads=ncores)
    t_prep = time.perf_counter() - t0
    total_px = sum(c.width * c.height for c in cams)
    rs = np.random.default_rng(123)
    n = 512
    t_pix, done = 0.0, 0
    while (done == 0 or t_prep + t_pix < budget_s) and done < total_px:
        n = min(n, total_px - done)
        vxy = np.stack([rs.integers(0, len(cams), n), rs.integers(0, cams[0].width, n),
                        rs.integers(0, cams[0].height, n)], 1)
        t0 = time.perf_counter()
        o.render_pixels(vxy)
        t_pix += time.perf_counter() - t0
        done += n
        n = min(n * 2, 65536)
    frame_s = t_prep + t_pix * (total_px / done)
    return {"value": 1.0 / frame_s, "unit": "stereo frames/s" if len(cams) == 2 else "frames/s", "cores": ncores,
            "kind": "oracle", "prep_s": t_prep, "cpu_model": cpu_model(),
            "sample": f"full preprocess+pairs+sort+ranges of the frame ({t_prep:.2f}s) + {done} random output "
                      f"pixels ({t_pix:.2f}s) of {total_px}, extrapolated per pixel"}


def run_reference(args):
    """The oracle (the paper published no code) on the host cores.  Each step is a
    bounded sample of the workload -- the whole per-Gaussian / pairs / sort /
    ranges pass of the frame plus a random sample of output pixels -- sized so
    the K + W steps end within ~2.5 minutes; ms_per_step is the measured time of
    one such step, value the stereo frames/s extrapolated per pixel."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    scene, cams, fov, masks = make_workload(args.config)
    n_runs = max(1, args.steps + args.warmup)
    t_prep = cpu_baseline(scene, cams, fov, masks, cfg["T"], budget_s=0.0)["prep_s"]
    budget = max(0.3, 150.0 / n_runs - t_prep) + t_prep
    vals, step_s = [], []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = cpu_baseline(scene, cams, fov, masks, cfg["T"], budget_s=budget)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            vals.append(r)
            step_s.append(dt)
    v = statistics.median([r["value"] for r in vals])
    line = {"metric": METRIC if args.config == "c2" else METRIC + f" [{args.config}]", "value": v,
            "unit": vals[0]["unit"], "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * float(np.mean(step_s)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": workload_config(args.config, scene, cams),
            "reference_step": "a bounded sample of the frame (see cpu_baseline.sample); value = full stereo "
                              "frames/s extrapolated per pixel, ms_per_step = measured time of one sampled step",
            "cpu_baseline": {"value": v, "unit": vals[0]["unit"], "cores": vals[0]["cores"], "kind": "oracle",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": vals[0]["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(name, scene, cams, world=1, extra=None):
    """The bench line's config object (the same for both arms)."""
    cfg = CONFIGS[name]
    out = {"workload": name, "desc": cfg["desc"], "gaussians": int(scene if isinstance(scene, int) else scene.n),
           "views": len(cams),
           "resolution": [cams[0].width, cams[0].height], "assign_tile": cfg["T"],
           "foveated": bool(cfg["fovea"]), "parallelism": f"views x{world} (replicated scene, weak)"}
    out.update(extra or {})
    return out


def run_c7(args):
    """Config C7: large-FOV protocol on the CUDA
    path.  Both eyes of the C2 stereo pair are rendered at W x H and at 3W x 3H
    with the same pixel focal length; the centre crop of the wide render casts
    the original rays pixel for pixel, so a projection without error reproduces
    the normal render exactly.  Reports crop-vs-normal PSNR (RGB) and max |diff|
    per projection, and the wide-render time."""
    import torch
    from paper_2505_10144_b200 import Renderer
    from paper_2505_10144_b200.protocol import centre_crop, psnr, wide_camera
    from paper_2505_10144_b200.vrs import split_views
    cfg = CONFIGS["c7"]
    scene = sg.vr_room(cfg["seed"], cfg["n"], sh_degree=cfg["sh"])
    cams = sg.stereo_pair(masks=False)
    wides = [wide_camera(c) for c in cams]
    rows = []
    stream = torch.cuda.Stream()
    for proj in (0, 1):
        r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=48 << 20, max_width=wides[0].width,
                     max_height=wides[0].height, assign_tile=cfg["T"], projection=proj)
        r.upload(scene)
        with torch.cuda.stream(stream):
            a = r.render(cams, None, stream=stream)
            normal = split_views(a[0].cpu().numpy(), a[1].cpu().numpy(), cams)
            r.vrs_set_instrumentation(counters=0, timing=1)
            rw, dw = r.alloc_outputs(wides)
            for _ in range(max(args.warmup, 1)):
                r.render(wides, None, rw, dw, stream=stream)
            ms = []
            for _ in range(max(args.steps // 4, 2)):
                r.render(wides, None, rw, dw, stream=stream)
                ms.append(r.stats()["stage_ms"][7])
            wide = split_views(rw.cpu().numpy(), dw.cpu().numpy(), wides)
        st = r.stats()
        for e in range(2):
            crop = centre_crop(wide[e][0], cams[e])
            nrm = normal[e][0]
            p = psnr(crop[..., :3], nrm[..., :3])
            rows.append({"projection": "OP" if proj == 0 else "EWA", "eye": e,
                         "crop_psnr_db": None if math.isinf(p) else p, "identical": bool(math.isinf(p)),
                         "max_abs_rgb_diff": float(np.abs(crop[..., :3] - nrm[..., :3]).max()),
                         "wide_pairs_per_eye": st["pairs"] / 2, "wide_stereo_ms": float(np.median(ms))})
        r.close()
        del rw, dw
        torch.cuda.empty_cache()
    ewa = [x["crop_psnr_db"] for x in rows if x["projection"] == "EWA"]
    ewa_v = float(np.mean([x for x in ewa if x is not None])) if any(x is not None for x in ewa) else None
    line = {"metric": "C7 large-FOV protocol: crop-vs-normal PSNR (dB) of the EWA baseline (OP: identical)",
            "value": ewa_v, "unit": "dB", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c7", "desc": cfg["desc"], "gaussians": scene.n, "normal": [cams[0].width,
                       cams[0].height], "wide": [wides[0].width, wides[0].height], "assign_tile": cfg["T"]},
            "rows": rows}
    print(json.dumps(line), flush=True)


def run_c9(args):
    """Config C9: one training step = forward render of a
    non-foveated stereo frame + vrs_backward of fixed synthetic gradient
    images (a stand-in loss; the paper's datasets are out of scope), timed
    with CUDA events on the stream; per-part times reported."""
    import torch
    from paper_2505_10144_b200 import Renderer
    cfg = CONFIGS["c9"]
    scene = sg.vr_room(cfg["seed"], cfg["n"], scale_mul=cfg["scale_mul"], sh_degree=cfg["sh"])
    cams = sg.stereo_pair(masks=False)
    r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=16 << 20, max_width=cams[0].width,
                 max_height=cams[0].height, assign_tile=cfg["T"])
    r.upload(scene)
    stream = torch.cuda.Stream()
    rgba, depth = r.alloc_outputs(cams)
    gen = torch.Generator(device="cuda").manual_seed(0)
    g_rgba = torch.randn(rgba.shape, device="cuda", generator=gen)
    g_depth = torch.randn(depth.shape, device="cuda", generator=gen) * 0.1
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        r.render(cams, None, rgba, depth, stream=stream)
        mid.record(stream)
        return r.vrs_backward(rgba, depth, g_rgba, g_depth, stream=stream)

    mid = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    fw, bw, tot = [], [], []
    with ClockSampler(0) as clk:
        for s_ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            mid = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                flush.fill_(s_ & 0xff)
                e0.record(stream)
                out = step()
                e1.record(stream)
            torch.cuda.synchronize()
            fw.append(e0.elapsed_time(mid))
            bw.append(mid.elapsed_time(e1))
            tot.append(e0.elapsed_time(e1))
    ms = float(np.mean(tot))
    line = {"metric": "training steps/s (forward + backward, stereo 2x2064x2208 non-foveated) [c9]",
            "value": 1000.0 / ms, "unit": "steps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": "c9", "desc": cfg["desc"], "gaussians": scene.n,
                                            "l2": "flushed between steps (outside the event pair)"},
            "stage_ms": {"forward": float(np.mean(fw)), "backward": float(np.mean(bw))},
            "grad_abs_max": {k: float(v.abs().max()) for k, v in out.items()},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_c5(args):
    """Config C5: FoV sweep 90-160 deg on the C2 scene, Optimal Projection vs the
    EWA baseline: pairs per eye, blend ms and frame ms per FoV (one GPU)."""
    import torch
    from paper_2505_10144_b200 import Renderer
    cfg = CONFIGS["c5"]
    scene = sg.vr_room(cfg["seed"], cfg["n"], sh_degree=cfg["sh"])
    fov = [sg.quest_fovea()] * 2
    rows = []
    stream = torch.cuda.Stream()
    for proj in (0, 1):
        r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=24 << 20, max_width=sg.QUEST_W,
                     max_height=sg.QUEST_H, assign_tile=32, projection=proj)
        r.upload(scene)
        rgba, depth = r.alloc_outputs(sg.stereo_pair(masks=False))
        for hfov in range(90, 161, 10):
            cams = sg.stereo_pair(hfov_deg=float(hfov), masks=False)
            r.vrs_set_instrumentation(counters=1, timing=0)
            r.render(cams, fov, rgba, depth, stream=stream)
            st = r.stats()
            r.vrs_set_instrumentation(counters=0, timing=1)
            for _ in range(args.warmup):
                r.render(cams, fov, rgba, depth, stream=stream)
            ms, blend = [], []
            for _ in range(args.steps):
                r.render(cams, fov, rgba, depth, stream=stream)
                t = r.stats()["stage_ms"]
                ms.append(t[7])
                blend.append(t[5])
            rows.append({"projection": "OP" if proj == 0 else "EWA", "hfov": hfov,
                         "pairs_per_eye": st["pairs"] / 2, "contributions": st["contributions"],
                         "frame_ms": float(np.median(ms)), "blend_ms": float(np.median(blend))})
        r.close()
    op110 = [x for x in rows if x["projection"] == "OP" and x["hfov"] == 110][0]
    line = {"metric": "C5 FoV sweep (OP vs EWA): stereo frames/s at 110 deg OP; pairs/eye and blend ms per FoV",
            "value": 1000.0 / op110["frame_ms"], "unit": "stereo frames/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": op110["frame_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c5", "desc": cfg["desc"]}, "sweep": rows}
    print(json.dumps(line), flush=True)


def run_c10(args):
    """Config C10: the C2 frame rendered with the
    paper's global-sort baselines -- Mini-Splatting (z) and (Dist): one depth per
    Gaussian, tile lists blended in list order, no per-pixel resort -- next to the
    method (OP + StopThePop K = 16): pairs per eye, contributions, blend and frame
    ms, and the PSNR of each baseline frame against the method's frame."""
    import torch
    from paper_2505_10144_b200 import Renderer
    cfg = CONFIGS["c10"]
    scene, cams, fov, masks = make_workload("c10")
    r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=8 << 20, max_width=sg.QUEST_W,
                 max_height=sg.QUEST_H, assign_tile=32)
    r.upload(scene)
    for k, m in masks.items():
        r.set_mask(k, m)
    stream = torch.cuda.Stream()
    rgba, depth = r.alloc_outputs(cams)
    rows, frames = [], {}
    for mode, name in ((0, "OP + StopThePop (K = 16)"), (1, "Mini-Splatting (z)"), (2, "Mini-Splatting (Dist)")):
        r.vrs_set_sort_mode(mode)
        r.vrs_set_instrumentation(counters=1, timing=0)
        r.render(cams, fov, rgba, depth, stream=stream)
        st = r.stats()
        frames[mode] = rgba.clone()
        r.vrs_set_instrumentation(counters=0, timing=1)
        for _ in range(args.warmup):
            r.render(cams, fov, rgba, depth, stream=stream)
        ms, blend = [], []
        for _ in range(args.steps):
            r.render(cams, fov, rgba, depth, stream=stream)
            t = r.stats()["stage_ms"]
            ms.append(t[7])
            blend.append(t[5])
        row = {"order": name, "sort_mode": mode, "pairs_per_eye": st["pairs"] / 2,
               "contributions": st["contributions"], "evaluations": st["evaluations"],
               "frame_ms": float(np.median(ms)), "blend_ms": float(np.median(blend))}
        if mode:
            d = (frames[mode][:, :3] - frames[0][:, :3]).double()
            mse = float((d * d).mean())
            row["psnr_vs_method_db"] = 10.0 * math.log10(1.0 / mse) if mse > 0 else None
        rows.append(row)
    r.close()
    line = {"metric": "C10 global-sort baselines (N3): stereo frames/s of Mini-Splatting (z) order at C2",
            "value": 1000.0 / rows[1]["frame_ms"], "unit": "stereo frames/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rows[1]["frame_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config("c10", scene, cams), "orders": rows}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5":
        return run_c5(args)
    if args.config == "c7":
        return run_c7(args)
    if args.config == "c9":
        return run_c9(args)
    if args.config == "c10":
        return run_c10(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: VRS_BENCH_ONE_GPU=1 runs every rank on cuda:0 over gloo (checks the multi-rank
    # logic on a one-GPU box; NCCL refuses two ranks on one device)
    one_gpu = os.environ.get("VRS_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]

    # ---- scene: rank 0 generates and uploads (host activation once); with N > 1 the activated
    # device buffers go to every rank as one blob by NCCL broadcast (the only data-path collective)
    scene = None
    if rank == 0:
        scene, cams, fov, masks = make_workload(args.config)
    else:
        cams, fov, masks = make_cams_only(args.config)
    from paper_2505_10144_b200 import Renderer

    W = max(c.width for c in cams)
    H = max(c.height for c in cams)
    two_pass = bool(cfg.get("two_pass"))
    r = Renderer(max_gaussians=cfg["n"], max_views=len(cams) * (2 if two_pass else 1),
                 max_pairs=16 << 20 if cfg["n"] > 1e6 or two_pass else 8 << 20,
                 max_width=W, max_height=H, assign_tile=cfg["T"], device=local, projection=args.projection)
    render = r.render_two_pass if two_pass else r.render
    if cfg.get("resort"):
        r.vrs_set_resort_mode(cfg["resort"])
    r.vrs_set_staging_mode(1 if args.staging == "tma" else 0)
    if rank == 0:
        r.upload(scene)
    scene_bcast_bytes = None
    if world > 1:
        from paper_2505_10144_b200.parallel import broadcast_uploaded_scene
        scene_bcast_bytes = broadcast_uploaded_scene(r, src=0)
    for k, m in masks.items():
        r.set_mask(k, m)
    stream = torch.cuda.Stream(device=local)
    rgba, depth = r.alloc_outputs(cams)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # counters run (outside timing): workload counters for the roofline
    r.vrs_set_instrumentation(counters=1, timing=0)
    with torch.cuda.stream(stream):
        render(cams, fov, rgba, depth, stream=stream)
    counters = r.stats()
    r.vrs_set_instrumentation(counters=0, timing=0)  # the timed frames run the bare product path
    # per-tile list-length histogram of that frame (SURVEY §8d reporting)
    try:
        rng = r.vrs_debug_ranges()
        lens = (rng[:, 1].astype(np.int64) - rng[:, 0].astype(np.int64))
        lens = lens[lens > 0]
        edges = [1, 65, 129, 257, 513, 1025, 2049, 4097]
        tile_hist = {f"{lo}-{hi - 1}" if hi else f">={lo}": int(((lens >= lo) & ((lens < hi) if hi else True)).sum())
                     for lo, hi in zip(edges, edges[1:] + [0])}
        tile_hist["max"] = int(lens.max()) if lens.size else 0
        tile_hist["mean"] = float(lens.mean()) if lens.size else 0.0
    except Exception as ex:  # (vrs_debug_ranges covers up to 1 M tiles)
        tile_hist = {"unavailable": str(ex)[:80]}

    for w in range(args.warmup):
        with torch.cuda.stream(stream):
            render(step_cams(args.config, cams, w, rank, world), fov, rgba, depth, stream=stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, stage = [], []
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                if not args.no_flush:
                    flush.fill_(s & 0xff)
                cs = step_cams(args.config, cams, s, rank, world)
                ev0[s].record(stream)
                render(cs, fov, rgba, depth, stream=stream)
                ev1[s].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [ev0[s].elapsed_time(ev1[s]) for s in range(args.steps)]
    # per-stage times: the same frames again with the library's stage events on (outside the timed steps)
    r.vrs_set_instrumentation(counters=0, timing=1)
    for s in range(args.steps):
        with torch.cuda.stream(stream):
            if not args.no_flush:
                flush.fill_(s & 0xff)
            render(step_cams(args.config, cams, s, rank, world), fov, rgba, depth, stream=stream)
        stage.append(r.stats()["stage_ms"])  # also raises VRS_E_CAPACITY if a frame overflowed
    r.vrs_set_instrumentation(counters=0, timing=0)
    ms = float(np.mean(step_ms))
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    stage_ms = np.mean(np.array(stage), axis=0).tolist()
    names = ["preprocess", "scan", "duplicate", "sort", "ranges", "blend", "compose"]

    # ---- end to end through the public API with HOST buffers (pinned), copies inside the timed region.
    # Headline: frames pipelined two deep -- frame s renders on the compute stream while frame s-1's
    # RGBA+depth D2H runs on a copy stream (double-buffered device and pinned host outputs; a buffer is
    # re-rendered only after its copy finished).  Also reported: the synchronous vrs_render_views_host
    # call (render + D2H + stream sync per frame).
    e2e = None
    if not args.no_e2e:
        unit = "stereo frames/s" if len(cams) == 2 else "frames/s"
        cam_bytes = len(cams) * (72 + 24)

        def measure_e2e(fmt):
            r.vrs_set_output_format(fmt)
            h = [r.alloc_outputs(cams, pinned_host=True) for _ in range(E2E_DEPTH)]
            d = [r.alloc_outputs(cams) for _ in range(E2E_DEPTH)]
            cstream = torch.cuda.Stream(device=local)
            rendered = [torch.cuda.Event() for _ in range(E2E_DEPTH)]
            copied = [torch.cuda.Event() for _ in range(E2E_DEPTH)]
            n_e2e = min(args.steps, 20)

            def pipelined(n):
                for s in range(n):
                    b = s % E2E_DEPTH
                    cs = step_cams(args.config, cams, s, rank, world)
                    if s >= E2E_DEPTH:
                        stream.wait_event(copied[b])
                    with torch.cuda.stream(stream):
                        render(cs, fov, d[b][0], d[b][1], stream=stream)
                        rendered[b].record(stream)
                    cstream.wait_event(rendered[b])
                    with torch.cuda.stream(cstream):  # byte views: the same copy for every format
                        h[b][0].view(torch.uint8).copy_(d[b][0].view(torch.uint8), non_blocking=True)
                        h[b][1].view(torch.uint8).copy_(d[b][1].view(torch.uint8), non_blocking=True)
                        copied[b].record(cstream)
                cstream.synchronize()

            def sync_call():
                if two_pass:  # public Python API: device render, then D2H into pinned memory on the same stream
                    with torch.cuda.stream(stream):
                        render(cams, fov, d[0][0], d[0][1], stream=stream)
                        h[0][0].view(torch.uint8).copy_(d[0][0].view(torch.uint8), non_blocking=True)
                        h[0][1].view(torch.uint8).copy_(d[0][1].view(torch.uint8), non_blocking=True)
                    stream.synchronize()
                else:
                    r.render_host(cams, fov, h[0][0], h[0][1], stream=stream)

            def timed(fn):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                fn()
                t = time.perf_counter() - t0
                e_t = torch.tensor([t], dtype=torch.float64, device="cuda")
                if world > 1:
                    dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
                return float(e_t.item())

            pipelined(4)
            for _ in range(2):
                sync_call()
            # median of three timed runs of n_e2e frames each (host clock: one run is exposed to
            # host-side noise)
            pipe_s = statistics.median(timed(lambda: pipelined(n_e2e)) for _ in range(3)) / n_e2e
            sync_s = statistics.median(timed(lambda: [sync_call() for _ in range(n_e2e)]) for _ in range(3)) / n_e2e
            r.vrs_set_output_format(0)
            nbytes = int(h[0][0].numel() * h[0][0].element_size() + h[0][1].numel() * h[0][1].element_size())
            return world / pipe_s, world / sync_s, nbytes

        r.vrs_set_instrumentation(counters=0, timing=0)  # no per-stage events on the end-to-end path
        v8, s8, b8 = measure_e2e(1)
        v32, s32, b32 = measure_e2e(0)
        v16, s16, b16 = measure_e2e(2)
        what = "render_two_pass" if two_pass else "render"
        # headline: the most compact output format that still meets the north_star tolerances on
        # every pixel (RGBA binary16: |rounding| <= 2^-11 |v| against the 2e-3 RGB bar; depth float)
        e2e = {"value": v16, "unit": unit, "h2d_bytes_per_step": cam_bytes, "d2h_bytes_per_step": b16,
               "sync_value": s16, "format": "VRS_OUT_RGBA16F_D32F (RGBA binary16 + depth float32, the half-float swap-chain "
                                            "format: within the parity tolerances on every pixel, "
                                            "tests/test_gpu_output_formats.py)",
               "f32": {"value": v32, "sync_value": s32, "d2h_bytes_per_step": b32,
                       "format": "VRS_OUT_F32 (RGBA float32 + depth float32)"},
               "display_packed": {"value": v8, "sync_value": s8, "d2h_bytes_per_step": b8,
                                  "format": "VRS_OUT_RGBA8_D16F (RGBA unorm8 + depth binary16, the HMD display "
                                            "format; depth quantised to 2^-11 relative, outside the 1e-4 bar)"},
               "note": what + " into device buffers with the D2H of the frame into pinned host memory on a copy "
                       "stream, " + str(E2E_DEPTH) + " frames in flight (value); sync_value = " +
                       ("render_two_pass + D2H + sync" if two_pass else "vrs_render_views_host") +
                       " per frame; host wall clock; camera/fovea structs travel as kernel parameters"}

    # ---- multi-GPU end to end: every step's frames gathered to rank 0 (grouped NCCL send/recv on a
    # side stream, overlapping the next step's render; SURVEY §8e "final frame gather")
    gather = measure_gather(args, r, render, cams, fov, stream, rank, world, local, one_gpu) if world > 1 else None

    if rank == 0:
        peaks, src = measured_peaks()
        clocks = clk.summary()
        sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        # dominant kernel: blend, issue-bound: algorithmic
        # lane-instructions = 11 per evaluation + 65 per contribution
        blend_ms = stage_ms[5]
        alg_ops = 11.0 * counters["evaluations"] + 65.0 * counters["contributions"]
        peak_ops = 148 * 4 * 32 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        achieved = alg_ops / (blend_ms * 1e-3) if blend_ms > 0 else 0.0
        traffic, winst = None, None
        tp = os.path.join(ROOT, "profiles", "blend_traffic.json")
        if os.path.exists(tp):
            try:
                tj = json.load(open(tp))
                traffic, winst = tj.get(args.config), tj.get(args.config + "_warp_instructions")
            except Exception:
                traffic = None
        n_views = len(cams)
        # k_cull, k_preprocess, k_color, k_tiletest_direct, k_tile_scan, k_ovf_bucket, k_tile_sort and ONE
        # k_blend (blend items, invisible fills and the in-launch compose); the hierarchical mode blends with
        # k_blend_hier + k_compose; the two-pass baseline adds k_two_pass_combine
        launches_per_step = 8 + (1 if cfg.get("resort") else 0) + (1 if two_pass else 0)
        line = {
            "metric": METRIC if args.config == "c2" else METRIC + f" [{args.config}]",
            "value": world * 1000.0 / ms_max,
            "unit": "stereo frames/s" if n_views == 2 else "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(args.config, r.n, cams, world, {
                "l2": "flushed between steps (256 MB write, outside the event pair)" if not args.no_flush
                else "not flushed", "staging": args.staging}),
            "stage_ms": dict(zip(names, stage_ms)),
            "workload_counters": {k: counters[k] for k in ("pairs", "samples", "evaluations", "contributions",
                                                           "overflow_samples", "terminated_samples", "work_items",
                                                           "visible_splats")},
            "tiles_by_class": dict(zip(["high", "low", "hybrid", "invisible"], counters["tiles_by_class"])),
            "tile_list_hist": tile_hist,
            "roofline": {"kernel": "k_blend", "bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12,
                         "unit": "T lane-instr/s", "frac": achieved / peak_ops, "traffic": traffic,
                         "peak_source": f"148 SM x 4 schedulers x 32 lanes x sm_max_mhz ({src} MEASURED_PEAKS)",
                         "algorithmic_ops_per_launch": alg_ops,
                         # executed warp instructions of the launch (ncu, profiles/) over the live blend time
                         # against the issue peak (148 SM x 4 schedulers x clock): how full the issue slots are
                         "issue_frac": (winst / (blend_ms * 1e-3 * 148 * 4 * float(peaks.get("sm_max_mhz", 1965.0))
                                                 * 1e6)) if winst and blend_ms > 0 else None},
            "stage_roofline": stage_roofline(counters, stage_ms, r.n, n_views, peaks),
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
            "gather": gather,
            "scene_broadcast_bytes": scene_bcast_bytes,
            "context": {"paper_rtx4090_ms_per_stereo_frame_0.5M_scenes": [9.89, 12.19],
                        "paper_headline": "72+ FPS on RTX 4090 at 2x2064x2272 (P:91, P:107)"},
        }
        if cfg.get("resort"):
            line["vs_flat"] = compare_flat(r, render, cams, fov, rgba, depth, stream, counters)
        if not args.no_cpu_baseline and world == 1 and not two_pass and not cfg.get("resort"):
            line["cpu_baseline"] = cpu_baseline(scene, cams, fov, masks, cfg["T"], budget_s=12.0)
            one = cpu_baseline(scene, cams, fov, masks, cfg["T"], budget_s=8.0, threads=1)
            line["cpu_baseline"]["single_thread"] = {k: one[k] for k in ("value", "cores", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_gather(args, r, render, cams, fov, stream, rank, world, local, one_gpu):
    """Render + gather per step: each rank renders its step's frame into one of two
    device buffers; a side stream waits for it and runs the grouped send/recv of
    the frame to rank 0 in the half-float format that meets the parity
    tolerances (VRS_OUT_RGBA16F_D32F: RGBA binary16 + depth f32, 12 B/px),
    which receives every rank's frame
    into its own double buffer; a buffer is re-rendered only after its send
    finished.  Host wall clock over the steps, max over ranks."""
    import torch
    import torch.distributed as dist
    n = min(args.steps, 20)
    cstream = torch.cuda.Stream(device=local)
    r.vrs_set_output_format(2)
    d = [r.alloc_outputs(cams) for _ in range(2)]
    sent = [torch.cuda.Event() for _ in range(2)]
    rendered = [torch.cuda.Event() for _ in range(2)]
    recv = None
    if rank == 0:
        recv = [[r.alloc_outputs(cams) for _ in range(world)] for _ in range(2)]
    bytes_per_rank = int(d[0][0].numel() * d[0][0].element_size() + d[0][1].numel() * d[0][1].element_size())

    def step(s):
        b = s & 1
        cs = step_cams(args.config, cams, s, rank, world)
        if s >= 2:
            stream.wait_event(sent[b])
        with torch.cuda.stream(stream):
            render(cs, fov, d[b][0], d[b][1], stream=stream)
            rendered[b].record(stream)
        cstream.wait_event(rendered[b])
        with torch.cuda.stream(cstream):
            if one_gpu:  # gloo test hook: host tensors
                cstream.synchronize()
                frames = [d[b][0].cpu(), d[b][1].cpu()]
            else:
                frames = [d[b][0], d[b][1]]
            if rank == 0:
                ops = []
                for src in range(1, world):
                    for k in range(2):
                        buf = recv[b][src][k] if not one_gpu else torch.empty_like(frames[k])
                        ops.append(dist.P2POp(dist.irecv, buf, src))
            else:
                ops = [dist.P2POp(dist.isend, t, 0) for t in frames]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            sent[b].record(cstream)

    try:
        for s in range(2):
            step(s)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(n):
            step(s)
        cstream.synchronize()
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    finally:
        r.vrs_set_output_format(0)
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    unit = "stereo frames/s" if len(cams) == 2 else "frames/s"
    return {"value": world * n / t, "unit": unit, "steps": n, "ms_per_step": 1000.0 * t / n,
            "gathered_bytes_per_step": bytes_per_rank * (world - 1),
            "note": "render + grouped send/recv of every rank's frame (RGBA binary16 + depth f32, within the "
                    "parity tolerances) to rank 0 on a side stream (double-buffered), host wall clock, max over "
                    "ranks; `value` above is render-only"}


def compare_flat(r, render, cams, fov, rgba, depth, stream, counters):
    """Hierarchical frame vs the flat K = 16 frame of the same cameras: PSNR of
    RGB, max |dRGBA|, and both modes' window-overflow counters (approximation
    events) and blend times."""
    import torch
    with torch.cuda.stream(stream):
        render(cams, fov, rgba, depth, stream=stream)
    torch.cuda.synchronize()
    hier = rgba.clone()
    r.vrs_set_resort_mode(0)
    r.vrs_set_instrumentation(counters=1, timing=1)
    with torch.cuda.stream(stream):
        render(cams, fov, rgba, depth, stream=stream)
    flat_counters = r.stats()
    blend_flat = []
    r.vrs_set_instrumentation(counters=0, timing=1)
    for _ in range(10):
        with torch.cuda.stream(stream):
            render(cams, fov, rgba, depth, stream=stream)
        blend_flat.append(r.stats()["stage_ms"][5])
    torch.cuda.synchronize()
    d = (hier[:, :3] - rgba[:, :3]).double()
    mse = float((d * d).mean())
    out = {"psnr_rgb_db": 10.0 * np.log10(1.0 / mse) if mse > 0 else float("inf"),
           "max_abs_rgba": float((hier - rgba).abs().max()),
           "overflow_samples": {"hier": counters["overflow_samples"], "flat": flat_counters["overflow_samples"]},
           "contributions": {"hier": counters["contributions"], "flat": flat_counters["contributions"]},
           "flat_blend_ms": float(np.mean(blend_flat))}
    r.vrs_set_resort_mode(1)
    return out


def make_cams_only(cfg_name):
    c = CONFIGS[cfg_name]
    if cfg_name == "c1":
        return [sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)], None, {}
    cams = sg.stereo_pair(masks=c["masks"])
    fov = [sg.quest_fovea()] * 2 if c["fovea"] else None
    masks = {0: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H), 1: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H)} if c["masks"] else {}
    return cams, fov, masks


if __name__ == "__main__":
    main()
