"""Backward run-to-run variance probe: several contexts in one process, each
timing vrs_backward of the C9 frame 8 times (CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import scenegen as sg  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402

cfg = bench.CONFIGS["c9"]
scene = sg.vr_room(cfg["seed"], cfg["n"], scale_mul=cfg["scale_mul"], sh_degree=cfg["sh"])
cams = sg.stereo_pair(masks=False)
keep = []
for ctx in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=16 << 20, max_width=cams[0].width,
                 max_height=cams[0].height, assign_tile=cfg["T"])
    r.upload(scene)
    rgba, depth = r.alloc_outputs(cams)
    gen = torch.Generator(device="cuda").manual_seed(0)
    g_rgba = torch.randn(rgba.shape, device="cuda", generator=gen)
    g_depth = torch.randn(depth.shape, device="cuda", generator=gen) * 0.1
    r.render(cams, None, rgba, depth)
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r.vrs_backward(rgba, depth, g_rgba, g_depth)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"ctx {ctx}: backward ms {np.round(ts, 2).tolist()}", flush=True)
    keep.append(r)  # keep the allocations alive so the next context gets other addresses
