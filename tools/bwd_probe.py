"""Time the N4 backward on a non-foveated stereo frame (C2 scene, T_a = 16):
forward render, then vrs_backward with random gradient images."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as sg  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
scene = sg.vr_room(2, n, scale_mul=1.0, sh_degree=3)
cams = sg.stereo_pair(masks=False)
r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=16 << 20, max_width=2064, max_height=2208, assign_tile=16)
r.upload(scene)
rgba, depth = r.render(cams)
g_rgba = torch.randn_like(rgba)
g_depth = torch.randn_like(depth) * 0.1
for _ in range(2):
    rgba, depth = r.render(cams, None, rgba, depth)
    out = r.vrs_backward(rgba, depth, g_rgba, g_depth)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
fw, bw = [], []
for _ in range(5):
    e[0].record()
    r.render(cams, None, rgba, depth)
    e[1].record()
    out = r.vrs_backward(rgba, depth, g_rgba, g_depth)
    e[2].record()
    torch.cuda.synchronize()
    fw.append(e[0].elapsed_time(e[1]))
    bw.append(e[1].elapsed_time(e[2]))
print(f"forward {np.median(fw):.3f} ms, backward {np.median(bw):.3f} ms, |g_means| {out['means'].abs().max().item():.3e}")
