"""Probe: the C2 frame enqueued directly vs replayed from a captured CUDA graph
(stream capture of vrs_render_views, including its side-stream fork/join)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402

scene, cams, fov, masks = bench.make_workload("c2")
r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=8 << 20, max_width=2064, max_height=2208, assign_tile=32)
r.upload(scene)
for k, m in masks.items():
    r.set_mask(k, m)
rgba, depth = r.alloc_outputs(cams)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        r.render(cams, fov, rgba, depth, stream=s)
torch.cuda.synchronize()
ref = rgba.clone()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    r.render(cams, fov, rgba, depth, stream=s)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
print("graph output identical:", bool(torch.equal(ref, rgba)))


def timeit(fn, n=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for _ in range(5):
            fn()
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print(f"direct {timeit(lambda: r.render(cams, fov, rgba, depth, stream=s)):.4f} ms/frame, "
      f"graph {timeit(lambda: g.replay()):.4f} ms/frame (back to back, L2 warm)")
