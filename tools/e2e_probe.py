"""Probe of the host-path pipeline: per-frame wall time of the pipelined
render + D2H loop for several frame counts, and the host-side submission
time per frame (how long the Python/C call chain takes to enqueue a frame)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402

scene, cams, fov, masks = bench.make_workload("c2")
r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=8 << 20, max_width=2064, max_height=2208, assign_tile=32)
r.upload(scene)
for k, m in masks.items():
    r.set_mask(k, m)
r.vrs_set_output_format(1)
stream, cstream = torch.cuda.Stream(), torch.cuda.Stream()
h = [r.alloc_outputs(cams, pinned_host=True) for _ in range(2)]
d = [r.alloc_outputs(cams) for _ in range(2)]
rendered = [torch.cuda.Event() for _ in range(2)]
copied = [torch.cuda.Event() for _ in range(2)]


def run(n, copy=True):
    sub = 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(n):
        b = s & 1
        ts = time.perf_counter()
        if s >= 2 and copy:
            stream.wait_event(copied[b])
        with torch.cuda.stream(stream):
            r.render(cams, fov, d[b][0], d[b][1], stream=stream)
            rendered[b].record(stream)
        if copy:
            cstream.wait_event(rendered[b])
            with torch.cuda.stream(cstream):
                h[b][0].copy_(d[b][0], non_blocking=True)
                h[b][1].copy_(d[b][1], non_blocking=True)
                copied[b].record(cstream)
        sub += time.perf_counter() - ts
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, sub / n * 1e3


run(5)
for n in (20, 50, 100):
    print(f"pipelined n={n}: {run(n)[0]:.3f} ms/frame, host submit {run(n)[1]:.3f} ms/frame")
print(f"render only n=100: {run(100, copy=False)[0]:.3f} ms/frame")
r.vrs_set_instrumentation(counters=0, timing=1)
print(f"with stage timing events: pipelined n=20: {run(20)[0]:.3f} ms/frame")
