"""Probe of the end-to-end host path at C2 in the half-float format: frames/s of
(a) the pipelined render loop without copies (host submission + render),
(b) the D2H copies alone (one stream vs the frame split over two copy streams),
(c) render + copy pipelined with one or two copy streams."""
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
r.vrs_set_output_format(2)
stream = torch.cuda.Stream()
cs = [torch.cuda.Stream(), torch.cuda.Stream()]
h = [r.alloc_outputs(cams, pinned_host=True) for _ in range(2)]
d = [r.alloc_outputs(cams) for _ in range(2)]
rendered = [torch.cuda.Event() for _ in range(2)]
copied = [[torch.cuda.Event() for _ in range(2)] for _ in range(2)]


def copy(b, nsplit):
    pieces = []
    for t_h, t_d in ((h[b][0], d[b][0]), (h[b][1], d[b][1])):
        hb, db = t_h.view(torch.uint8).view(-1), t_d.view(torch.uint8).view(-1)
        n = hb.numel()
        cuts = [n * i // nsplit for i in range(nsplit + 1)]
        pieces += [(hb[cuts[i]:cuts[i + 1]], db[cuts[i]:cuts[i + 1]], i) for i in range(nsplit)]
    for hh, dd, i in pieces:
        with torch.cuda.stream(cs[i]):
            hh.copy_(dd, non_blocking=True)


def loop(n, do_render=True, do_copy=True, nsplit=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(n):
        b = s & 1
        if s >= 2 and do_copy:
            for i in range(nsplit):
                stream.wait_event(copied[b][i])
        if do_render:
            with torch.cuda.stream(stream):
                r.render(cams, fov, d[b][0], d[b][1], stream=stream)
                rendered[b].record(stream)
        if do_copy:
            for i in range(nsplit):
                cs[i].wait_event(rendered[b])
            copy(b, nsplit)
            for i in range(nsplit):
                copied[b][i].record(cs[i])
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t0)


for _ in range(2):
    loop(6)
print(f"render only      {loop(30, do_copy=False):7.1f} frames/s")
print(f"copy only, 1 str {loop(30, do_render=False, nsplit=1):7.1f} frames/s")
print(f"copy only, 2 str {loop(30, do_render=False, nsplit=2):7.1f} frames/s")
print(f"render+copy 1    {loop(30, nsplit=1):7.1f} frames/s")
print(f"render+copy 2    {loop(30, nsplit=2):7.1f} frames/s")
