"""Probe: the C2 frame written by the kernels straight into pinned (UVA-mapped)
host memory, against rendering into device memory (+ a D2H copy).  Reports the
per-frame time of back-to-back renders into each destination and the blend
stage time, for the half-float and f32 output formats."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402
from paper_2505_10144_b200.vrs import lib  # noqa: E402

scene, cams, fov, masks = bench.make_workload("c2")
r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=8 << 20, max_width=2064, max_height=2208, assign_tile=32)
r.upload(scene)
for k, m in masks.items():
    r.set_mask(k, m)
stream = torch.cuda.Stream()


def raw_render(rgba, depth):
    carr, farr = r._views_structs(cams, fov)
    rc = lib().vrs_render_views(r.h, len(cams), C.cast(carr, C.c_void_p), C.cast(farr, C.c_void_p),
                                C.c_void_p(rgba.data_ptr()), C.c_void_p(depth.data_ptr()),
                                C.c_void_p(stream.cuda_stream))
    assert rc == 0, rc


for fmt in (2, 0):
    r.vrs_set_output_format(fmt)
    dev = r.alloc_outputs(cams)
    host = r.alloc_outputs(cams, pinned_host=True)
    for name, (a, d) in (("device", dev), ("mapped-host", host)):
        for _ in range(3):
            raw_render(a, d)
        torch.cuda.synchronize()
        n = 20
        t0 = time.perf_counter()
        for _ in range(n):
            raw_render(a, d)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / n
        r.vrs_set_instrumentation(counters=0, timing=1)
        raw_render(a, d)
        st = r.stats()["stage_ms"]
        r.vrs_set_instrumentation(counters=0, timing=0)
        print(f"fmt {fmt} {name:12s} {ms:.3f} ms/frame ({1000 / ms:.1f} stereo frames/s), blend {st[5]:.3f} ms")
    # correctness: the mapped frame equals the device frame
    raw_render(*dev)
    raw_render(*host)
    torch.cuda.synchronize()
    print("  identical:", torch.equal(dev[0].cpu().view(torch.uint8), host[0].view(torch.uint8)),
          torch.equal(dev[1].cpu().view(torch.uint8), host[1].view(torch.uint8)))
