"""Probe: the C3 workload (3M Gaussians, stereo, no foveation) with 16x16 vs
32x32 assignment tiles (T_a = 32 renders every coarse tile as four full-rate
16x16 items sharing the coarse list): frame ms and stage ms of each."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402

scene, cams, fov, masks = bench.make_workload("c3")
for T in (16, 32):
    r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=24 << 20, max_width=2064, max_height=2208,
                 assign_tile=T)
    r.upload(scene)
    rgba, depth = r.alloc_outputs(cams)
    for _ in range(3):
        r.render(cams, None, rgba, depth)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        r.render(cams, None, rgba, depth)
    e1.record()
    torch.cuda.synchronize()
    r.vrs_set_instrumentation(counters=1, timing=1)
    r.render(cams, None, rgba, depth)
    st = r.stats()
    print(f"T={T}: {e0.elapsed_time(e1) / 20:.3f} ms/frame, stages {[round(x, 3) for x in st['stage_ms'][:7]]}, "
          f"pairs {st['pairs']}, evaluations {st['evaluations']}, contributions {st['contributions']}")
    r.close()
