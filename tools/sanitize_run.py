"""Small renders through every kernel family for compute-sanitizer runs:
flat foveated stereo (T=32, masks; thread and TMA staging; the in-launch
compose), non-foveated T=16 + backward, hierarchical mode, EWA, two-pass,
packed output, the global-sort baselines, and a 640x480 stereo frame
(2400 tiles: the multi-chunk look-back of k_tile_scan)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen as sg  # noqa: E402
from paper_2505_10144_b200 import Renderer  # noqa: E402

W, H = 96, 80
scene = sg.vr_room(3, 4000, sh_degree=2)
f = sg.focal_for_hfov(W, 110.0)
cams = [sg.look_camera((x, 0, 0), 0.2, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
        for e, x in enumerate((-0.0315, 0.0315))]
fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
for proj in (0, 1):
    r = Renderer(max_gaussians=scene.n, max_views=4, max_pairs=1 << 20, max_width=W, max_height=H,
                 assign_tile=32, projection=proj)
    r.upload(scene)
    for e in range(2):
        r.set_mask(e, sg.ellipse_mask(W, H))
    r.vrs_set_instrumentation(counters=1)
    r.render(cams, fov)
    r.vrs_set_staging_mode(1)  # TMA staging
    r.render(cams, fov)
    r.vrs_set_staging_mode(0)
    r.vrs_set_sort_mode(1)     # global-sort baseline
    r.render(cams, fov)
    r.vrs_set_sort_mode(0)
    if proj == 0:
        r.render_two_pass(cams, fov)
        r.vrs_set_resort_mode(1)
        r.render(cams, fov)
        r.vrs_set_resort_mode(0)
        r.vrs_set_output_format(1)
        r.render(cams, fov)
        r.vrs_set_output_format(2)  # half-float RGBA + float depth
        r.render(cams, fov)
        r.render_two_pass(cams, fov)
        r.vrs_set_output_format(0)
    torch.cuda.synchronize()
    r.close()
r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 20, max_width=W, max_height=H, assign_tile=16)
r.upload(scene)
nofov = [sg.look_camera((x, 0, 0), 0.2, 0.1, 0.0, f=f, width=W, height=H) for x in (-0.0315, 0.0315)]
rgba, depth = r.render(nofov)
out = r.vrs_backward(rgba, depth, torch.ones_like(rgba), torch.ones_like(depth))
torch.cuda.synchronize()
r.close()
# > 1024 tiles: k_tile_scan's multi-chunk look-back; > 256-pair tiles: the block sort path
W2, H2 = 640, 480
r = Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 21, max_width=W2, max_height=H2, assign_tile=16)
r.upload(scene)
f2 = sg.focal_for_hfov(W2, 110.0)
r.render([sg.look_camera((x, 0, 0), 0.2, 0.1, 0.0, f=f2, width=W2, height=H2) for x in (-0.0315, 0.0315)])
torch.cuda.synchronize()
r.close()
print("sanitize run done", float(out["means"].abs().max()))
