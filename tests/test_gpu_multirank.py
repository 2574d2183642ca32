"""Multi-rank view sharding on the CUDA path: two ranks (one
process each, gloo, both on cuda:0 since the GPU tests run on one device);
rank 0 uploads the scene and replicates the activated device buffers to rank
1 (parallel.broadcast_uploaded_scene: vrs_export_scene / vrs_import_scene);
the ranks render their contiguous shards of a head-motion trajectory's stereo
pairs and gather the frames to rank 0 with parallel.gather_frames; rank 0's
gathered frames equal a single-rank render of every pair bit for bit (views
are independent units: no exchange inside a frame)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_PAIRS, W, H = 5, 192, 160


def _pair_cams(t):
    import scenegen as sg
    head, yaw, pitch, roll = sg.trajectory_pose(t * 37)
    f = sg.focal_for_hfov(W, 110.0)
    cyw = np.cos(yaw)
    cams = []
    for e, x in enumerate((-0.0315, 0.0315)):
        c = sg.look_camera((head[0] + x * cyw, head[1], head[2] - x * np.sin(yaw)), yaw, pitch, roll, f=f,
                           width=W, height=H)
        cams.append(c)
    return cams


def _renderer(upload=True):
    import scenegen as sg
    from paper_2505_10144_b200 import Renderer
    r = Renderer(max_gaussians=30000, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H, assign_tile=32)
    if upload:
        r.upload(sg.vr_room(4, 30000, scale_mul=0.707, sh_degree=3))
    return r


def _render_pairs(pairs, r=None):
    import scenegen as sg
    r = r or _renderer()
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    out = []
    for p in pairs:
        rgba, depth = r.render(_pair_cams(p), fov)
        torch.cuda.synchronize()
        out += [rgba.cpu().clone(), depth.cpu().clone()]
    r.close()
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_10144_b200.parallel import broadcast_uploaded_scene, gather_frames, shard_range
        # rank 0 uploads; the activated scene reaches rank 1 as a device blob (no second upload)
        r = _renderer(upload=(rank == 0))
        broadcast_uploaded_scene(r, src=0)
        a, b = shard_range(N_PAIRS, world, rank)
        local = _render_pairs(range(a, b), r)
        per_rank = [shard_range(N_PAIRS, world, k)[1] - shard_range(N_PAIRS, world, k)[0] for k in range(world)]
        # gather_frames moves equally shaped tensors: the RGBA frames, then the depth frames
        rgba = gather_frames(local[0::2], per_rank, dst=0)
        dep = gather_frames(local[1::2], per_rank, dst=0)
        if rank == 0:
            q.put(("frames", [t.numpy() for pair in zip(rgba, dep) for t in pair]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gather_equals_one_rank():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    tag, frames = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    ref = _render_pairs(range(N_PAIRS))
    assert len(frames) == len(ref) == 2 * N_PAIRS
    for a, b in zip(frames, ref):
        assert np.array_equal(a, b.numpy())


def test_scene_export_import_roundtrip():
    """vrs_export_scene -> vrs_import_scene into a second context gives the same
    frames bit for bit, and the blob has the documented size."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    from paper_2505_10144_b200 import vrs as V
    a = _renderer()
    blob, n, deg = a.vrs_export_scene()
    assert blob.numel() == V.lib().vrs_scene_blob_bytes(n, deg) and n == a.n and deg == 3
    b = _renderer(upload=False)
    b.vrs_import_scene(n, deg, blob)
    fa = _render_pairs([1, 3], a)
    fb = _render_pairs([1, 3], b)
    for x, y in zip(fa, fb):
        assert torch.equal(x, y)
    with pytest.raises(V.VrsError):
        b.vrs_import_scene(n, deg, blob[:-256])
