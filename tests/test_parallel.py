"""Multi-process (gloo, world_size 2, CPU) tests of the view-sharding host
logic: shards partition the views without splitting stereo pairs, the scene
broadcast is byte-identical on every rank, and the frame gather returns the
frames to rank 0 in view order."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_10144_b200.parallel import gather_frames, max_over_ranks, shard_range, shard_views


def test_shard_partition_properties():
    for n in (0, 1, 7, 360):
        for world in (1, 2, 3, 4, 8):
            seen = []
            sizes = []
            for r in range(world):
                a, b = shard_range(n, world, r)
                seen.extend(range(a, b))
                sizes.append(b - a)
                views = shard_views(n, world, r)
                assert all(views[i] // 2 == views[i + 1] // 2 for i in range(0, len(views), 2))
            assert seen == list(range(n))
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scenegen as sg
        from paper_2505_10144_b200.parallel import broadcast_scene
        scene = sg.vr_room(5, 2000, sh_degree=3) if rank == 0 else None
        got = broadcast_scene(scene, 2000, 3)
        ref = sg.vr_room(5, 2000, sh_degree=3)
        ok_bcast = all(np.array_equal(getattr(got, f), getattr(ref, f))
                       for f in ("means", "quats", "log_scales", "logits", "sh"))
        n_pairs = 5
        views = shard_views(n_pairs, world, rank)
        frames = [torch.full((3, 4), float(v)) for v in views]
        per_rank = [len(shard_views(n_pairs, world, r)) for r in range(world)]
        out = gather_frames(frames, per_rank, dst=0)
        order_ok = True
        if rank == 0:
            order_ok = [int(t[0, 0].item()) for t in out] == list(range(2 * n_pairs))
        mx = max_over_ranks(float(rank + 1))
        q.put((rank, ok_bcast, order_ok, mx))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_bcast, order_ok, mx in res:
        assert ok_bcast and order_ok and mx == 2.0
