"""Multi-GPU host logic: views shard across ranks.

Views (left/right eye, trajectory frames) are independent units, so every
rank holds a replica of the scene and renders a contiguous block of stereo
pairs; there is no exchange inside a frame.  Collectives are used only to
broadcast the scene once (``broadcast_uploaded_scene``: the activated device
buffers, device to device; ``broadcast_scene``: the raw arrays) and to gather finished frames
to rank 0 (``gather_frames``, grouped point-to-point sends, since NCCL has no
gather collective).  Works with ``nccl`` (CUDA tensors) and ``gloo`` (CPU
tensors, used by the tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_units: int, world: int, rank: int):
    """Contiguous block [a, b) of ``n_units`` for ``rank``; sizes differ by <= 1."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_units, world)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


def shard_views(n_pairs: int, world: int, rank: int):
    """View indices (2 per stereo pair, a pair never split) owned by ``rank``."""
    a, b = shard_range(n_pairs, world, rank)
    return [v for p in range(a, b) for v in (2 * p, 2 * p + 1)]


_FIELDS = ("means", "quats", "log_scales", "logits", "sh")


def broadcast_scene(scene, n: int, sh_degree: int, device=None, src: int = 0):
    """Broadcast the raw scene arrays from ``src`` (the only data-path collective).
    ``scene`` is a scenegen.RawScene on ``src`` and ignored elsewhere."""
    import torch
    import torch.distributed as dist

    from scenegen import RawScene
    k = (sh_degree + 1) ** 2
    shapes = {"means": (n, 3), "quats": (n, 4), "log_scales": (n, 3), "logits": (n,), "sh": (n, k, 3)}
    rank = dist.get_rank()
    out = {}
    for f in _FIELDS:
        if rank == src:
            t = torch.from_numpy(np.ascontiguousarray(getattr(scene, f), np.float32))
        else:
            t = torch.empty(shapes[f], dtype=torch.float32)
        if device is not None:
            t = t.to(device)
        dist.broadcast(t, src)
        out[f] = t.cpu().numpy()
    return RawScene(out["means"], out["quats"], out["log_scales"], out["logits"], out["sh"], sh_degree)


def broadcast_uploaded_scene(renderer, src: int = 0):
    """Device-to-device scene replication: ``src`` has uploaded the
    scene (host activation once); its activated buffers travel as one device
    blob by ``dist.broadcast`` (NCCL over NVLink; gloo test hook: host copy) and
    every other rank imports it -- no host round trip, no second activation.
    Returns the blob's byte count."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    dev = torch.device("cuda", renderer.device)
    gloo = dist.get_backend() == "gloo"
    meta = torch.zeros(3, dtype=torch.int64, device="cpu" if gloo else dev)
    blob = None
    if rank == src:
        blob, n, deg = renderer.vrs_export_scene()
        meta[0], meta[1], meta[2] = n, deg, blob.numel()
    dist.broadcast(meta, src)
    n, deg, nbytes = (int(x) for x in meta.tolist())
    if rank != src:
        blob = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    if gloo:
        torch.cuda.synchronize(dev)
        hb = blob.cpu()
        dist.broadcast(hb, src)
        blob.copy_(hb)
    else:
        dist.broadcast(blob, src)
    if rank != src:
        renderer.vrs_import_scene(n, deg, blob)
    torch.cuda.synchronize(dev)
    return nbytes


def gather_frames(local_frames, views_per_rank, dst: int = 0):
    """Grouped send/recv of each rank's frames (list of equally shaped tensors)
    to ``dst``; returns the full ordered list on ``dst`` and None elsewhere.
    ``views_per_rank[r]`` is the number of frames rank r contributes."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank != dst:
        ops = [dist.P2POp(dist.isend, t.contiguous(), dst) for t in local_frames]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return None
    out = []
    for r in range(world):
        if r == rank:
            out.extend(local_frames)
            continue
        like = local_frames[0] if local_frames else None
        bufs = [torch.empty_like(like) for _ in range(views_per_rank[r])]
        ops = [dist.P2POp(dist.irecv, b, r) for b in bufs]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        out.extend(bufs)
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank timing over all ranks (multi-GPU numbers are max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
