"""Pins of the oracle's N2 hierarchical resort mode (DESIGN
"N2 hierarchical resort"): a block queue of K_B entries per 4x4 sample block
ahead of a per-sample window of K_P entries.  CPU only.

H1  K_B = 0 releases every entry at admission: identical (bit for bit, and
    every workload counter) to the flat per-sample window with K = K_P.
H2  K_B, K_P >= any list length: every sample blends ALL its Gaussians in
    full (tau, g) order -- identical to the tile-free brute-force renderer
    (the textbook per-pixel full sort, pin P9's reference).
H3  Queue mechanics on given streams (orc_hier_core): (a) a hand-derived
    three-entry example where the block order, the stream order and the
    per-sample order all differ; (b) the cascade theorem: with tau_B equal to
    every sample's tau and every sample a member, min-queues of K_B and K_P
    in series emit exactly what one min-queue of K_B + K_P emits.
H4  Invariants on foveated renders (A = 1 - T in [0, 1], RGB >= 0,
    determinism across thread counts).
"""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg


def _stereo(W, H):
    f = sg.focal_for_hfov(W, 110.0)
    return [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H) for x in (-0.0315, 0.0315)]


def _c1(seed):
    return sg.random_scene(seed, n=1000, sh_degree=0), sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("kp", [1, 4, 8])
def test_h1_zero_block_queue_is_flat_window(oracle_mod, seed, kp):
    scene, cam = _c1(seed)
    o = oracle_mod.Oracle(scene)
    o.prepare([cam], assign_tile=16, window_k=kp)
    (a, da), = o.render()
    sa = o.stats()
    o.prepare([cam], assign_tile=16, window_k=kp, resort=1, block_queue=0)
    (b, db), = o.render()
    assert np.array_equal(a, b) and np.array_equal(da, db)
    assert o.stats() == sa


def test_h1_foveated_lowres_blocks(oracle_mod):
    """H1 on a foveated, masked frame: LowRes blocks are 4x4 2x2-groups (8x8 px)."""
    W, H = 200, 136
    scene = sg.vr_room(5, 20000, scale_mul=1.0, sh_degree=1)
    cams = _stereo(W, H)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    o = oracle_mod.Oracle(scene)
    o.prepare(cams, fov, assign_tile=32, window_k=4)
    ra = o.render()
    sa = o.stats()
    o.prepare(cams, fov, assign_tile=32, window_k=4, resort=1, block_queue=0)
    rb = o.render()
    for (a, da), (b, db) in zip(ra, rb):
        assert np.array_equal(a, b) and np.array_equal(da, db)
    assert o.stats() == sa


@pytest.mark.parametrize("seed", [0, 3])
def test_h2_unbounded_queues_are_the_full_sort(oracle_mod, seed):
    scene, cam = _c1(seed)
    o = oracle_mod.Oracle(scene)
    o.prepare([cam], assign_tile=16, window_k=1 << 20, resort=1, block_queue=1 << 20)
    (a, da), = o.render()
    bf, bfd = o.bruteforce(0)
    assert np.array_equal(a, bf) and np.array_equal(da, bfd)


def test_h3_hand_derived_three_entries(oracle_mod):
    """Stream order e0, e1, e2; block depths tau_B = (3, 1, 2) -> with K_B = 3
    the block releases e1, e2, e0 at stream end; per-sample depths
    tau = (1, 2, 3) (true order e0, e1, e2); alpha = 1/2 each; K_P = 1.
    Window of one: e1 | e2 arrives -> blend e1 (T 1 -> 1/2) | e0 arrives ->
    blend e0 (T -> 1/4) | drain e2 (T -> 1/8).  Colours e_i = unit vector i:
    RGB = (1/4, 1/2, 1/8), A = 7/8, depth = 2/2 + 1/4 + 3/8 = 13/8."""
    n = 3
    tau_b = np.array([3, 1, 2], np.float32)
    g = np.array([10, 11, 12], np.uint32)
    member = np.full(n, 0xFFFF, np.uint32)
    tau = np.repeat(np.array([1, 2, 3], np.float32)[:, None], 16, 1)
    alpha = np.full((n, 16), 0.5, np.float32)
    rgb = np.eye(3, dtype=np.float32)
    out, st = oracle_mod.hier_core(tau_b, g, member, tau, alpha, rgb, kb=3, kp=1)
    np.testing.assert_array_equal(out, np.tile([0.25, 0.5, 0.125, 0.875, 1.625], (16, 1)))
    assert (st[:, 1] == 3).all() and (st[:, 2] == 1).all() and (st[:, 3] == 0).all()
    # the same stream with K_P = 3 resorts fully: e0, e1, e2 -> (1/2, 1/4, 1/8)
    out, _ = oracle_mod.hier_core(tau_b, g, member, tau, alpha, rgb, kb=3, kp=3)
    np.testing.assert_array_equal(out[0, :3], [0.5, 0.25, 0.125])
    # a partial membership: sample 5 only sees e2 -> alpha 1/2 of blue
    member2 = member.copy()
    member2[:2] &= ~np.uint32(1 << 5)
    out, st = oracle_mod.hier_core(tau_b, g, member2, tau, alpha, rgb, kb=3, kp=1)
    np.testing.assert_array_equal(out[5], [0, 0, 0.5, 0.5, 1.5])
    assert st[5, 1] == 1


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("kb,kp", [(1, 1), (2, 3), (4, 4), (8, 8), (3, 13)])
def test_h3_cascade_equals_one_queue(oracle_mod, seed, kb, kp):
    rng = np.random.default_rng(seed)
    n = 60
    t = rng.permutation(np.arange(1, n + 1)).astype(np.float32) * 0.25
    t[rng.integers(0, n, 5)] = t[0]  # some ties: broken by g
    g = rng.permutation(1000)[:n].astype(np.uint32)
    member = np.full(n, 0xFFFF, np.uint32)
    tau = np.repeat(t[:, None], 16, 1)
    alpha = rng.uniform(0.01, 0.3, (n, 16)).astype(np.float32)
    rgb = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    a, sa = oracle_mod.hier_core(t, g, member, tau, alpha, rgb, kb=kb, kp=kp)
    b, sb = oracle_mod.hier_core(t, g, member, tau, alpha, rgb, kb=0, kp=kb + kp)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(sa[:, [0, 3]], sb[:, [0, 3]])


def test_h4_invariants_and_determinism(oracle_mod):
    W, H = 160, 128
    scene = sg.vr_room(6, 20000, scale_mul=1.0, sh_degree=2)
    cams = _stereo(W, H)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    o = oracle_mod.Oracle(scene)
    outs = []
    for threads in (1, 4):
        o.prepare(cams, fov, assign_tile=32, window_k=8, resort=1, block_queue=8, threads=threads)
        outs.append(o.render())
    for (a, da), (b, db) in zip(*outs):
        assert np.array_equal(a, b) and np.array_equal(da, db)
        assert (a[..., :3] >= 0).all() and (a[..., 3] >= 0).all() and (a[..., 3] <= 1).all()
        assert (da >= 0).all()
    st = o.stats()
    assert st["contributions"] > 0 and st["samples"] > 0


# --------------------------------------------------------------------- the 2x2 group level (K_G > 0)

def test_h3_hand_derived_group_level(oracle_mod):
    """The H3 stream with a group queue of one between the block queue and the
    windows: block releases e1, e2, e0 (tau_B = 3, 1, 2) enter every group's
    queue ordered by tau_G = (2, 3, 1): e1 waits; e2 arrives -> e2 released;
    e0 arrives -> e0 released; drain -> e1.  Samples (K_P = 1, tau = 1, 2, 3,
    alpha 1/2) receive e2, e0, e1: e0 arrives -> blend e0 (T 1 -> 1/2); e1 ->
    blend e1 (T -> 1/4); drain e2 (T -> 1/8): RGB = (1/2, 1/4, 1/8), A = 7/8,
    depth = 1/2 + 2/4 + 3/8 = 11/8."""
    n = 3
    tau_b = np.array([3, 1, 2], np.float32)
    tau_g = np.repeat(np.array([2, 3, 1], np.float32)[:, None], 4, 1)
    g = np.array([10, 11, 12], np.uint32)
    member = np.full(n, 0xFFFF, np.uint32)
    tau = np.repeat(np.array([1, 2, 3], np.float32)[:, None], 16, 1)
    alpha = np.full((n, 16), 0.5, np.float32)
    rgb = np.eye(3, dtype=np.float32)
    out, st = oracle_mod.hier_core(tau_b, g, member, tau, alpha, rgb, kb=3, kp=1, kg=1, tau_g=tau_g)
    np.testing.assert_array_equal(out, np.tile([0.5, 0.25, 0.125, 0.875, 1.375], (16, 1)))
    # a group whose samples are not members never sees the entry
    member2 = member.copy()
    member2[0] = 0xFFFF & ~np.uint32(0x0033)  # e0 misses group 0 (samples 0, 1, 4, 5)
    out2, _ = oracle_mod.hier_core(tau_b, g, member2, tau, alpha, rgb, kb=3, kp=1, kg=1, tau_g=tau_g)
    np.testing.assert_array_equal(out2[15], out[15])
    assert not np.array_equal(out2[0], out[0])


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("kb,kg,kp", [(1, 1, 1), (2, 3, 4), (8, 4, 8), (0, 5, 3)])
def test_h3_three_level_cascade_equals_one_queue(oracle_mod, seed, kb, kg, kp):
    rng = np.random.default_rng(100 + seed)
    n = 60
    t = rng.permutation(np.arange(1, n + 1)).astype(np.float32) * 0.25
    t[rng.integers(0, n, 5)] = t[0]
    g = rng.permutation(1000)[:n].astype(np.uint32)
    member = np.full(n, 0xFFFF, np.uint32)
    tau = np.repeat(t[:, None], 16, 1)
    alpha = rng.uniform(0.01, 0.3, (n, 16)).astype(np.float32)
    rgb = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    a, sa = oracle_mod.hier_core(t, g, member, tau, alpha, rgb, kb=kb, kp=kp, kg=kg)
    b, sb = oracle_mod.hier_core(t, g, member, tau, alpha, rgb, kb=0, kp=kb + kg + kp, kg=0)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("seed", [0, 3])
def test_h2_three_levels_unbounded_are_the_full_sort(oracle_mod, seed):
    scene, cam = _c1(seed)
    o = oracle_mod.Oracle(scene)
    o.prepare([cam], assign_tile=16, window_k=1 << 20, resort=1, block_queue=1 << 20, group_queue=1 << 20)
    (a, da), = o.render()
    bf, bfd = o.bruteforce(0)
    assert np.array_equal(a, bf) and np.array_equal(da, bfd)


def test_h4_three_levels_foveated_invariants(oracle_mod):
    W, H = 160, 128
    scene = sg.vr_room(6, 20000, scale_mul=1.0, sh_degree=2)
    cams = _stereo(W, H)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    o = oracle_mod.Oracle(scene)
    outs = []
    for threads in (1, 4):
        o.prepare(cams, fov, assign_tile=32, window_k=8, resort=1, block_queue=8, group_queue=4, threads=threads)
        outs.append(o.render())
    for (a, da), (b, db) in zip(*outs):
        assert np.array_equal(a, b) and np.array_equal(da, db)
        assert (a[..., :3] >= 0).all() and (a[..., 3] >= 0).all() and (a[..., 3] <= 1).all()
