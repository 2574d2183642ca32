"""GPU parity: the CUDA path (through the C ABI) against the C++ oracle on
the same seeded inputs.  Bars (BASELINE.json north_star): bit-exact per-tile
pair counts, sorted key order, values and ranges; per-channel |dRGB| <= 2e-3
and |dDepth| <= 1e-4 relative on every compared pixel."""
from __future__ import annotations

import numpy as np
import pytest

import scenegen as sg
from helpers import identity_camera, scene_from, tiny_set

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RGB_TOL = 2e-3
DEPTH_REL = 1e-4
# decision fields of the 48-float splat record that must be bit-identical
EXACT_FIELDS = list(range(1, 34)) + [37, 38, 39, 40, 41, 42, 47]


@pytest.fixture(scope="module")
def vrs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_10144_b200 import build
    build.build()
    import paper_2505_10144_b200 as p
    return p


def render_both(vrs, oracle_mod, scene, cams, foveas=None, T=16, masks=None, max_pairs=1 << 22, counters=True,
                no_cull=False, oracle_render=True, projection=0, staging=0):
    W = max(c.width for c in cams)
    H = max(c.height for c in cams)
    r = vrs.Renderer(max_gaussians=max(scene.n, 1), max_views=len(cams), max_pairs=max_pairs, max_width=W,
                     max_height=H, assign_tile=T, projection=projection)
    r.upload(scene)
    o = oracle_mod.Oracle(scene)
    for slot, m in (masks or {}).items():
        r.set_mask(slot, m)
        o.set_mask(slot, m)
    r.vrs_set_instrumentation(counters=counters, no_cull=no_cull)
    r.vrs_set_staging_mode(staging)
    rgba, depth = r.render(cams, foveas)
    torch.cuda.synchronize()
    g_imgs = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), cams)
    o.prepare(cams, foveas, assign_tile=T, projection=projection)
    o_imgs = o.render() if oracle_render else None
    return r, o, g_imgs, o_imgs


def assert_images_close(g_imgs, o_imgs):
    for (gi, gd), (oi, od) in zip(g_imgs, o_imgs):
        drgb = np.abs(gi[..., :3] - oi[..., :3])
        assert drgb.max() <= RGB_TOL, f"max |dRGB| {drgb.max()} at {np.unravel_index(drgb.argmax(), drgb.shape)}"
        da = np.abs(gi[..., 3] - oi[..., 3])
        assert da.max() <= RGB_TOL, f"max |dA| {da.max()}"
        dd = np.abs(gd - od) - DEPTH_REL * np.abs(od)
        assert dd.max() <= 1e-6, f"depth excess {dd.max()} at {np.unravel_index(dd.argmax(), dd.shape)}"


def assert_lists_equal(r, o):
    assert np.array_equal(r.vrs_debug_counts(), o.counts()), "per-(view,g) pair counts differ"
    # emitted (unsorted) pairs: the GPU emits in arbitrary block order, so the
    # multisets are compared (the sorted list below is compared in order)
    ku, vu = r.vrs_debug_pairs(False)
    oku, ovu = o.pairs(False)
    gi, oi = np.lexsort((vu, ku)), np.lexsort((ovu, oku))
    assert np.array_equal(ku[gi], oku[oi]) and np.array_equal(vu[gi], ovu[oi]), "emitted pairs differ"
    k, v = r.vrs_debug_pairs(True)
    ok, ov = o.pairs(True)
    assert np.array_equal(k, ok), "sorted keys differ"
    assert np.array_equal(v, ov), "sorted values differ"
    assert np.array_equal(r.vrs_debug_ranges(), o.ranges()), "tile ranges differ"


def test_c1_parity(vrs, oracle_mod):
    """Config C1: 1000 Gaussians, SH0, 128^2, 90 deg, 16x16 tiles, no foveation."""
    scene = sg.random_scene(0, n=1000, sh_degree=0)
    cam = sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)
    r, o, g, oi = render_both(vrs, oracle_mod, scene, [cam])
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    st, ost = r.stats(), o.stats()
    for k in ("pairs", "samples", "evaluations", "contributions", "overflow_samples", "terminated_samples"):
        assert st[k] == ost[k], (k, st[k], ost[k])


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_c1_seeds_parity(vrs, oracle_mod, seed):
    """C1 seeds 0-24 subset, with SH degree 3 colour."""
    scene = sg.random_scene(seed, n=1000, sh_degree=3)
    cam = sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)
    r, o, g, oi = render_both(vrs, oracle_mod, scene, [cam])
    assert_lists_equal(r, o)
    assert_images_close(g, oi)


def test_preprocess_records_parity(vrs, oracle_mod):
    """Step 1: per-Gaussian records -- decision fields bit-exact, colour 1e-5."""
    scene = sg.random_scene(5, n=2000, sh_degree=3, xy_frac=1.5)
    cams = [sg.look_camera((-0.03, 0, 0), 0.1, -0.05, 0.02, f=90.0, width=200, height=150),
            sg.look_camera((0.03, 0, 0), 0.1, -0.05, 0.02, f=90.0, width=200, height=150)]
    r, o, _, _ = render_both(vrs, oracle_mod, scene, cams, oracle_render=False)
    for view in range(2):
        gs, os_ = r.vrs_debug_splats(view), o.splats(view)
        valid = os_[:, 0] == 1
        assert np.array_equal(gs[:, 0], os_[:, 0]), "valid flags differ"
        for f in EXACT_FIELDS:
            a, b = gs[valid, f], os_[valid, f]
            bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
            assert not bad.any(), f"field {f} differs at {np.nonzero(bad)[0][:5]}: {a[bad][:3]} vs {b[bad][:3]}"
        np.testing.assert_allclose(gs[valid, 34:37], os_[valid, 34:37], atol=1e-5)
        np.testing.assert_allclose(gs[valid, 43:47], os_[valid, 43:47], rtol=1e-6, atol=1e-4)


def test_foveated_masked_stereo_parity(vrs, oracle_mod):
    """Single-launch foveation with hybrid tiles, LowRes 2x2 groups, compose,
    visibility masks, stereo in one frame (T_a = 32)."""
    scene = sg.vr_room(7, 20000, sh_degree=3)
    W, H = 320, 256
    f = sg.focal_for_hfov(W, 110.0)
    cams = []
    for e, x in enumerate((-0.0315, 0.0315)):
        c = sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
        cams.append(c)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10)] * 2
    masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)}
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, masks=masks)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    for view in range(2):
        gc, gv = r.vrs_debug_tile_info(view, 32)
        oc, ov = o.tile_info(view)
        assert np.array_equal(gc, oc) and np.array_equal(gv, ov)
        assert set(np.unique(oc)) == {0, 1, 2, 3}
    st, ost = r.stats(), o.stats()
    assert st["tiles_by_class"] == [ost["tiles_high"], ost["tiles_low"], ost["tiles_hybrid"], ost["tiles_invisible"]]
    assert st["samples"] == ost["samples"] and st["work_items"] == ost["work_items"]


def test_front_end_statistics(vrs, oracle_mod):
    """vrs_frame_stats' front-end counters (the units of bench.py's per-stage
    HBM roofline) obey their definitions: every Gaussian with a pair passed the
    conservative cone cull for some view, candidates are (view, Gaussian) with
    1 <= views per Gaussian <= n_views, every visible (view, Gaussian) was a
    candidate, every pair was a tested tile; masked and unmasked views alike."""
    scene = sg.vr_room(7, 20000, sh_degree=1)
    W, H = 320, 256
    f = sg.focal_for_hfov(W, 110.0)
    for masked in (True, False):
        cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e if masked else -1)
                for e, x in enumerate((-0.0315, 0.0315))]
        masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)} if masked else None
        r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, None, T=16, masks=masks)
        assert_lists_equal(r, o)
        st = r.stats()
        k, v = r.vrs_debug_pairs(True)
        assert 0 < st["frustum_gaussians"] <= scene.n
        assert st["frustum_gaussians"] <= st["candidates"] <= 2 * st["frustum_gaussians"]
        assert len(np.unique(v)) <= st["frustum_gaussians"]
        assert st["visible_splats"] <= st["candidates"]
        assert st["pairs"] <= st["tile_tests"]
        assert st["pairs"] == len(k) == o.stats()["pairs"]


@pytest.mark.parametrize("W,H,T", [(37, 29, 16), (65, 33, 32), (16, 16, 16), (1, 1, 16), (300, 17, 32)])
def test_odd_sizes_and_edges(vrs, oracle_mod, W, H, T):
    """Ragged image borders (partial tiles, odd widths, 1x1)."""
    scene = sg.random_scene(11, n=600, sh_degree=1, xy_frac=1.2)
    cam = identity_camera(W, H, max(W, H) * 0.6)
    fov = [sg.Fovea((W / 2, H / 2), (W / 5 + 1, H / 5 + 1), 0.2)] if T == 32 else None
    r, o, g, oi = render_both(vrs, oracle_mod, scene, [cam], fov, T=T)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)


def test_empty_and_fully_culled_scenes(vrs, oracle_mod):
    cam = identity_camera(64, 48, 40.0)
    # empty scene
    r, o, g, oi = render_both(vrs, oracle_mod, scene_from(np.zeros((0, 3)), 0.1), [cam])
    assert np.all(g[0][0][..., 3] == 0) and np.all(g[0][1] == 0)
    # everything behind the camera
    sc = scene_from(np.array([[0, 0, -3.0], [1, 1, -2.0]]), 0.2)
    r, o, g, oi = render_both(vrs, oracle_mod, sc, [cam])
    assert r.stats()["pairs"] == 0
    assert_images_close(g, oi)


def test_max_gaussian_index_parity(vrs, oracle_mod):
    """The largest scene the context accepts (max_gaussians = 2^24 - 1: the
    blend stages a Gaussian index in 24 bits beside its 8-warp mask): all but
    1500 Gaussians sit behind the camera, the visible ones carry the highest
    indices (and one has index 0); pairs bit-exact, images within tolerance."""
    n = (1 << 24) - 1
    vis = sg.random_scene(7, n=1500, sh_degree=0)
    means = np.zeros((n, 3), np.float32)
    means[:, 2] = -5.0
    quats = np.zeros((n, 4), np.float32)
    quats[:, 0] = 1.0
    log_scales = np.full((n, 3), np.log(0.05), np.float32)
    logits = np.zeros(n, np.float32)
    sh = np.zeros((n, 1, 3), np.float32)
    idx = np.concatenate([[0], np.arange(n - 1499, n)])
    means[idx], quats[idx], log_scales[idx] = vis.means, vis.quats, vis.log_scales
    logits[idx], sh[idx] = vis.logits, vis.sh
    scene = sg.RawScene(means, quats, log_scales, logits, sh, 0)
    cam = identity_camera(128, 96, 64.0)
    r, o, g, oi = render_both(vrs, oracle_mod, scene, [cam])
    assert r.stats()["visible_splats"] > 1000
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    k, v = r.vrs_debug_pairs(True)
    assert v.max() >= n - 1499 and v.min() == 0


@pytest.mark.parametrize("seed", list(range(100, 110)))
def test_tiny_scenes_parity(vrs, oracle_mod, seed):
    sc, cam = tiny_set(seed)
    r, o, g, oi = render_both(vrs, oracle_mod, sc, [cam])
    assert_lists_equal(r, o)
    assert_images_close(g, oi)


def test_window_overflow_parity(vrs, oracle_mod):
    """Depth complexity >> K = 16: window overflows must match exactly (same pops)."""
    rs = np.random.default_rng(1)
    n = 300
    means = np.stack([rs.uniform(-0.3, 0.3, n), rs.uniform(-0.3, 0.3, n), rs.uniform(3, 3.6, n)], 1)
    sc = scene_from(means, [0.4, 0.4, 0.03], opacities=0.05)
    sc.quats[:] = np.stack([np.ones(n), rs.normal(0, 0.6, n), rs.normal(0, 0.6, n), np.zeros(n)], 1)
    cam = identity_camera(64, 64, 48.0)
    r, o, g, oi = render_both(vrs, oracle_mod, sc, [cam])
    st, ost = r.stats(), o.stats()
    assert ost["overflow_samples"] > 100
    assert st["overflow_samples"] == ost["overflow_samples"]
    assert st["contributions"] == ost["contributions"]
    assert_images_close(g, oi)


def test_warp_culling_never_changes_results(vrs, oracle_mod):
    """P12: the warp-block footprint skip changes work, never results (bit-identical)."""
    scene = sg.vr_room(3, 20000)
    W, H = 256, 192
    cams = sg.stereo_pair(width=W, height=H, masks=False)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    outs = []
    for nc in (False, True):
        r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H,
                         assign_tile=32)
        r.upload(scene)
        r.vrs_set_instrumentation(counters=0, no_cull=nc)
        rgba, depth = r.render(cams, fov)
        torch.cuda.synchronize()
        outs.append((rgba.cpu().numpy(), depth.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def _needle_scene(seed, n):
    """Thin needles (one long axis, two ~100x shorter) and sheets at random
    orientations, some close to the camera: the ellipses whose bounding boxes
    are loose, where the footprint's separating axis culls most."""
    base = sg.random_scene(seed, n=n, sh_degree=1, z_range=(0.6, 6.0), xy_frac=1.4)
    rs = np.random.default_rng(seed)
    ls = np.log(rs.uniform(0.001, 0.006, (n, 3)))
    ls[:, 0] = np.log(rs.uniform(0.05, 0.6, n))
    sheet = rs.random(n) < 0.3
    ls[sheet, 1] = np.log(rs.uniform(0.05, 0.4, int(sheet.sum())))
    return sg.RawScene(base.means, base.quats, ls.astype(np.float32), base.logits, base.sh, base.sh_degree)


@pytest.mark.parametrize("case", ["foveated_t32", "full_t16_wide", "tma", "hier"])
def test_footprint_axis_never_changes_results(vrs, oracle_mod, case):
    """P12 for the footprint's separating axis (record slot 7): needle and
    sheet splats at random orientations, 110-150 deg stereo; every warp-skip
    variant (thread / TMA staging, flat / hierarchical resort) renders the same
    bytes and the same counters with and without the skip, and the oracle's
    counters."""
    scene = _needle_scene(11, 6000)
    W, H = 320, 256
    hfov = 150.0 if case == "full_t16_wide" else 110.0
    T = 16 if case == "full_t16_wide" else 32
    cams = sg.stereo_pair(width=W, height=H, hfov_deg=hfov, masks=False)
    fov = None if case == "full_t16_wide" else [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    outs = []
    for nc in (False, True):
        r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H,
                         assign_tile=T)
        r.upload(scene)
        r.vrs_set_instrumentation(counters=1, no_cull=nc)
        if case == "tma":
            r.vrs_set_staging_mode(1)
        if case == "hier":
            r.vrs_set_resort_mode(1)
        rgba, depth = r.render(cams, fov)
        torch.cuda.synchronize()
        outs.append((rgba.cpu().numpy(), depth.cpu().numpy(), r.stats()))
        r.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    for k in ("contributions", "overflow_samples", "terminated_samples"):
        assert outs[0][2][k] == outs[1][2][k], k
    if case in ("foveated_t32", "full_t16_wide"):
        o = oracle_mod.Oracle(scene)
        o.prepare(cams, fov, assign_tile=T)
        o.render()
        ost = o.stats()
        for k in ("pairs", "contributions", "overflow_samples", "terminated_samples"):
            assert outs[0][2][k] == ost[k], (k, outs[0][2][k], ost[k])


@pytest.mark.parametrize("cap", [64, 128])
def test_binned_sort_merge_path_parity(vrs, oracle_mod, cap):
    """Binned sort: tiles larger than the shared-memory capacity are sorted in
    chunks and merged in global memory; forcing a tiny capacity sends most
    tiles of a dense foveated stereo frame through that path -- sorted pairs,
    ranges and images must still equal the oracle's exactly."""
    scene = sg.vr_room(8, 20000, sh_degree=1)
    W, H = 256, 192
    cams = sg.stereo_pair(width=W, height=H, masks=False)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    r.vrs_debug_set_sort_smem_cap(cap)
    rgba, depth = r.render(cams, fov)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene)
    o.prepare(cams, fov, assign_tile=32)
    rng = o.ranges()
    assert (rng[:, 1] - rng[:, 0]).max() > 2 * cap, "test needs tiles spanning several merge rounds"
    k, v = r.vrs_debug_pairs(True)
    ok, ov = o.pairs(True)
    assert np.array_equal(k, ok) and np.array_equal(v, ov)
    assert np.array_equal(r.vrs_debug_ranges(), rng)
    g = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), cams)
    assert_images_close(g, o.render())
    with pytest.raises(Exception):
        r.vrs_debug_set_sort_smem_cap(100)  # not a power of two


def test_determinism(vrs):
    """P14: two renders are byte-identical."""
    scene = sg.vr_room(4, 30000)
    W, H = 256, 256
    cams = sg.stereo_pair(width=W, height=H, masks=False)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    a = [t.cpu().numpy() for t in r.render(cams, fov)]
    b = [t.cpu().numpy() for t in r.render(cams, fov)]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_large_fov_identity_gpu(vrs):
    """P13 on the CUDA path: crop of the 3x render equals the 1x render bit for bit."""
    sc = sg.random_scene(6, n=800, z_range=(1.5, 6.0), xy_frac=2.0)
    W, H = 64, 48
    small = identity_camera(W, H, 40.0)
    large = identity_camera(3 * W, 3 * H, 40.0, cx=small.cx + W, cy=small.cy + H)
    outs = []
    for cam in (small, large):
        r = vrs.Renderer(max_gaussians=sc.n, max_views=1, max_pairs=1 << 20, max_width=cam.width,
                         max_height=cam.height, assign_tile=16)
        r.upload(sc)
        rgba, depth = r.render([cam])
        outs.append(vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), [cam])[0])
    (a, ad), (b, bd) = outs
    assert np.array_equal(a, b[H:2 * H, W:2 * W]) and np.array_equal(ad, bd[H:2 * H, W:2 * W])


@pytest.mark.parametrize("n", [1, 100, 4095, 4096, 4097, 100000, 1234567])
def test_onesweep_sort_bit_exact(vrs, n):
    """Step 4: stable sort equals numpy's stable argsort (ties keep input order)."""
    rs = np.random.default_rng(n)
    tiles = rs.integers(0, 9000, n).astype(np.uint64)
    depth = rs.uniform(0.2, 40.0, n).astype(np.float32).view(np.uint32).astype(np.uint64)
    depth[rs.random(n) < 0.2] = np.uint64(0x3e4ccccd)  # many exact ties (near-clamped depths)
    keys = (tiles << np.uint64(32)) | depth
    vals = np.arange(n, dtype=np.uint32)
    r = vrs.Renderer(max_gaussians=1, max_views=1, max_pairs=max(n, 1), max_width=16, max_height=16)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    vt = torch.from_numpy(vals.view(np.int32)).cuda()
    r.vrs_sort_pairs(kt, vt, key_bits=46)
    torch.cuda.synchronize()
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(kt.cpu().numpy().view(np.uint64), keys[order])
    assert np.array_equal(vt.cpu().numpy().view(np.uint32), vals[order])


@pytest.mark.parametrize("n", [1, 17, 4096, 4097, 300001])
def test_scan_exact(vrs, n):
    rs = np.random.default_rng(n)
    x = rs.integers(0, 50, n).astype(np.uint32)
    r = vrs.Renderer(max_gaussians=n, max_views=1, max_pairs=16, max_width=16, max_height=16)
    xt = torch.from_numpy(x.view(np.int32)).cuda()
    out = torch.empty_like(xt)
    tot = torch.zeros(1, dtype=torch.int32, device="cuda")
    r.vrs_exclusive_scan(xt, out, tot)
    torch.cuda.synchronize()
    ref = np.concatenate([[0], np.cumsum(x)[:-1]]).astype(np.uint32)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)
    assert int(tot.cpu().numpy().view(np.uint32)[0]) == int(x.sum())


def test_host_output_path_matches_device_path(vrs):
    scene = sg.random_scene(2, n=1000)
    cam = sg.look_camera((0, 0, 0), f=64.0, width=128, height=96)
    r = vrs.Renderer(max_gaussians=1000, max_views=1, max_pairs=1 << 16, max_width=128, max_height=96)
    r.upload(scene)
    rgba, depth = r.render([cam])
    torch.cuda.synchronize()
    hr, hd = r.render_host([cam])
    assert np.array_equal(rgba.cpu().numpy(), hr) and np.array_equal(depth.cpu().numpy(), hd)


def test_invalid_camera_rejected(vrs):
    r = vrs.Renderer(max_gaussians=10, max_views=1, max_pairs=100, max_width=64, max_height=64)
    r.upload(scene_from([[0, 0, 3]], 0.1))
    cam = identity_camera(64, 64, 32.0)
    cam.R_wc = cam.R_wc * 1.01
    with pytest.raises(vrs.VrsError) as e:
        r.render([cam])
    assert e.value.status == vrs.vrs.VRS_E_INVALID_ARG
    big = identity_camera(128, 64, 32.0)
    with pytest.raises(vrs.VrsError):
        r.render([big])


def test_capacity_overflow_reported(vrs):
    scene = sg.random_scene(0, n=1000)
    cam = sg.look_camera((0, 0, 0), f=64.0, width=128, height=128)
    r = vrs.Renderer(max_gaussians=1000, max_views=1, max_pairs=500, max_width=128, max_height=128)
    r.upload(scene)
    r.render([cam])
    with pytest.raises(vrs.VrsError) as e:
        r.stats()
    assert e.value.status == vrs.vrs.VRS_E_CAPACITY


def _quest_workload(seed, n, scale_mul, fovea, T, masks):
    scene = sg.vr_room(seed, n, scale_mul=scale_mul, sh_degree=3)
    cams = sg.stereo_pair(masks=masks)
    fov = [sg.quest_fovea()] * 2 if fovea else None
    mk = {0: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H), 1: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H)} if masks else {}
    return scene, cams, fov, mk


def test_c2_full_size_parity(vrs, oracle_mod):
    """Config C2 at full size, in bench.py's launch configuration: 500k SH3,
    stereo 2x2064x2208, 110 deg, foveated, masks, T_a = 32.  Pair list, ranges
    and per-splat counts bit-exact; EVERY output pixel of both eyes within the
    tolerances; workload counters equal."""
    scene, cams, fov, mk = _quest_workload(2, 500_000, 1.0, True, 32, True)
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, masks=mk, max_pairs=6 << 20)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    st, ost = r.stats(), o.stats()
    for k in ("pairs", "samples", "evaluations", "contributions", "overflow_samples", "terminated_samples",
              "work_items", "visible_splats"):
        assert st[k] == ost[k], (k, st[k], ost[k])


def test_c3_full_size_parity(vrs, oracle_mod):
    """Config C3 at full size, in bench.py's launch configuration (3M
    Gaussians, stereo 2x2064x2208, no foveation, T_a = 16): pair list, ranges
    and per-splat counts bit-exact; EVERY output pixel of both eyes within the
    tolerances; workload counters equal."""
    scene, cams, fov, mk = _quest_workload(3, 3_000_000, (1 / 6) ** 0.5, False, 16, False)
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, None, T=16, max_pairs=16 << 20)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    st, ost = r.stats(), o.stats()
    for k in ("pairs", "samples", "evaluations", "contributions", "overflow_samples", "terminated_samples",
              "work_items", "visible_splats"):
        assert st[k] == ost[k], (k, st[k], ost[k])


# --------------------------------------------------------------------- EWA baseline (config C5)

@pytest.mark.parametrize("seed", [0, 3])
def test_ewa_parity_small(vrs, oracle_mod, seed):
    """EWA baseline mode (config C5's comparison): pairs bit-exact, images within tolerance."""
    scene = sg.random_scene(seed, n=1000, sh_degree=3, xy_frac=1.5)
    cam = sg.look_camera((0, 0, 0), f=48.0, width=160, height=128)
    r, o, g, oi = render_both(vrs, oracle_mod, scene, [cam], projection=1)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    gs, os_ = r.vrs_debug_splats(0), o.splats(0)
    valid = os_[:, 0] == 1
    assert np.array_equal(gs[:, 0], os_[:, 0])
    assert np.array_equal(gs[valid][:, 20:25], os_[valid][:, 20:25])


@pytest.mark.parametrize("hfov", [90.0, 160.0])
def test_ewa_wide_fov_foveated_stereo(vrs, oracle_mod, hfov):
    """C5-style FoV sweep end points on a reduced vr_room, OP and EWA, foveated stereo."""
    scene = sg.vr_room(5, 30000, sh_degree=3)
    W, H = 256, 256
    cams = sg.stereo_pair(width=W, height=H, hfov_deg=hfov, masks=False)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    for proj in (0, 1):
        r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, projection=proj)
        assert_lists_equal(r, o)
        assert_images_close(g, oi)


@pytest.mark.parametrize("W,H,seed", [(320, 256, 13), (333, 251, 14)])
def test_two_pass_baseline_parity(vrs, oracle_mod, W, H, seed):
    """SURVEY §8f N1 (App. A): the two-pass foveated baseline through the C
    ABI against oracle/twopass.py -- stereo, visibility masks (pass 2 only,
    2x2-OR reduced), odd sizes; the 4-view pass frame's sorted pair list and
    ranges bit-exact, every output pixel within the tolerances."""
    from oracle import twopass as tpo
    scene = sg.vr_room(seed, 20000, sh_degree=3)
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
            for e, x in enumerate((-0.0315, 0.0315))]
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10), sg.Fovea((W / 2 + 7.3, H / 2 - 5.1), (W / 5, H / 4), 0.2)]
    masks = {0: sg.ellipse_mask(W, H), 1: sg.ellipse_mask(W, H, 1.0)}
    r = vrs.Renderer(max_gaussians=scene.n, max_views=4, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    for s, m in masks.items():
        r.set_mask(s, m)
    rgba, depth = r.render_two_pass(cams, fov)
    torch.cuda.synchronize()
    g = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), cams)
    out, o = tpo.render_two_pass(oracle_mod, scene, cams, fov, masks=masks, assign_tile=32)
    k, v = r.vrs_debug_pairs(True)
    ok, ov = o.pairs(True)
    assert np.array_equal(k, ok) and np.array_equal(v, ov)
    assert np.array_equal(r.vrs_debug_ranges(), o.ranges())
    assert_images_close(g, [(c.astype(np.float32), d.astype(np.float32)) for c, d in out])
    # the second render reuses the cached half masks and per-eye setup
    rgba2, depth2 = r.render_two_pass(cams, fov)
    assert torch.equal(rgba, rgba2) and torch.equal(depth, depth2)


@pytest.mark.parametrize("cap", [4096, 128])
def test_binned_sort_tile_overflow_parity(vrs, oracle_mod, cap):
    """Binned sort with tiles holding more pairs than their direct bucket
    (kTileCap = 1024 slots): the overflow pairs take the overflow list and are
    merged back per tile -- sorted pairs, ranges and images equal the oracle's
    (also with the merge path forced by a small shared-memory capacity)."""
    rng = np.random.default_rng(21)
    n = 5000
    means = np.column_stack([rng.normal(0, 0.05, n), rng.normal(0, 0.05, n), rng.uniform(2.0, 4.0, n)])
    scene = scene_from(means, np.exp(rng.uniform(np.log(0.01), np.log(0.05), (n, 3))),
                       opacities=rng.uniform(0.05, 0.6, n), dc=rng.normal(0, 0.5, (n, 3)))
    cam = identity_camera(96, 64, 200.0)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=1, max_pairs=1 << 20, max_width=96, max_height=64,
                     assign_tile=16)
    r.upload(scene)
    r.vrs_debug_set_sort_smem_cap(cap)
    rgba, depth = r.render([cam])
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene).prepare([cam], assign_tile=16)
    rng_o = o.ranges()
    assert (rng_o[:, 1] - rng_o[:, 0]).max() > 2048, "test needs tiles past the direct bucket capacity"
    k, v = r.vrs_debug_pairs(True)
    ok, ov = o.pairs(True)
    assert np.array_equal(k, ok) and np.array_equal(v, ov)
    assert np.array_equal(r.vrs_debug_ranges(), rng_o)
    g = vrs.vrs.split_views(rgba.cpu().numpy(), depth.cpu().numpy(), [cam])
    assert_images_close(g, o.render())


# --------------------------------------------------------------------- packed display output format

def _pack_ref(rgba, depth):
    q = np.rint(np.clip(rgba, 0.0, 1.0).astype(np.float32) * np.float32(255.0)).astype(np.uint8)
    return q, depth.astype(np.float16)


@pytest.mark.parametrize("mode", ["single", "two_pass", "hier", "host"])
def test_packed_output_is_the_quantised_f32_frame(vrs, mode):
    """VRS_OUT_RGBA8_D16F writes round(clamp(v,0,1)*255) and binary16 of the
    very float values the F32 format writes (bit-exact), on every path."""
    W, H = 320, 256
    scene = sg.vr_room(7, 20000, sh_degree=3)
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.3, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
            for e, x in enumerate((-0.0315, 0.0315))]
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.10)] * 2
    r = vrs.Renderer(max_gaussians=scene.n, max_views=4, max_pairs=1 << 22, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    for e in range(2):
        r.set_mask(e, sg.ellipse_mask(W, H))
    if mode == "hier":
        r.vrs_set_resort_mode(1)
    fn = r.render_two_pass if mode == "two_pass" else r.render

    def run():
        if mode == "host":
            a, d = r.vrs_render_views_host(cams, fov)
            return np.asarray(a).copy(), np.asarray(d).copy()
        a, d = fn(cams, fov)
        torch.cuda.synchronize()
        return a.cpu().numpy(), d.cpu().numpy()

    a32, d32 = run()
    r.vrs_set_output_format(1)
    a8, d16 = run()
    assert a8.dtype == np.uint8 and d16.dtype == np.float16
    qa, qd = _pack_ref(a32, d32)
    assert np.array_equal(a8, qa)
    assert np.array_equal(d16.view(np.uint16), qd.view(np.uint16))
    with pytest.raises(vrs.vrs.VrsError):
        r.vrs_set_output_format(7)


# --------------------------------------------------------------------- more full-size and maximum-size cases

@pytest.mark.parametrize("t", [45, 300])
def test_c4_trajectory_pose_full_size_parity(vrs, oracle_mod, t):
    """Config C4 at full size at two trajectory poses (1M Gaussians, scales x0.707,
    foveated, masks, T_a = 32): sorted pair list and ranges bit-exact, EVERY
    output pixel of both eyes within tolerance, workload counters equal."""
    scene = sg.vr_room(4, 1_000_000, scale_mul=0.707, sh_degree=3)
    head, yaw, pitch, roll = sg.trajectory_pose(t)
    cams = sg.stereo_pair(head, yaw, pitch, roll, masks=True)
    fov = [sg.quest_fovea()] * 2
    mk = {0: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H), 1: sg.ellipse_mask(sg.QUEST_W, sg.QUEST_H)}
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, masks=mk, max_pairs=8 << 20)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    st, ost = r.stats(), o.stats()
    for k in ("pairs", "samples", "evaluations", "contributions", "terminated_samples"):
        assert st[k] == ost[k], (k, st[k], ost[k])


def test_c5_ewa_160_full_size_parity(vrs, oracle_mod):
    """Config C5's widest point at full size: C2 scene, 160 deg, EWA baseline
    (footprints blow up): lists bit-exact, EVERY pixel in tolerance."""
    scene = sg.vr_room(2, 500_000, scale_mul=1.0, sh_degree=3)
    cams = sg.stereo_pair(hfov_deg=160.0, masks=False)
    fov = [sg.quest_fovea()] * 2
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32, max_pairs=8 << 20, projection=1)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)


def test_maximum_views_in_one_call(vrs, oracle_mod):
    """VRS_MAX_VIEWS = 8 views (4 stereo pairs at different head poses) in one
    frame: one sort and one blend over all of them, every pixel compared."""
    W, H = 192, 160
    scene = sg.vr_room(21, 20000, sh_degree=2)
    f = sg.focal_for_hfov(W, 110.0)
    cams = []
    for t in (0, 30, 60, 90):
        head, yaw, pitch, roll = sg.trajectory_pose(t)
        cams += sg.stereo_pair(head, yaw, pitch, roll, width=W, height=H, masks=False)
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 8
    r, o, g, oi = render_both(vrs, oracle_mod, scene, cams, fov, T=32)
    assert_lists_equal(r, o)
    assert_images_close(g, oi)
    assert r.stats()["work_items"] > 0


@pytest.mark.parametrize("cap", [512, 1024, 2048])
def test_binned_sort_run_merge_parity(vrs, oracle_mod, cap):
    """Big tiles: chunks of up to `cap` keys are sorted as 256-key register runs
    merged in shared memory (2048 = the default), larger tiles additionally
    merged in global memory -- sorted pairs and ranges equal the oracle's."""
    scene = sg.vr_room(12, 400_000, scale_mul=1.5, sh_degree=0)
    W, H = 256, 192
    cams = sg.stereo_pair(width=W, height=H, masks=False)
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 23, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    if cap != 2048:
        r.vrs_debug_set_sort_smem_cap(cap)
    rgba, depth = r.render(cams, None)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(scene)
    o.prepare(cams, None, assign_tile=32)
    rng = o.ranges()
    sizes = rng[:, 1] - rng[:, 0]
    assert sizes.max() > 2 * cap and (sizes > 256).sum() > 10, "test needs big tiles"
    k, v = r.vrs_debug_pairs(True)
    ok, ov = o.pairs(True)
    assert np.array_equal(k, ok) and np.array_equal(v, ov)
    assert np.array_equal(r.vrs_debug_ranges(), rng)


def test_frame_is_cuda_graph_capturable(vrs):
    """A frame (both streams, every kernel) captured into a CUDA graph by
    stream capture and replayed gives the directly rendered frame bit for bit
    (per-eye setup cached beforehand: a setup cache miss synchronises)."""
    W, H = 256, 192
    scene = sg.vr_room(9, 20000, sh_degree=3)
    f = sg.focal_for_hfov(W, 110.0)
    cams = [sg.look_camera((x, 0, 0), 0.2, 0.1, 0.0, f=f, width=W, height=H, mask_slot=e)
            for e, x in enumerate((-0.0315, 0.0315))]
    fov = [sg.Fovea((W / 2, H / 2), (W / 4, H / 4), 0.1)] * 2
    r = vrs.Renderer(max_gaussians=scene.n, max_views=2, max_pairs=1 << 21, max_width=W, max_height=H,
                     assign_tile=32)
    r.upload(scene)
    for e in range(2):
        r.set_mask(e, sg.ellipse_mask(W, H))
    rgba, depth = r.alloc_outputs(cams)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        r.render(cams, fov, rgba, depth, stream=s)
    torch.cuda.synchronize()
    ref_rgba, ref_depth = rgba.clone(), depth.clone()
    rgba.zero_()
    depth.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        r.render(cams, fov, rgba, depth, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(rgba, ref_rgba) and torch.equal(depth, ref_depth)
