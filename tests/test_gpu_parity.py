"""GPU parity: the B200 render path (through the C-ABI) against the CPU oracle on the same
seeded inputs — the reference's scene fixtures (test_renderer.cpp:13-37,
test_crowd.cpp:14-44), BASELINE configs 1-3 at full size, and the edge cases the
reference tests (empty crowd, culling, tile sizes 1..40, static pose, forced LoD,
hysteresis, footprint locality, determinism)."""
import numpy as np
import pytest

import paper_2501_17792_b200 as P
from oracle import orc
from tests.parity import check_cull_invariance, check_frame, render_both

pytestmark = pytest.mark.gpu


def fixture_scene(count=4, rows=2, cols=2, seed=42, sh=False):
    cfg = P.SceneConfig(template_count=1, template_seed_base=1, level_counts=(80, 30, 12), with_sh=sh,
                        motion_count=1, motion_seed_base=2, motion_frames=24, grid_rows=rows, grid_cols=cols,
                        grid_spacing=1.2, crowd_count=count, crowd_seed=seed, cam_pos=(0.6, 1.5, -3.5),
                        cam_look=(0.6, 1.0, 2.0), width=200, height=120)
    return P.Scene(cfg)


def basic_scene(count=16, rows=4, cols=4, seed=77, templates=2, motions=3, sh=True):
    cfg = P.SceneConfig(template_count=templates, level_counts=(60, 24, 8), with_sh=sh, motion_count=motions,
                        motion_frames=24, grid_rows=rows, grid_cols=cols, crowd_count=count, crowd_seed=seed,
                        cam_pos=(0.0, 1.6, -3.0), cam_look=(0.0, 1.0, 5.0), width=160, height=90)
    return P.Scene(cfg)


def parity(scene, time_s=0.0, **kw):
    r = P.Renderer(scene)
    o = orc.from_scene(scene)
    g, c = render_both(scene, r, o, time_s, **kw)
    return check_frame(scene, r, o, g, c, tile_size=kw.get("tile_size", 16))


@pytest.mark.parametrize("time_s", [0.0, 0.37, 1.3])
def test_fixture_scene(time_s):
    parity(fixture_scene(), time_s, background=(0.1, 0.1, 0.15))


@pytest.mark.parametrize("tile_size", [1, 3, 8, 16, 17, 32, 40])
def test_tile_sizes(tile_size):
    parity(fixture_scene(9, 3, 3, seed=55), 0.37, tile_size=tile_size, background=(0.2, 0.4, 0.6))


def test_crowd_with_sh_and_lod_mix():
    rep = parity(basic_scene(), 0.7, background=(0.05, 0.05, 0.05))
    assert rep["S"] > 0


@pytest.mark.parametrize("forced", [0, 1, 2, 5])
def test_forced_lod(forced):
    parity(basic_scene(sh=False), 0.4, forced_lod=forced)


def test_static_pose():
    parity(basic_scene(), 0.0, static_pose=True, background=(0.3, 0.2, 0.1))


def test_empty_crowd_is_background():
    s = basic_scene()
    s.instances = s.instances[:0]
    r = P.Renderer(s)
    rgb, T = r.render_frame(0.0, P.RenderSettings(background=(0.2, 0.4, 0.6)))
    assert np.all(rgb == np.array([0.2, 0.4, 0.6], np.float32)) and np.all(T == 1.0)
    assert r.counts() == (0, 0, 0)


def test_culled_instances_behind_and_offscreen():
    s = basic_scene(count=4, rows=2, cols=2)
    inst = s.instances
    inst["z"] = [-10.0, -3.0, 5.0, 500.0]   # behind, at the camera plane, visible, far
    inst["x"] = [0.0, 0.0, 60.0, 0.0]        # the visible-depth one is far off-screen sideways
    s.instances = inst
    rep = parity(s, 0.2)
    assert rep["S"] < rep["G"]
    r = P.Renderer(s)
    assert check_cull_invariance(r, 0.2) >= 2  # the one behind and the one far sideways


def test_hysteresis_across_frames():
    s = basic_scene(count=4, rows=1, cols=4, sh=False)
    s.set_lod_policy((3.0, 6.0), hysteresis=1.0)
    r = P.Renderer(s)
    o = orc.from_scene(s)
    o.set_lod((3.0, 6.0), 1.0)
    for z in (-0.5, 0.0, 0.3, 0.6, 0.3, -0.2, 3.0, 3.4, 2.8, 3.2):
        s.set_camera((0.0, 1.6, -3.0 - z), (0.0, 1.0, 5.0))
        o.set_camera((0.0, 1.6, -3.0 - z), (0.0, 1.0, 5.0), 50.0, 160, 90)
        g, c = render_both(s, r, o, 0.1)
        check_frame(s, r, o, g, c)
        assert np.array_equal(s.instances["active_lod"], r.lods())


def test_static_equals_motion_on_bind_pose_clip():
    s = fixture_scene(4, 2, 2, seed=5)
    clip = np.zeros((1, 4 + 96), np.float32)
    clip[0, 7::4] = 1.0
    s.set_motion(0, 1.0, clip, 24)
    r = P.Renderer(s)
    a, _ = r.render_frame(0.0, P.RenderSettings(), static_pose=False)
    b, _ = r.render_frame(0.0, P.RenderSettings(), static_pose=True)
    assert a.tobytes() == b.tobytes()


def test_moving_one_instance_changes_only_its_footprint():
    near = fixture_scene(4, 2, 2, seed=9)
    far = fixture_scene(4, 2, 2, seed=9)
    inst = far.instances
    inst["z"][1] += 9.0
    far.instances = inst
    st = P.RenderSettings(background=(0.05, 0.05, 0.05))
    rn, rf = P.Renderer(near), P.Renderer(far)
    box = [10 ** 9, 10 ** 9, -1, -1]
    imgs = []
    for s, r in ((near, rn), (far, rf)):
        r.set_debug(2)
        img, _ = r.render_frame(0.2, st)
        imgs.append(img)
        rec = r.splat_records()
        mine = rec[rec["instance_id"] == 1]
        box = [min(box[0], mine["rect"][:, 0].min()), min(box[1], mine["rect"][:, 1].min()),
               max(box[2], mine["rect"][:, 2].max()), max(box[3], mine["rect"][:, 3].max())]
    diff = np.any(imgs[0] != imgs[1], axis=2)
    ys, xs = np.nonzero(diff)
    assert len(xs) > 0
    assert (xs >= box[0]).all() and (xs < box[2]).all() and (ys >= box[1]).all() and (ys < box[3]).all()


def test_long_equal_depth_runs_are_ordered_by_ordinal():
    """Stacked same-pose characters give every template Gaussian one depth per stack, so
    every cell holds runs of equal (cell, depth) pairs of each stack's size: <= 32
    (k_cell_fixup, shared memory), <= 2048 (k_pair_long_runs, shared-memory bitonic) and
    beyond (k_pair_long_runs, global bitonic). The reference orders ties by (instance,
    gaussian) (renderer.cpp:91-96)."""
    cfg = P.SceneConfig(template_count=1, template_seed_base=5, level_counts=(24, 12, 6), with_sh=False,
                        motion_count=1, motion_frames=8, grid_rows=1, grid_cols=1, crowd_count=1, crowd_seed=1,
                        cam_pos=(0.0, 1.0, -4.0), cam_look=(0.0, 1.0, 6.0), width=160, height=96)
    s = P.Scene(cfg)
    proto = s.instances[:1]
    stacks = [5, 33, 200, 257, 1500, 4097, 5000]
    inst = np.concatenate([np.repeat(proto, n) for n in stacks])
    inst["instance_id"] = np.arange(len(inst))
    inst["yaw"] = 0.0
    inst["phase_offset_s"] = 0.0
    inst["x"] = np.concatenate([np.full(n, -1.2 + 0.4 * g, np.float32) for g, n in enumerate(stacks)])
    inst["z"] = np.concatenate([np.full(n, 0.25 * g, np.float32) for g, n in enumerate(stacks)])
    rng = np.random.default_rng(5)
    inst = inst[rng.permutation(len(inst))]  # stacks interleaved in instance order
    inst["instance_id"] = np.arange(len(inst))
    s.instances = inst
    rep = parity(s, 0.0, static_pose=True, forced_lod=0)
    assert rep["S"] > 0
    # the runs really are long: one depth value per (stack, gaussian)
    r = P.Renderer(s)
    r.set_debug(2)
    r.render_frame(0.0, P.RenderSettings(), True, 0)
    _, run_len = np.unique(r.splat_records()["depth"], return_counts=True)
    assert run_len.max() >= 4097


@pytest.mark.parametrize("bits", [6, 12, 18])
def test_truncated_depth_sort_is_exact(bits, monkeypatch):
    """The splat sort orders only the top GSCG_DEPTH_SORT_BITS varying depth bits; the
    per-cell fix-up restores the full (depth bits, instance, gaussian) order. Few sorted
    bits make most pairs tie inside their cells (long runs through k_pair_long_runs),
    and every per-cell list must still equal the oracle's bins."""
    monkeypatch.setenv("GSCG_DEPTH_SORT_BITS", str(bits))
    rep = parity(basic_scene(count=48, rows=6, cols=8), 0.6)
    assert rep["K"] > 0


@pytest.mark.parametrize("bits", [25, 12])
def test_lsd_depth_sort_is_exact(bits, monkeypatch):
    """Frames past GSCG_BUCKET_MAX_SPLATS (config 5) take the LSD depth passes instead of
    the bucket sort; forced here on a small crowd, both must give the oracle's bins."""
    monkeypatch.setenv("GSCG_BUCKET_MAX_SPLATS", "0")
    monkeypatch.setenv("GSCG_DEPTH_SORT_BITS", str(bits))
    rep = parity(basic_scene(count=48, rows=6, cols=8), 0.6)
    assert rep["K"] > 0


def test_bucket_sort_large_buckets_are_exact(monkeypatch):
    """Config 2 sorted on 14 depth bits: 3.3 M splats in at most 16,384 buckets, thousands
    per bucket where the crowd is dense, so the bucket sort's multi-chunk coalesced and
    streamed local paths both run; every per-cell list must still equal the oracle's."""
    monkeypatch.setenv("GSCG_DEPTH_SORT_BITS", "14")
    s, extra = config_scene(2, sh=False)
    rep = parity(s, extra["time_s"], forced_lod=extra["forced_lod"])
    assert rep["S"] > 3_000_000


def test_repeated_frames_are_byte_identical():
    s = basic_scene(count=16)
    r = P.Renderer(s)
    outs = [r.render_frame(0.55, P.RenderSettings())[0].tobytes() for _ in range(3)]
    assert outs[0] == outs[1] == outs[2]


def test_pinned_output_matches_fresh_arrays():
    scene = basic_scene()
    r1, r2 = P.Renderer(scene), P.Renderer(scene)
    st = P.RenderSettings(background=(0.2, 0.1, 0.0))
    rgb, T = r1.render_frame(0.5, st)
    out = r2.alloc_frame(pinned=True)
    rgb2, T2 = r2.render_frame(0.5, st, out=out)
    assert rgb2 is out[0] and T2 is out[1]
    assert rgb.tobytes() == rgb2.tobytes() and T.tobytes() == T2.tobytes()
    with pytest.raises(ValueError):
        r2.render_frame(0.5, st, out=(out[0][:, :-1], out[1]))
    out[0][:] = 0
    rgb3, T3 = r2.render_frame(0.5, st, out=(out[0], None))  # colour only, as the reference render_frame
    assert T3 is None and rgb3.tobytes() == rgb.tobytes()


@pytest.mark.parametrize("which", ["basic", "config2"])
def test_pipelined_frames_match_synchronous(which):
    """render_frame(pipelined=True) (gscg_render_frame_async): frame k's read-back runs
    while frame k+1 renders into the second device framebuffer; every frame equals the
    synchronous render."""
    s = basic_scene(count=16) if which == "basic" else P.Scene(P.baseline_config(2)[0])
    st = P.RenderSettings()
    times = [0.1, 0.45, 0.8, 1.15, 1.5]
    sync = P.Renderer(s)
    ref = [tuple(a.copy() for a in sync.render_frame(t, st)) for t in times]
    r = P.Renderer(s)
    bufs = [r.alloc_frame(pinned=True), r.alloc_frame(pinned=True)]
    got = []
    for k, t in enumerate(times):
        r.render_frame(t, st, out=bufs[k % 2], pipelined=True)
        if k:
            r.wait_readback(1)
            got.append(tuple(a.copy() for a in bufs[(k - 1) % 2]))
    r.wait_readback(0)
    got.append(tuple(a.copy() for a in bufs[(len(times) - 1) % 2]))
    for (a, b), (c, d) in zip(got, ref):
        assert a.tobytes() == c.tobytes() and b.tobytes() == d.tobytes()
    # a synchronous frame after pipelined ones still returns its own image
    again = r.render_frame(times[0], st)
    assert again[0].tobytes() == ref[0][0].tobytes()


def test_memory_usage_counts_the_shared_store_once():
    scene = basic_scene(count=16, templates=2, sh=True)
    r = P.Renderer(scene)
    r.render_frame(0.0)
    mu = r.memory_usage()
    expect = 0
    for t in range(2):
        for l in range(scene.level_count(t)):
            n = len(scene.level_view(t, l)["opacities"])
            expect += n * 64 + n * 16 + ((n + 255) // 256) * 256 * 45 * 4
    assert mu["template_bytes"] == expect  # independent of the 16 instances
    assert mu["frame_bytes"] > 0 and mu["device_total_bytes"] > mu["device_free_bytes"]


def test_loaded_template_reuploads_and_matches(tmp_path):
    scene = basic_scene(templates=2, sh=True)
    r = P.Renderer(scene)
    rgb0, T0 = r.render_frame(0.4)
    path = tmp_path / "t0.gsat"
    scene.save_template(1, path)
    scene.load_template(path, 0)  # slot 0 <- template 1: a new store, re-uploaded on the next frame
    rgb1, _ = r.render_frame(0.4)
    assert rgb1.tobytes() != rgb0.tobytes()
    o = orc.from_scene(scene)
    g, c = render_both(scene, r, o, 0.4)
    check_frame(scene, r, o, g, c)


def test_device_expf_replica_matches_libm_on_every_raster_argument():
    """The rasteriser's alpha = opacity * expf(power) (renderer.cpp:205) uses a device
    replica of the host libm's expf (gscg_expf.cuh). power <= 0 always, and power >=
    power_floor = log(cutoff / opacity) > -104 for any cutoff in (0, 1): every float in
    [-103.97, -0] (1.12 G values) must match the host libm bit for bit."""
    from paper_2501_17792_b200 import native as N

    r = P.Renderer(basic_scene(count=1, rows=1, cols=1))
    r.render_frame(0.0)  # creates the context
    first, last = 0x80000000, 0xC2CFF1B4
    chunk = 1 << 26
    bad = 0
    for b in range(first, last + 1, chunk):
        n = min(chunk, last + 1 - b)
        dev = np.empty(n, np.float32)
        N.check_gscg(N.gscg().gscg_eval_expf(r.gpu, b, n, dev.ctypes.data), r.gpu)
        host = orc.libm_expf_range(b, n)
        bad += int(np.count_nonzero(dev.view(np.uint32) != host.view(np.uint32)))
    assert bad == 0, f"{bad} arguments differ from the host expf"


def test_device_sinf_replica_matches_libm():
    import ctypes as C

    from paper_2501_17792_b200 import native as N

    r = P.Renderer(basic_scene())
    bits = np.arange(0, np.float32(np.pi / 2).view(np.uint32) + 1, 53, dtype=np.uint32)
    rng = np.random.default_rng(5)
    x = np.concatenate([bits.view(np.float32), rng.uniform(0, np.pi / 2, 1 << 20).astype(np.float32),
                        np.array([0.0, 1e-30, 2.4e-4, 0.785398, 0.7853982, 1.5707963, 1.5707964], np.float32)])
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    N.check_gscg(N.gscg().gscg_eval_sinf(r.gpu, x.ctypes.data, out.ctypes.data, x.size), r.gpu)
    ref = orc.libm_sinf(x)
    bad = np.nonzero(out.view(np.uint32) != ref.view(np.uint32))[0]
    assert bad.size == 0, f"{bad.size} mismatches, e.g. x={x[bad[:3]]}"


@pytest.mark.parametrize("time_s", [0.0, 0.37, 1.3, 7.9])
def test_device_pose_sampling_is_bit_identical(time_s):
    from paper_2501_17792_b200 import native as N

    scene = basic_scene(count=16, templates=2, motions=3)
    host, dev = P.Renderer(scene), P.Renderer(scene, device_poses=True)
    for r in (host, dev):
        r.set_debug(N.GSCG_DEBUG_POSED)
    a = host.render_frame(time_s)
    b = dev.render_frame(time_s)
    assert host.posed_means().tobytes() == dev.posed_means().tobytes()
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    sa = host.render_frame(time_s, static_pose=True)
    sb = dev.render_frame(time_s, static_pose=True)
    assert sa[0].tobytes() == sb[0].tobytes()


def test_device_pose_sampling_config2_against_oracle():
    cfg, extra = P.baseline_config(2)
    scene = P.Scene(cfg)
    r = P.Renderer(scene, device_poses=True)
    o = orc.from_scene(scene)
    g, c = render_both(scene, r, o, 0.73)
    check_frame(scene, r, o, g, c)


def test_lod_quality_sweep_on_device_matches_host_psnr():
    cfg = P.SceneConfig(template_count=1, template_seed_base=9, level_counts=(4000, 900, 200), with_sh=True,
                        motion_count=1, motion_frames=10, grid_rows=1, grid_cols=1, crowd_count=1,
                        width=256, height=192, fov_y_deg=45.0)
    scene = P.Scene(cfg)
    dists = [2.0, 6.0]
    rows = scene.lod_quality_sweep(0, dists)
    assert len(rows) == 6 and all(r["level"] == i % 3 for i, r in enumerate(rows))
    assert [r["gaussian_count"] for r in rows[:3]] == [4000, 900, 200]
    P.place_origin_instance(scene)
    r = P.Renderer(scene)
    for k, d in enumerate(dists):
        scene.set_camera((0.0, 0.95, -d), (0.0, 0.95, 0.0), 45.0, 256, 192)
        frames = [r.render_frame(0.0, static_pose=True, forced_lod=l)[0] for l in range(3)]
        for l in range(3):
            got = rows[3 * k + l]["psnr_db"]
            want = 99.0 if l == 0 else P.psnr(frames[l], frames[0])
            assert abs(got - want) < 1e-3, (d, l, got, want)
            if l:
                assert got < 99.0


def test_invalid_settings_raise():
    s = basic_scene(count=1, rows=1, cols=1)
    r = P.Renderer(s)
    with pytest.raises(ValueError):
        r.render_frame(0.0, P.RenderSettings(tile_size=0))
    with pytest.raises(ValueError):
        r.render_frame(0.0, P.RenderSettings(alpha_cutoff=1.5))
    with pytest.raises(ValueError):
        r.render_frame(0.0, P.RenderSettings(transmittance_floor=0.0))


def test_convex_hull_and_transmittance_range():
    s = basic_scene(count=16)
    r = P.Renderer(s)
    rgb, T = r.render_frame(0.3, P.RenderSettings(background=(0.3, 0.3, 0.3), sh_colour=False))
    assert rgb.min() >= 0.0 and rgb.max() <= 1.0 + 1e-5
    assert T.min() >= 0.0 and T.max() <= 1.0


def config_scene(idx, sh=True):
    cfg, extra = P.baseline_config(idx)
    cfg.with_sh = sh
    s = P.Scene(cfg)
    if extra["origin_instance"]:
        P.place_origin_instance(s)
    return s, extra


@pytest.mark.parametrize("idx", [1, 2])
def test_baseline_config(idx):
    s, extra = config_scene(idx)
    rep = parity(s, extra["time_s"], forced_lod=extra["forced_lod"])
    assert rep["S"] > 0 and rep["K"] > 0
    check_cull_invariance(P.Renderer(s), extra["time_s"], forced_lod=extra["forced_lod"])


# Cameras inside and around a crowd, looking along and across the rows, tilted, with wide
# and narrow fields of view: instances straddle every frustum side and the near plane.
CULL_CAMERAS = [
    ((5.5, 1.6, -3.0), (5.5, 1.0, 5.0), 50.0, 16),
    ((5.5, 1.7, 5.5), (12.0, 1.2, 6.0), 50.0, 16),
    ((5.5, 1.7, 5.5), (-3.0, 1.0, 4.0), 70.0, 8),
    ((5.5, 1.7, 5.5), (5.0, 1.5, -4.0), 30.0, 16),
    ((5.5, 6.0, 5.5), (6.0, 0.0, 8.0), 60.0, 16),
    ((5.5, 0.3, 2.0), (5.5, 2.5, 9.0), 40.0, 3),
    ((14.0, 1.6, 5.5), (-1.0, 1.0, 5.5), 90.0, 16),
    ((5.5, 1.0, 5.2), (5.6, 1.0, 5.9), 50.0, 16),   # nose against one character
]


@pytest.mark.parametrize("cam", CULL_CAMERAS)
def test_instance_cull_is_invisible(cam):
    pos, look, fov, tile = cam
    cfg = P.SceneConfig(template_count=3, level_counts=(400, 120, 40), with_sh=True, motion_count=3,
                        motion_frames=24, grid_rows=12, grid_cols=12, crowd_count=144, crowd_seed=5,
                        cam_pos=pos, cam_look=look, width=320, height=200)
    s = P.Scene(cfg)
    s.set_camera(pos, look, fov_y_deg=fov, width=320, height=200)
    r = P.Renderer(s)
    culled = check_cull_invariance(r, 0.4, P.RenderSettings(tile_size=tile))
    assert 0 <= culled < 144


@pytest.mark.slow
def test_baseline_config3_headline():
    s, extra = config_scene(3)
    r = P.Renderer(s)
    o = orc.from_scene(s)
    g, c = render_both(s, r, o, 0.5)
    rep = check_frame(s, r, o, g, c)
    assert rep["G"] == 14972565 and rep["S"] > 10_000_000
    again, _ = r.render_frame(0.5, P.RenderSettings())
    assert again.tobytes() == g[0].tobytes()
    assert check_cull_invariance(r, 0.5) > 500  # about a quarter of the crowd is off-screen


@pytest.mark.slow
def test_baseline_config4_4k_ten_thousand():
    """BASELINE config 4 at full size (10,000 characters, 3840x2160; 17-bit quadrant cell
    ids): every bit-exact bar against the oracle, with device pose sampling."""
    s, extra = config_scene(4)
    r = P.Renderer(s, device_poses=True)
    o = orc.from_scene(s)
    g, c = render_both(s, r, o, 0.25)
    rep = check_frame(s, r, o, g, c)
    assert rep["S"] > 20_000_000 and rep["K"] > 50_000_000
    assert check_cull_invariance(r, 0.25) > 1000


def test_instance_cull_is_invisible_for_any_camera_matrix():
    """The C-ABI takes any world_to_view matrix, not only the rotation CameraBasis builds
    (math.cpp:118-129). The cull bounds the camera-space ball by |W|_2 and the rect by
    |W0 - u W2|, so a scaled and sheared matrix must still give a byte-identical frame."""
    import ctypes as C
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import gscg_settings

    pos, look = (5.5, 1.7, 5.5), (12.0, 1.2, 6.0)
    cfg = P.SceneConfig(template_count=3, level_counts=(400, 120, 40), with_sh=True, motion_count=3,
                        motion_frames=24, grid_rows=12, grid_cols=12, crowd_count=144, crowd_seed=5,
                        cam_pos=pos, cam_look=look, width=320, height=200)
    s = P.Scene(cfg)
    r = P.Renderer(s, device_poses=True)
    r.render_frame(0.4, P.RenderSettings())  # uploads templates and motion tables
    tids, place, _ = r.sample_crowd(0.4)
    n = len(tids)
    inst = s.instances
    mids = np.ascontiguousarray(inst["motion_id"]).astype(np.uint32)
    phase = np.ascontiguousarray(inst["phase_offset_s"]).astype(np.float32)
    cam = s.camera_basis()
    scale = [1.3, 1.3, 1.3, 0.8, 0.8, 0.8, 1.1, 1.1, 1.1]
    for i in range(9):
        cam.world_to_view[i] *= scale[i]
    cam.world_to_view[1] += 0.25  # shear
    rs = gscg_settings(P.RenderSettings())
    lp = N.GscgLodPolicy()
    lp.threshold_count = len(cfg.lod_thresholds)
    for i, v in enumerate(cfg.lod_thresholds):
        lp.thresholds_m[i] = v
    lib, ctx = N.gscg(), r.gpu
    out = []
    for flags in (N.GSCG_DEBUG_RECORDS | N.GSCG_DEBUG_NO_CULL, N.GSCG_DEBUG_RECORDS):
        N.check_gscg(lib.gscg_set_debug(ctx, flags), ctx)
        lods = np.full(n, 0xFFFFFFFF, dtype=np.uint32)
        fd = N.GscgFrameDesc()
        fd.instance_count, fd.joint_stride = n, r.joint_stride
        fd.template_ids, fd.placement = tids.ctypes.data, place.ctypes.data
        fd.active_lod, fd.forced_lod = lods.ctypes.data, -1
        fd.memory, fd.pose_source, fd.time_s = N.GSCG_MEM_HOST, N.GSCG_POSES_SAMPLED, 0.4
        fd.motion_ids, fd.phase_offsets = mids.ctypes.data, phase.ctypes.data
        rgb = np.zeros((cfg.height, cfg.width, 3), np.float32)
        T = np.zeros((cfg.height, cfg.width), np.float32)
        N.check_gscg(lib.gscg_render_frame(ctx, C.byref(fd), C.byref(cam), C.byref(rs), C.byref(lp),
                                           rgb.ctypes.data, T.ctypes.data, None), ctx)
        rec = r.splat_records()
        rec = rec[np.argsort(rec["ordinal"], kind="stable")]
        out.append((rgb, T, r.counts(), rec.tobytes(), r.sorted_ordinals().copy(), r.instances_culled()))
    (a, b) = out
    assert a[5] == 0 and a[2] == b[2] and a[3] == b[3]
    assert np.array_equal(a[4], b[4])
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    assert a[2][1] > 0  # something is on screen


def config5_scene(count: int):
    """BASELINE config 5 (LoD off: every character at the full 202,738-Gaussian level,
    crowd.cpp:94-96 forced LoD) on its own grid and camera, the first `count` characters
    (row-major cells: the near field, where splats are largest and pairs densest)."""
    cfg, extra = P.baseline_config(5)
    cfg.crowd_count = count
    return P.Scene(cfg), extra


@pytest.mark.slow
def test_config5_forced_lod0_crowd_against_oracle():
    """Config-5 code paths at crowd scale: 240 characters at LoD 0, 1920x1080 (48.7 M
    instance-Gaussians, 5.9 M splats, near-field cells with long tied runs), every
    bit-exact bar against the oracle."""
    s, extra = config5_scene(240)
    r = P.Renderer(s, device_poses=True)
    o = orc.from_scene(s)
    g, c = render_both(s, r, o, 0.25, forced_lod=extra["forced_lod"])
    rep = check_frame(s, r, o, g, c)
    assert rep["G"] == 240 * 202738 and rep["S"] > 5_000_000 and rep["K"] > rep["S"]


def test_pair_count_past_32_bits_is_reported_as_oom():
    """K >= 2^32 tile-splat pairs (config 5 at tile size 1: every splat's rect is at least
    4x4 pixels after the 0.3 px^2 dilation, so K > 16 x 519 M) must surface as
    GSCG_ERR_OOM (the reference's bench skips such a cell as "out of memory",
    bench.cpp:94-97) before any buffer is grown, not alias into the splat count; the
    context stays usable afterwards."""
    from paper_2501_17792_b200 import native as N

    s, extra = config5_scene(3500)
    r = P.Renderer(s, device_poses=True)
    with pytest.raises(N.NativeError) as e:
        r.render_frame(0.0, P.RenderSettings(tile_size=1), forced_lod=0)
    assert e.value.status == N.GSCG_ERR_OOM  # std::bad_alloc through the C++ API, as bench.cpp:94-97 expects
    rgb, _ = r.render_frame(0.0, P.RenderSettings(), forced_lod=2)  # same context, a normal frame
    assert r.counts()[1] > 0 and np.isfinite(rgb).all()


def test_instance_gaussians_past_32_bit_ordinals_is_reported_as_oom():
    """Global ordinals (instance base + gaussian index, the reference's (instance,
    gaussian) tie-break) are 32-bit: 22,500 characters at LoD 0 (4.56 G instance-
    Gaussians) must fail with GSCG_ERR_OOM rather than wrap and break the sort order."""
    from paper_2501_17792_b200 import native as N

    cfg, _ = P.baseline_config(5)
    cfg.grid_rows, cfg.grid_cols, cfg.crowd_count = 150, 150, 22500
    r = P.Renderer(P.Scene(cfg), device_poses=True)
    with pytest.raises(N.NativeError) as e:
        r.render_frame(0.0, P.RenderSettings(), forced_lod=0)
    assert e.value.status == N.GSCG_ERR_OOM


def gpu_vs_reference_build(idx: int, device_poses: bool = False) -> dict:
    """The CUDA path against the REFERENCE's own render_frame (oracle/_ref: its unmodified
    sources built against the Eigen-subset shim; prebuilt .so shipped with the repo), on
    the reference's own synthetic scene (RGB colour: the reference has no SH)."""
    from oracle import ref

    if not ref.LIB_PATH.exists():
        pytest.skip("prebuilt reference (oracle/_ref/libgsc_ref.so) not shipped")
    s, extra = config_scene(idx, sh=False)
    rc, rextra = ref.baseline(idx)
    rs = ref.RefScene(rc, rextra["origin_instance"])
    assert s.instances.tobytes() == rs.instances.tobytes()
    r = P.Renderer(s, device_poses=device_poses)
    from paper_2501_17792_b200 import native as N
    r.set_debug(N.GSCG_DEBUG_POSED | N.GSCG_DEBUG_RECORDS)
    t = extra["time_s"] + 0.25
    rgb, T = r.render_frame(t, P.RenderSettings(sh_colour=False), forced_lod=extra["forced_lod"])
    out_r = rs.render(t, ref.settings(), forced_lod=extra["forced_lod"])
    return check_frame(s, r, rs, (rgb, T), out_r)


@pytest.mark.parametrize("idx", [1, 2])
def test_gpu_matches_reference_build(idx):
    rep = gpu_vs_reference_build(idx)
    assert rep["S"] > 90_000


@pytest.mark.slow
def test_gpu_matches_reference_build_config3():
    rep = gpu_vs_reference_build(3, device_poses=True)
    assert rep["G"] == 14972565


BAND_SPLITS = [
    (1080, [0, 1080]),
    (1080, [0, 208, 512, 1080]),
    (1080, [0, 16, 32, 400, 416, 1072, 1080]),
]


@pytest.mark.parametrize("split", BAND_SPLITS)
def test_band_frames_assemble_the_whole_frame_bit_for_bit(split):
    """gscg_set_band (the multi-GPU band frame): each band renders only its
    rows; stacking the bands must give the whole frame byte for byte (RGB and T), the
    per-band tile lists being the reference's bins (config 2, device poses)."""
    s, extra = config_scene(2)
    r = P.Renderer(s, device_poses=True)
    t = 0.4
    full_rgb, full_T = r.render_frame(t, P.RenderSettings())
    full_rgb, full_T = full_rgb.copy(), full_T.copy()
    _, rows = split
    rb = P.Renderer(s, device_poses=True)
    parts_rgb, parts_T = [], []
    for b in range(len(rows) - 1):
        rb.set_band(rows[b], rows[b + 1])
        rgb, T = rb.render_frame(t, P.RenderSettings())
        assert rgb.shape == (rows[b + 1] - rows[b], 1920, 3)
        parts_rgb.append(rgb.copy())
        parts_T.append(T.copy())
    assert np.concatenate(parts_rgb).tobytes() == full_rgb.tobytes()
    assert np.concatenate(parts_T).tobytes() == full_T.tobytes()
    rb.set_band(0, 0)
    again, _ = rb.render_frame(t, P.RenderSettings())
    assert again.tobytes() == full_rgb.tobytes()


def test_group_single_rank_frame_equals_render_frame():
    """gscg_group_render_frame with one rank (its own NCCL communicator, no peers): the
    assembled frame equals gscg_render_frame's byte for byte, and the row costs sum to
    the frame's binned cell pairs."""
    import ctypes as C
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import BandGroup, gscg_settings

    s, extra = config_scene(2)
    r = P.Renderer(s, device_poses=True)
    full_rgb, full_T = r.render_frame(0.3, P.RenderSettings())
    full_rgb, full_T = full_rgb.copy(), full_T.copy()
    K = r.counts()[2]
    g = BandGroup(r, 0, 1)
    rec = r.instance_records()
    n = len(rec["template_ids"])
    fd = N.GscgFrameDesc()
    fd.instance_count = n
    fd.joint_stride = r.joint_stride
    fd.template_ids = rec["template_ids"].ctypes.data
    fd.placement = rec["placement"].ctypes.data
    lods = np.full(n, 0xFFFFFFFF, np.uint32)
    fd.active_lod = lods.ctypes.data
    fd.forced_lod = -1
    fd.memory = N.GSCG_MEM_HOST
    fd.pose_source = N.GSCG_POSES_SAMPLED
    fd.time_s = 0.3
    fd.motion_ids = rec["motion_ids"].ctypes.data
    fd.phase_offsets = rec["phase_offsets"].ctypes.data
    cfg = s.cfg
    lp = N.GscgLodPolicy()
    lp.threshold_count = len(cfg.lod_thresholds)
    for i, v in enumerate(cfg.lod_thresholds):
        lp.thresholds_m[i] = v
    rgb = np.empty((cfg.height, cfg.width, 3), np.float32)
    T = np.empty((cfg.height, cfg.width), np.float32)
    g.render(fd, s.camera_basis(), gscg_settings(P.RenderSettings()), lp, rgb, T)
    assert rgb.tobytes() == full_rgb.tobytes() and T.tobytes() == full_T.tobytes()
    costs = g.tile_costs()
    assert int(costs.sum()) == K and costs.shape == ((cfg.height + 15) // 16, (cfg.width + 15) // 16)
    cuts = g.rebalance()  # column cuts (the default split axis)
    assert cuts[0] == 0 and cuts[-1] == cfg.width
    g.close()


@pytest.mark.parametrize("forced", [None, 0])
def test_naive_layout_renders_the_same_frame(forced):
    """gscg_set_layout(NAIVE): every instance reads its own copy of its level's attributes
    (the config-5 ablation); the frame must be byte-identical to the shared store's, and
    the copies must hold 80 B per instance-Gaussian."""
    s, extra = config_scene(2, sh=False)
    r = P.Renderer(s, device_poses=True)
    st = P.RenderSettings(sh_colour=False)
    a, Ta = r.render_frame(0.6, st, forced_lod=forced)
    a, Ta = a.copy(), Ta.copy()
    r.set_layout(True)
    b, Tb = r.render_frame(0.6, st, forced_lod=forced)
    G = r.counts()[0]
    assert a.tobytes() == b.tobytes() and Ta.tobytes() == Tb.tobytes()
    assert r.memory_usage()["naive_attribute_bytes"] == 80 * G
    c, _ = r.render_frame(0.7, st, forced_lod=forced)  # second frame reuses the copies
    r.set_layout(False)
    d, _ = r.render_frame(0.7, st, forced_lod=forced)
    assert c.tobytes() == d.tobytes() and r.memory_usage()["naive_attribute_bytes"] == 0


COL_SPLITS = [[0, 1920], [0, 640, 1280, 1920], [0, 16, 512, 528, 1904, 1920]]


@pytest.mark.parametrize("cols", COL_SPLITS)
def test_column_regions_assemble_the_whole_frame_bit_for_bit(cols):
    """gscg_set_region with column splits (the multi-GPU frame's default axis): the
    full-height column regions side by side equal the whole frame byte for byte."""
    s, extra = config_scene(2)
    r = P.Renderer(s, device_poses=True)
    full_rgb, full_T = r.render_frame(0.4, P.RenderSettings())
    full_rgb, full_T = full_rgb.copy(), full_T.copy()
    rb = P.Renderer(s, device_poses=True)
    parts_rgb, parts_T = [], []
    for b in range(len(cols) - 1):
        rb.set_region(cols[b], 0, cols[b + 1], 0)
        rgb, T = rb.render_frame(0.4, P.RenderSettings())
        assert rgb.shape == (1080, cols[b + 1] - cols[b], 3)
        parts_rgb.append(rgb.copy())
        parts_T.append(T.copy())
    assert np.concatenate(parts_rgb, axis=1).tobytes() == full_rgb.tobytes()
    assert np.concatenate(parts_T, axis=1).tobytes() == full_T.tobytes()


def test_pipelined_device_frames_follow_the_lod_chain():
    """Device-memory frames enqueued back to back without a host wait (the bench's path:
    a frame's update + projection run under the previous frame's sort and raster, two frame
    slots), the camera moving so hysteresis flips levels: every frame equals the oracle's,
    which carries the LoD state frame to frame (the front half must see the previous
    frame's levels)."""
    import ctypes as C

    import torch

    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import gscg_settings

    s = basic_scene(count=16, rows=4, cols=4, sh=False)
    s.set_lod_policy((3.5, 6.0), hysteresis=1.0)
    r = P.Renderer(s, device=0, device_poses=True)
    o = orc.from_scene(s)
    o.set_lod((3.5, 6.0), 1.0)
    st = P.RenderSettings(sh_colour=False)
    r.render_frame(0.0, st)  # templates + motion tables
    rec = r.instance_records()
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int32) if v.dtype == np.uint32 else v).to(dev)
         for k, v in rec.items()}
    d_lods = torch.full((len(rec["lods"]),), -1, dtype=torch.int32, device=dev)
    n, lib, ctx = len(rec["lods"]), N.gscg(), r.gpu
    rs = gscg_settings(st)
    lp = N.GscgLodPolicy()
    lp.threshold_count = 2
    lp.thresholds_m[0], lp.thresholds_m[1] = 3.5, 6.0
    lp.hysteresis_band_m = 1.0
    zs = (-0.5, 0.0, 0.4, 0.8, 0.4, -0.3, 2.8, 3.3, 2.9)
    H, W = s.cfg.height, s.cfg.width
    outs = [torch.empty((H, W, 3), dtype=torch.float32, device=dev) for _ in zs]
    cams = []
    for f, z in enumerate(zs):
        s.set_camera((0.0, 1.6, -3.0 - z), (0.0, 1.0, 5.0))
        cam = s.camera_basis()
        cams.append(cam)
        fd = N.GscgFrameDesc()
        fd.instance_count, fd.joint_stride = n, r.joint_stride
        fd.template_ids, fd.placement = d["template_ids"].data_ptr(), d["placement"].data_ptr()
        fd.active_lod, fd.forced_lod = d_lods.data_ptr(), -1
        fd.memory, fd.pose_source, fd.time_s = N.GSCG_MEM_DEVICE, N.GSCG_POSES_SAMPLED, 0.1 + f / 30.0
        fd.motion_ids, fd.phase_offsets = d["motion_ids"].data_ptr(), d["phase_offsets"].data_ptr()
        N.check_gscg(lib.gscg_render_frame(ctx, C.byref(fd), C.byref(cam), C.byref(rs), C.byref(lp),
                                           C.c_void_p(outs[f].data_ptr()), None, None), ctx)
    N.check_gscg(lib.gscg_synchronize(ctx), ctx)
    flips = 0
    prev = None
    for f, z in enumerate(zs):
        o.set_camera((0.0, 1.6, -3.0 - z), (0.0, 1.0, 5.0), 50.0, W, H)
        orgb, _, _ = o.render(0.1 + f / 30.0, orc.settings(sh_colour=False))
        lods = o.lods(n)
        flips += int(prev is not None and not np.array_equal(prev, lods))
        prev = lods.copy()
        assert outs[f].cpu().numpy().tobytes() == orgb.tobytes(), f"frame {f} differs from the oracle"
    assert flips >= 2  # the sequence really moves levels
    assert np.array_equal(d_lods.cpu().numpy().astype(np.uint32), prev)


def _patch_extreme_gaussians(path):
    """Rewrites level 0 of a v1 GSAT file (io.cpp layout, tests/test_io.py) with extreme but
    valid Gaussians (the LodLevel invariants, avatar.cpp validate): a near-zero and two
    screen-covering scales, tiny / denormal / unit opacities, a pure-blue colour, a mean far
    above the crowd and one behind the camera, equal four-joint weights."""
    import struct

    b = bytearray(path.read_bytes())
    J = int.from_bytes(b[8:10], "little")
    off = 11 + 66 * J
    n = int.from_bytes(b[off:off + 4], "little")
    means = off + 4
    rot = means + 12 * n
    sc = rot + 16 * n
    op = sc + 12 * n
    col = op + 4 * n
    sw = col + 12 * n + 8 * n

    def put(base, i, vals):
        stride = 4 * len(vals)
        b[base + stride * i:base + stride * (i + 1)] = struct.pack("<%df" % len(vals), *vals)

    put(sc, 0, (1e-30, 1e-30, 1e-30))
    put(sc, 1, (50.0, 50.0, 50.0))
    put(sc, 2, (30.0, 1e-3, 1e-3))
    put(op, 3, (1e-30,))
    put(op, 4, (1.0,))
    put(op, 5, (1.4e-45,))
    put(col, 6, (0.0, 0.0, 1.0))
    put(means, 7, (0.0, 1e6, 0.0))
    put(means, 8, (0.0, 0.0, -1e3))
    put(sw, 9, (0.25, 0.25, 0.25, 0.25))
    path.write_bytes(bytes(b))


@pytest.mark.parametrize("size,tile", [((200, 120), 16), ((640, 360), 16), ((200, 120), 8)])
def test_extreme_gaussians_match_the_oracle(tmp_path, size, tile):
    """Screen-covering splats (every cell's list, emission blocks past the staged-pair
    capacity at 640x360), vanishing ones, opacities that never or always saturate, and
    splats culled far away or behind the camera: the frame still equals the oracle's."""
    w, h = size
    cfg = P.SceneConfig(template_count=1, template_seed_base=1, level_counts=(60, 24, 8), with_sh=False,
                        motion_count=1, motion_seed_base=2, motion_frames=24, grid_rows=2, grid_cols=2,
                        grid_spacing=1.2, crowd_count=4, crowd_seed=42, cam_pos=(0.6, 1.5, -3.5),
                        cam_look=(0.6, 1.0, 2.0), width=w, height=h)
    s = P.Scene(cfg)
    path = tmp_path / "extreme.gsat"
    s.save_template(0, path)
    _patch_extreme_gaussians(path)
    s.load_template(path, 0)
    r = P.Renderer(s)
    o = orc.from_scene(s)
    for t, static in ((0.3, False), (0.0, True)):
        g, c = render_both(s, r, o, t, tile_size=tile, static_pose=static, forced_lod=0, sh=False)
        rep = check_frame(s, r, o, g, c, tile_size=tile)
        assert rep["S"] <= 4 * 58  # the far and the behind-camera Gaussians culled in every instance


# (pos, look, fov_y_deg, (width, height), near_m, tile): nose against a character, the
# widest and narrowest fields of view, degenerate resolutions, a tiny and a far near plane.
EXTREME_CAMERAS = [
    ((2.5, 1.1, 2.3), (2.6, 1.0, 3.5), 50.0, (160, 96), 0.1, 16),
    ((2.5, 1.7, -1.0), (2.5, 1.0, 5.0), 170.0, (160, 96), 0.1, 16),
    ((2.5, 1.7, -8.0), (2.5, 1.0, 5.0), 1.0, (160, 96), 0.1, 16),
    ((2.5, 1.7, -3.0), (2.5, 1.0, 5.0), 50.0, (17, 3), 0.1, 16),
    ((2.5, 1.7, -3.0), (2.5, 1.0, 5.0), 50.0, (1, 1), 0.1, 4),
    ((2.5, 1.2, 1.0), (2.5, 1.0, 5.0), 60.0, (160, 96), 1e-3, 16),
    ((2.5, 1.7, -3.0), (2.5, 1.0, 5.0), 50.0, (160, 96), 5.0, 16),
]


@pytest.mark.parametrize("cam", EXTREME_CAMERAS)
def test_extreme_cameras_match_the_oracle(cam):
    pos, look, fov, (w, h), near, tile = cam
    cfg = P.SceneConfig(template_count=2, level_counts=(200, 60, 20), with_sh=False, motion_count=2,
                        motion_frames=24, grid_rows=6, grid_cols=6, crowd_count=36, crowd_seed=9,
                        cam_pos=pos, cam_look=look, width=w, height=h)
    s = P.Scene(cfg)
    s.set_camera(pos, look, fov_y_deg=fov, width=w, height=h, near_m=near)
    r = P.Renderer(s)
    o = orc.from_scene(s)
    g, c = render_both(s, r, o, 0.25, tile_size=tile, background=(0.1, 0.2, 0.3), sh=False)
    check_frame(s, r, o, g, c, tile_size=tile)


def test_group_frames_in_flight_follow_the_lod_chain():
    """Region-split frames as the multi-GPU bench times them (one-rank NCCL group,
    device-memory inputs, no stage times read, so frames stay in flight back to back) with
    the camera moving through hysteresis: the last gathered frame equals the oracle's after
    the same LoD chain, and a time-based rebalance keeps one rank's cuts whole."""
    import ctypes as C

    import torch

    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import BandGroup, gscg_settings

    s = basic_scene(count=16, rows=4, cols=4, sh=False)
    s.set_lod_policy((3.5, 6.0), hysteresis=1.0)
    r = P.Renderer(s, device=0, device_poses=True)
    o = orc.from_scene(s)
    o.set_lod((3.5, 6.0), 1.0)
    st = P.RenderSettings(sh_colour=False)
    r.render_frame(0.0, st)  # templates + motion tables
    rec = r.instance_records()
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int32) if v.dtype == np.uint32 else v).to(dev)
         for k, v in rec.items()}
    n = len(rec["lods"])
    d_lods = torch.full((n,), -1, dtype=torch.int32, device=dev)
    lp = N.GscgLodPolicy()
    lp.threshold_count = 2
    lp.thresholds_m[0], lp.thresholds_m[1] = 3.5, 6.0
    lp.hysteresis_band_m = 1.0
    g = BandGroup(r, 0, 1)
    H, W = s.cfg.height, s.cfg.width
    zs = (-0.5, 0.0, 0.4, 0.8, 0.4, -0.3, 2.8, 3.3, 2.9)
    rgb = np.empty((H, W, 3), np.float32)
    for f, z in enumerate(zs):
        s.set_camera((0.0, 1.6, -3.0 - z), (0.0, 1.0, 5.0))
        fd = N.GscgFrameDesc()
        fd.instance_count, fd.joint_stride = n, r.joint_stride
        fd.template_ids, fd.placement = d["template_ids"].data_ptr(), d["placement"].data_ptr()
        fd.active_lod, fd.forced_lod = d_lods.data_ptr(), -1
        fd.memory, fd.pose_source, fd.time_s = N.GSCG_MEM_DEVICE, N.GSCG_POSES_SAMPLED, 0.1 + f / 30.0
        fd.motion_ids, fd.phase_offsets = d["motion_ids"].data_ptr(), d["phase_offsets"].data_ptr()
        last = f == len(zs) - 1
        g.render(fd, s.camera_basis(), gscg_settings(st), lp, rgb if last else None, stage_times=last)
    for f, z in enumerate(zs):
        o.set_camera((0.0, 1.6, -3.0 - z), (0.0, 1.0, 5.0), 50.0, W, H)
        orgb, _, _ = o.render(0.1 + f / 30.0, orc.settings(sh_colour=False))
    assert rgb.tobytes() == orgb.tobytes()
    assert np.array_equal(d_lods.cpu().numpy().astype(np.uint32), o.lods(n))
    assert g.rebalance_by_time(0.5) == [0, W]
    g.close()


def test_group_async_readback_matches_blocking_frames():
    """gscg_group_render_frame_async (rank 0's host read-back under the next frame, two
    device frame buffers alternating): every frame read back equals the blocking call's."""
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.api import pinned_array
    from paper_2501_17792_b200.multigpu import BandGroup, gscg_settings

    s, extra = config_scene(2)
    r = P.Renderer(s, device_poses=True)
    r.render_frame(0.3, P.RenderSettings())
    g = BandGroup(r, 0, 1)
    rec = r.instance_records()
    n = len(rec["template_ids"])
    lods = np.full(n, 0xFFFFFFFF, np.uint32)
    cfg = s.cfg
    lp = N.GscgLodPolicy()
    lp.threshold_count = len(cfg.lod_thresholds)
    for i, v in enumerate(cfg.lod_thresholds):
        lp.thresholds_m[i] = v

    def fd_at(t):
        fd = N.GscgFrameDesc()
        fd.instance_count, fd.joint_stride = n, r.joint_stride
        fd.template_ids, fd.placement = rec["template_ids"].ctypes.data, rec["placement"].ctypes.data
        fd.active_lod, fd.forced_lod = lods.ctypes.data, -1
        fd.memory, fd.pose_source, fd.time_s = N.GSCG_MEM_HOST, N.GSCG_POSES_SAMPLED, t
        fd.motion_ids, fd.phase_offsets = rec["motion_ids"].ctypes.data, rec["phase_offsets"].ctypes.data
        return fd

    times = (0.3, 0.5, 0.7, 0.9)
    st = gscg_settings(P.RenderSettings())
    cam = s.camera_basis()
    ref = []
    for t in times:
        out = np.empty((cfg.height, cfg.width, 3), np.float32)
        g.render(fd_at(t), cam, st, lp, out)
        ref.append(out)
    bufs = [pinned_array((cfg.height, cfg.width, 3)) for _ in range(2)]
    for wait_each in (True, False):  # each frame checked, then frames streamed back to back
        lods[:] = 0xFFFFFFFF  # the blocking pass's LoD chain start
        got = []
        for k, t in enumerate(times):
            g.render(fd_at(t), cam, st, lp, bufs[k % 2], stage_times=False, pipelined=True)
            if wait_each:
                g.wait_readback()
                got.append(bufs[k % 2].copy())
        g.wait_readback()
        if wait_each:
            assert all(a.tobytes() == b.tobytes() for a, b in zip(got, ref))
        assert bufs[(len(times) - 1) % 2].tobytes() == ref[-1].tobytes()
        assert bufs[(len(times) - 2) % 2].tobytes() == ref[-2].tobytes()
    # a blocking frame right after async ones (the buffer's read-back may be in flight)
    g.render(fd_at(times[0]), cam, st, lp, bufs[0], stage_times=False, pipelined=True)
    out = np.empty((cfg.height, cfg.width, 3), np.float32)
    g.render(fd_at(times[-1]), cam, st, lp, out)
    g.wait_readback()
    assert out.tobytes() == ref[-1].tobytes() and bufs[0].tobytes() == ref[0].tobytes()
    g.close()
