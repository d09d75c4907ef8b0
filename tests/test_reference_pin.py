"""Pins the oracle and the product's host generator against the REFERENCE's own code.

oracle/_ref/libgsc_ref.so is /root/reference/proj/src/{math,avatar,synthetic,lod,crowd,
renderer,metrics,bench}.cpp compiled unmodified against the from-scratch Eigen subset in
oracle/eigen_shim (oracle/Makefile). These CPU tests require, bit for bit:
  * the product's synthetic templates / motions / crowd == the reference's generator
    (synthetic.cpp, crowd.cpp:46-84), so both sides render the same inputs;
  * the oracle restatement (oracle/orc.cpp) == the reference's render_frame
    (renderer.cpp:249-280): LoD, posed means, the sorted splat frame, the per-tile bins,
    every pixel and the final transmittance; across tile sizes, forced LoD, static pose,
    hysteresis, background colours, thread counts and BASELINE configs 1-2.
The GPU path is checked against the oracle (tests/parity.py) and, where the prebuilt
reference .so is present, against the reference directly (test_gpu_parity.py).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2501_17792_b200 as P
from oracle import orc, ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference build (oracle/_ref) unavailable")

LEVEL_KEYS = ("means", "rotations", "scales", "opacities", "colors", "skin_indices", "skin_weights", "cov6")


def small_cfg(**kw) -> P.SceneConfig:
    base = dict(template_count=3, level_counts=(3000, 700, 150), with_sh=False, motion_count=3, motion_frames=24,
                grid_rows=4, grid_cols=4, crowd_count=16, crowd_seed=77, cam_pos=(1.5, 1.6, -3.0),
                cam_look=(1.5, 1.0, 5.0), width=320, height=180, lod_thresholds=(3.5, 5.5))
    base.update(kw)
    return P.SceneConfig(**base)


def assert_same_inputs(scene: P.Scene, rs: ref.RefScene) -> None:
    nt, nm, n = scene.counts()
    assert (nt, nm, n) == rs.counts()
    for t in range(nt):
        a, b = scene.skeleton(t), rs.skeleton(t)
        assert np.array_equal(a["parents"], b["parents"])
        assert a["inverse_bind"].tobytes() == b["inverse_bind"].tobytes()
        for l in range(scene.level_count(t)):
            la, lb = scene.level_view(t, l), rs.level(t, l)
            for k in LEVEL_KEYS:
                assert la[k].tobytes() == lb[k].tobytes(), f"template {t} level {l}: {k} differs from the reference"
    for m in range(nm):
        assert scene.motion(m)["data"].tobytes() == rs.motion(m)["data"].tobytes(), f"motion {m}"
    assert scene.instances.tobytes() == rs.instances.tobytes(), "build_crowd placement differs"


def assert_same_frame(o: orc.OracleScene, rs: ref.RefScene, cfg, tile_size: int, out_o, out_r) -> dict:
    (orgb, oT, ot), (rrgb, rT, rt) = out_o, out_r
    assert (ot.gaussian_count, ot.splat_count, ot.pair_count) == (rt.gaussian_count, rt.splat_count, rt.pair_count)
    assert np.array_equal(o.lods(len(rs.instances)), rs.lods()), "LoD"
    assert o.posed().tobytes() == rs.posed().tobytes(), "posed means"
    assert o.splats().tobytes() == rs.splats().tobytes(), "sorted splat frame"
    tiles = ((cfg.width + tile_size - 1) // tile_size) * ((cfg.height + tile_size - 1) // tile_size)
    oc, oi = o.bins(tiles)
    rc, ri = rs.bins(tiles)
    assert np.array_equal(oc, rc) and np.array_equal(oi, ri), "per-tile bins"
    assert orgb.tobytes() == rrgb.tobytes(), "pixels"
    assert oT.tobytes() == rT.tobytes(), "transmittance"
    return {"G": rt.gaussian_count, "S": rt.splat_count, "K": rt.pair_count}


def render_pair(cfg, time_s=0.37, tile_size=16, background=(0.0, 0.0, 0.0), static_pose=False, forced_lod=None,
                threads=0, frames=1):
    scene = P.Scene(cfg)
    rs = ref.RefScene(ref.RefConfig.like(cfg))
    assert_same_inputs(scene, rs)
    o = orc.from_scene(scene)
    rep = None
    for f in range(frames):  # successive frames carry LoD state (hysteresis)
        t = time_s + f / 30.0
        out_o = o.render(t, orc.settings(tile_size=tile_size, background=background, sh_colour=False), static_pose,
                         forced_lod, threads=threads)
        out_r = rs.render(t, ref.settings(tile_size=tile_size, background=background), static_pose, forced_lod,
                          threads=threads)
        rep = assert_same_frame(o, rs, cfg, tile_size, out_o, out_r)
    return rep


def test_reference_build_exports_every_entry_point():
    for name in ref._SIGS:
        assert hasattr(ref.lib(), name)


def test_paper_template_generator_matches_reference():
    """One full BASELINE template (202,738 / 12,661 / 3,176 Gaussians): every attribute
    and the finalize() covariance cache, including the Gaussians whose normal is nearly
    opposite +z (setFromTwoVectors' SVD branch)."""
    cfg = P.SceneConfig(template_count=1, template_seed_base=105, level_counts=ref.LEVELS_PAPER, with_sh=False,
                        motion_count=2, motion_frames=60)
    assert_same_inputs(P.Scene(cfg), ref.RefScene(ref.RefConfig.like(cfg)))


@pytest.mark.parametrize("time_s", [0.0, 0.37, 1.3])
def test_oracle_equals_reference_frame(time_s):
    rep = render_pair(small_cfg(), time_s, background=(0.1, 0.1, 0.15))
    assert rep["S"] > 0 and rep["K"] > 0


@pytest.mark.parametrize("tile_size", [1, 3, 8, 16, 17, 40])
def test_oracle_equals_reference_tile_sizes(tile_size):
    render_pair(small_cfg(crowd_count=9, grid_rows=3, grid_cols=3, crowd_seed=55), 0.2, tile_size=tile_size,
                background=(0.2, 0.4, 0.6))


@pytest.mark.parametrize("forced", [0, 1, 2, 7])
def test_oracle_equals_reference_forced_lod(forced):
    render_pair(small_cfg(), 0.4, forced_lod=forced)


def test_oracle_equals_reference_static_pose():
    render_pair(small_cfg(), 0.0, static_pose=True, background=(0.3, 0.2, 0.1), frames=2)


def test_oracle_equals_reference_hysteresis_across_frames():
    cfg = small_cfg(lod_thresholds=(3.0, 4.0, 6.0), lod_hysteresis=1.5)
    render_pair(cfg, 0.1, frames=3)


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_equals_reference_any_thread_count(threads):
    render_pair(small_cfg(), 0.6, threads=threads)


@pytest.mark.parametrize("idx", [1, 2])
def test_oracle_equals_reference_baseline_config(idx):
    """BASELINE configs 1 and 2 at full size (RGB: the reference has no SH)."""
    cfg, extra = P.baseline_config(idx)
    cfg.with_sh = False
    scene = P.Scene(cfg)
    rc, rextra = ref.baseline(idx)
    rs = ref.RefScene(rc, rextra["origin_instance"])
    if extra["origin_instance"]:
        P.place_origin_instance(scene)
    assert_same_inputs(scene, rs)
    o = orc.from_scene(scene)
    t = extra["time_s"]
    rep = assert_same_frame(o, rs, cfg, 16, o.render(t, orc.settings(sh_colour=False)), rs.render(t, ref.settings()))
    assert rep["S"] > 90_000


def test_reference_psnr_matches_host_psnr():
    rng = np.random.default_rng(3)
    a = rng.random((20, 30, 3), dtype=np.float32)
    b = (a + rng.normal(0, 0.01, a.shape)).astype(np.float32)
    assert abs(ref.psnr(a, b) - P.psnr(a, b)) < 1e-4
    assert ref.psnr(a, a) == 99.0
