"""Stage functions on the GPU (reference renderer.hpp:81-103: gather_splats, sort_splats,
rasterize_full) through the C-ABI, against the oracle and the reference's own stage
tests: sort vs a stable comparison sort with duplicated depths (test_renderer.cpp:89-123)
and the tiled raster vs the naive per-pixel loop (test_renderer.cpp:175-194)."""
import numpy as np
import pytest

import paper_2501_17792_b200 as P
from oracle import orc
from tests.parity import PIXEL_TOL, psnr
from tests.test_oracle import random_frame, raster, sort_splats

pytestmark = pytest.mark.gpu


def scene():
    cfg = P.SceneConfig(template_count=2, template_seed_base=100, level_counts=(3000, 700, 150), with_sh=True,
                        motion_count=2, motion_frames=40, grid_rows=3, grid_cols=3, crowd_count=9, crowd_seed=4,
                        cam_pos=(1.0, 1.5, -3.0), cam_look=(1.0, 1.0, 4.0), width=256, height=176,
                        lod_thresholds=(3.5, 5.0))
    return P.Scene(cfg)


def test_gather_splats_equals_oracle_projection():
    s = scene()
    r = P.Renderer(s)
    g = r.gather_splats(0.3)
    o = orc.from_scene(s)
    o.render(0.3, orc.settings(sh_colour=True))
    ref = o.splats()  # sorted; back to (instance, gaussian) order
    ref = ref[np.lexsort((ref["gaussian_index"], ref["instance_id"]))]
    assert len(g) == len(ref) > 1000
    for f in ("instance_id", "gaussian_index", "mean_px", "cov_xx", "cov_xy", "cov_yy", "depth", "rect", "opacity"):
        assert g[f].tobytes() == ref[f].tobytes(), f
    assert np.abs(g["color"] - ref["color"]).max() <= 1e-5
    # the crowd's LoD state follows the update, as update_crowd sets it
    assert np.array_equal(s.instances["active_lod"], o.lods(9))


def test_sort_splats_matches_oracle_and_stable_comparison_sort():
    s = scene()
    r = P.Renderer(s)
    g = r.gather_splats(0.8)
    rng = np.random.default_rng(3)
    shuffled = g[rng.permutation(len(g))]
    got = r.sort_splats(shuffled)
    assert got.tobytes() == sort_splats(g).tobytes()
    # duplicated depths across instances (reference test_renderer.cpp:89-123)
    fr = random_frame(np.random.default_rng(19), 128, 128, 300)
    fr["depth"][1::8] = fr["depth"][0::8][: len(fr["depth"][1::8])]
    ref = sorted(range(len(fr)), key=lambda i: (fr["depth"][i], fr["instance_id"][i], fr["gaussian_index"][i]))
    out = r.sort_splats(fr)
    assert np.array_equal(out["instance_id"], fr["instance_id"][ref])
    assert np.array_equal(out["gaussian_index"], fr["gaussian_index"][ref])
    assert r.sort_splats(fr[:1]).tobytes() == fr[:1].tobytes() and len(r.sort_splats(fr[:0])) == 0


@pytest.mark.parametrize("tile", [16, 8, 5, 32])
def test_rasterize_full_matches_oracle_raster(tile):
    s = scene()
    r = P.Renderer(s)
    frame = sort_splats(r.gather_splats(0.55))
    st = P.RenderSettings(tile_size=tile, background=(0.1, 0.2, 0.3))
    rgb, T = r.rasterize_full(frame, 256, 176, st)
    ost = orc.settings(tile_size=tile, background=(0.1, 0.2, 0.3))
    orgb, oT = raster(frame, 256, 176, ost)
    assert np.abs(rgb - orgb).max() <= PIXEL_TOL and np.abs(T - oT).max() <= PIXEL_TOL
    assert psnr(rgb, orgb) >= 50.0
    # the full-frame path renders the same image
    full, _ = r.render_frame(0.55, st)
    assert np.abs(full - rgb).max() <= 1e-6


def test_rasterize_random_frames_match_naive_loop():
    rng = np.random.default_rng(101)
    r = P.Renderer(scene())
    for _ in range(4):
        w, h = 96 + int(rng.integers(64)), 64 + int(rng.integers(48))
        fr = sort_splats(random_frame(rng, w, h, 80 + int(rng.integers(421))))
        tile = 1 + int(rng.integers(40))
        bg = tuple(float(x) for x in rng.uniform(0, 1, 3))
        rgb, T = r.rasterize_full(fr, w, h, P.RenderSettings(tile_size=tile, background=bg))
        nrgb, nT = raster(fr, w, h, orc.settings(tile_size=tile, background=bg), naive=True)
        assert np.abs(rgb - nrgb).max() <= PIXEL_TOL and np.abs(T - nT).max() <= PIXEL_TOL


def test_rasterize_empty_frame_is_background():
    r = P.Renderer(scene())
    rgb, T = r.rasterize_full(np.zeros(0, P.api.FRAME_SPLAT_DTYPE), 33, 17,
                              P.RenderSettings(background=(0.2, 0.4, 0.6)))
    assert np.all(rgb[..., 0] == np.float32(0.2)) and np.all(T == 1.0)
