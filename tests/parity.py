"""GPU-vs-oracle parity checks shared by the GPU tests and smoke().

Bars (BASELINE.json north_star): LoD, splat set, depth bits, rects, tile ranges and the
per-tile (sort) order bit-exact; skinned positions within 1e-3 (they are in fact
bit-identical and checked as such); pixels max abs <= 1e-3 per channel and PSNR >= 50 dB
(they are bit-identical too with RGB colour, and T always: checked as such).
"""
from __future__ import annotations

import numpy as np

from paper_2501_17792_b200 import native as N

PIXEL_TOL = 1e-3
PSNR_MIN = 50.0


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """metrics.cpp:8-23 (double accumulation, cap 99 dB)."""
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return 99.0 if mse == 0 else min(99.0, 10.0 * np.log10(1.0 / mse))


def render_both(scene, renderer, oracle_scene, time_s=0.0, tile_size=16, background=(0.0, 0.0, 0.0),
                static_pose=False, forced_lod=None, sh=True, debug=True):
    import paper_2501_17792_b200 as P
    from oracle import orc

    if debug:
        renderer.set_debug(N.GSCG_DEBUG_POSED | N.GSCG_DEBUG_RECORDS)
    st = P.RenderSettings(tile_size=tile_size, background=background, sh_colour=sh)
    rgb, T = renderer.render_frame(time_s, st, static_pose, forced_lod)
    orgb, oT, times = oracle_scene.render(time_s, orc.settings(tile_size=tile_size, background=background,
                                                               sh_colour=sh), static_pose, forced_lod)
    return (rgb, T), (orgb, oT, times)


def check_frame(scene, renderer, oracle_scene, gpu_out, orc_out, tile_size=16, full=True) -> dict:
    rgb, T = gpu_out
    orgb, oT, times = orc_out
    n = scene.counts()[2]
    cfg = scene.cfg
    report = {}
    lods = renderer.lods()
    assert np.array_equal(lods, oracle_scene.lods(n)), "LoD selection differs"
    G, S, K = renderer.counts()
    assert (G, S) == (times.gaussian_count, times.splat_count), \
        f"counts G/S gpu {(G, S)} oracle {(times.gaussian_count, times.splat_count)}"
    if renderer.cell_layout()[1] == 1:
        assert K == times.pair_count, f"pairs gpu {K} oracle {times.pair_count}"
    last = getattr(renderer, "last_times", None)
    if last is not None:  # the reference's (tile, splat) bin entries, counted by k_project
        assert last.tile_pair_count == times.pair_count, \
            f"tile pairs gpu {last.tile_pair_count} oracle {times.pair_count}"
    report.update(G=G, S=S, K=K)
    if full:
        pm, opm = renderer.posed_means(), oracle_scene.posed()
        assert pm.shape == opm.shape
        if len(pm):
            err = float(np.abs(pm - opm).max())
            assert err <= 1e-3, f"posed means max abs {err}"
            assert pm.tobytes() == opm.tobytes(), "posed means are not bit-identical"
        rec = renderer.splat_records()
        osp = oracle_scene.splats()
        base = renderer.instance_base()
        oord = base[osp["instance_id"]].astype(np.int64) + osp["gaussian_index"]
        by_ord = np.argsort(oord, kind="stable")
        o_sorted = osp[by_ord]
        assert np.array_equal(rec["ordinal"], oord[by_ord]), "surviving splat set differs"
        for f in ("depth", "cov_xx", "cov_xy", "cov_yy"):
            assert rec[f].tobytes() == o_sorted[f].tobytes(), f"{f} not bit-identical"
        assert rec["mean_px"].tobytes() == o_sorted["mean_px"].tobytes(), "mean_px not bit-identical"
        assert np.array_equal(rec["rect"], o_sorted["rect"]), "pixel rects differ"
        if len(rec):
            report["color_max_abs"] = float(np.abs(rec["color"] - o_sorted["color"]).max())
            assert report["color_max_abs"] <= 1e-5
        report["colors_exact"] = rec["color"].tobytes() == o_sorted["color"].tobytes()
        tiles_x = (cfg.width + tile_size - 1) // tile_size
        tiles_y = (cfg.height + tile_size - 1) // tile_size
        tiles, cpt = renderer.cell_layout()
        assert tiles == tiles_x * tiles_y
        ranges = renderer.cell_ranges()
        counts, items = oracle_scene.bins(tiles)
        sorted_ord = renderer.sorted_ordinals().astype(np.int64)
        if cpt == 1:
            exp_counts, exp_ord = counts.astype(np.int64), oord[items]
        else:
            # Each 8x8 quadrant cell must hold exactly the reference tile list filtered to
            # the splats whose rect meets the quadrant, in the reference's order.
            tile_of = np.repeat(np.arange(tiles), counts)
            rect = osp["rect"][items]
            tx, ty = tile_of % tiles_x, tile_of // tiles_x
            cell_ids, order, ords = [], [], []
            for q in range(4):
                qx0 = tx * 16 + (q & 1) * 8
                qy0 = ty * 16 + (q >> 1) * 8
                m = (rect[:, 0] < qx0 + 8) & (rect[:, 2] > qx0) & (rect[:, 1] < qy0 + 8) & (rect[:, 3] > qy0)
                cell_ids.append(tile_of[m] * 4 + q)
                order.append(np.nonzero(m)[0])
                ords.append(oord[items[m]])
            cell_ids, order, ords = map(np.concatenate, (cell_ids, order, ords))
            perm = np.lexsort((order, cell_ids))
            exp_ord = ords[perm]
            exp_counts = np.bincount(cell_ids, minlength=tiles * 4)
            lut = np.zeros(max(G, 1), np.int64)
            lut[rec["ordinal"]] = rec["depth"].view(np.uint32)
            tcounts, titems = renderer.tile_lists(lambda o: lut[o])
            assert np.array_equal(tcounts, counts) and np.array_equal(titems, oord[items]), \
                "merged per-tile lists differ from the reference bins"
        assert K == int(exp_counts.sum()), f"cell pairs gpu {K} expected {int(exp_counts.sum())}"
        assert np.array_equal((ranges[:, 1] - ranges[:, 0]).astype(np.int64), exp_counts), "per-cell pair counts differ"
        starts = np.concatenate([[0], np.cumsum(exp_counts)[:-1]])
        nz = exp_counts > 0
        assert np.array_equal(ranges[nz, 0].astype(np.int64), starts[nz]), "cell ranges are not the prefix layout"
        assert np.array_equal(sorted_ord, exp_ord), "per-cell sort order differs"
    diff = np.abs(rgb - orgb)
    report["max_abs"] = float(diff.max()) if diff.size else 0.0
    report["T_max_abs"] = float(np.abs(T - oT).max()) if T.size else 0.0
    report["psnr"] = psnr(rgb, orgb)
    # The blend is single-rounded in the reference order with a bit-exact expf replica
    # (gscg_expf.cuh): T is bit-identical always, and so are the pixels whenever every
    # splat colour is (RGB colour; the SH-3 extension evaluates with FMAs and a hardware
    # rsqrt, within 1e-5 of the oracle, so its pixels are tolerance-checked).
    assert T.tobytes() == oT.tobytes(), "transmittance not bit-identical"
    if report.get("colors_exact"):
        assert rgb.tobytes() == orgb.tobytes(), f"pixels not bit-identical (max abs {report['max_abs']})"
    assert report["max_abs"] <= PIXEL_TOL, f"pixel max abs {report['max_abs']}"
    assert report["T_max_abs"] <= PIXEL_TOL, f"transmittance max abs {report['T_max_abs']}"
    assert report["psnr"] >= PSNR_MIN, f"PSNR {report['psnr']}"
    return report


def check_cull_invariance(renderer, time_s=0.0, settings=None, static_pose=False, forced_lod=None) -> int:
    """The instance frustum cull (k_inst_cull) only drops instances none of whose splats
    can survive gather_splats' cull (renderer.cpp:38-50), so the frame with it must be
    byte-identical to the frame without it: counts, the surviving splat records, the
    per-cell sort order and ranges, pixels and T. Returns the number of culled instances."""
    import paper_2501_17792_b200 as P

    settings = settings or P.RenderSettings()
    out = []
    for flags in (N.GSCG_DEBUG_RECORDS | N.GSCG_DEBUG_NO_CULL, N.GSCG_DEBUG_RECORDS):
        renderer.set_debug(flags)
        rgb, T = renderer.render_frame(time_s, settings, static_pose, forced_lod)
        rec = renderer.splat_records()
        rec = rec[np.argsort(rec["ordinal"], kind="stable")]
        out.append((rgb.copy(), T.copy(), renderer.counts(), rec.tobytes(), renderer.sorted_ordinals().copy(),
                    renderer.cell_ranges().copy(), renderer.instances_culled()))
    (a, b) = out
    assert a[6] == 0, "GSCG_DEBUG_NO_CULL still culled instances"
    assert a[2] == b[2], f"counts with/without cull {b[2]} / {a[2]}"
    assert a[3] == b[3], "surviving splat records differ with the instance cull"
    assert np.array_equal(a[4], b[4]), "per-cell sort order differs with the instance cull"
    assert np.array_equal(a[5], b[5]), "cell ranges differ with the instance cull"
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes(), "pixels differ with the cull"
    return b[6]
