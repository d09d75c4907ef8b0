"""Dev probe: render one small scene on the GPU and diff every stage against the oracle."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2501_17792_b200 as P
from paper_2501_17792_b200 import native as N
from oracle import orc

def probe(cfg, time_s=0.37, ts=16, bg=(0.1, 0.1, 0.15), forced=None, static=False):
    scene = P.Scene(cfg)
    r = P.Renderer(scene)
    r.set_debug(N.GSCG_DEBUG_POSED | N.GSCG_DEBUG_RECORDS)
    st = P.RenderSettings(tile_size=ts, background=bg)
    t0 = time.time(); rgb, T = r.render_frame(time_s, st, static, forced); t1 = time.time()
    o = orc.from_scene(scene)
    orgb, oT, ot = o.render(time_s, orc.settings(tile_size=ts, background=bg), static, forced)
    n = scene.counts()[2]
    print("render s", t1 - t0)
    print("lod eq", np.array_equal(r.lods(), o.lods(n)))
    g, s, k = r.counts()
    print("counts gpu", (g, s, k), "orc", (ot.gaussian_count, ot.splat_count, ot.pair_count))
    pm, opm = r.posed_means(), o.posed()
    if pm.shape == opm.shape:
        print("posed bit-eq", np.array_equal(pm.view(np.uint32), opm.view(np.uint32)), "maxabs", np.abs(pm - opm).max())
    rec = r.splat_records()
    osp = o.splats()
    base = r.instance_base()
    oord = base[osp["instance_id"]] + osp["gaussian_index"]
    order = np.argsort(oord)
    os_ = osp[order]
    if len(rec) == len(os_):
        print("ordinals eq", np.array_equal(rec["ordinal"], oord[order]))
        for f in ["depth", "cov_xx", "cov_xy", "cov_yy"]:
            print(f, "bit-eq", np.array_equal(rec[f].view(np.uint32), os_[f].view(np.uint32)))
        print("mean eq", np.array_equal(rec["mean_px"].view(np.uint32), os_["mean_px"].view(np.uint32)))
        print("rect eq", np.array_equal(rec["rect"], os_["rect"]))
        print("color maxabs", np.abs(rec["color"] - os_["color"]).max())
    tiles_x = (cfg.width + ts - 1) // ts; tiles_y = (cfg.height + ts - 1) // ts
    ranges = r.tile_ranges(tiles_x * tiles_y)
    counts, items = o.bins(tiles_x * tiles_y)
    print("tile counts eq", np.array_equal(ranges[:, 1] - ranges[:, 0], counts))
    sorted_ord = r.sorted_ordinals()
    oitems_ord = oord[items]  # items index into sorted splat array
    # build per tile lists in gpu order
    ok = True
    pos = 0
    for t in range(tiles_x * tiles_y):
        a, b = ranges[t]
        c = counts[t]
        if c and not np.array_equal(sorted_ord[a:b], oitems_ord[pos:pos + c]):
            ok = False; print("tile list mismatch at", t); break
        pos += c
    print("tile lists eq", ok)
    err = np.abs(rgb - orgb).max(); terr = np.abs(T - oT).max()
    mse = np.mean((rgb.astype(np.float64) - orgb) ** 2)
    print("pixel maxabs", err, "T maxabs", terr, "psnr", 10 * np.log10(1 / mse) if mse > 0 else 99)

if __name__ == "__main__":
    cfg = P.SceneConfig(template_count=2, level_counts=(4000, 900, 200), with_sh=True, motion_count=2, motion_frames=60,
                        grid_rows=3, grid_cols=3, crowd_count=9, crowd_seed=7, cam_pos=(1.0, 1.5, -3.0),
                        cam_look=(1.0, 1.0, 4.0), width=320, height=240, lod_thresholds=(3.5, 5.0))
    probe(cfg)
    probe(cfg, ts=7)
    cfg1, ex = P.baseline_config(2)
    probe(cfg1, time_s=0.0)
