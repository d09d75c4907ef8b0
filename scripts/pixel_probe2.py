import sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2501_17792_b200 as P
from paper_2501_17792_b200 import native as N
from oracle import orc
libm = ctypes.CDLL("libm.so.6"); libm.logf.restype = ctypes.c_float; libm.logf.argtypes = [ctypes.c_float]
libm.expf.restype = ctypes.c_float; libm.expf.argtypes = [ctypes.c_float]
cfg, ex = P.baseline_config(2)
scene = P.Scene(cfg)
r = P.Renderer(scene); r.set_debug(N.GSCG_DEBUG_RECORDS)
st = P.RenderSettings(background=(0.1, 0.1, 0.15))
rgb, T = r.render_frame(0.0, st)
rec = r.splat_records()
ords = r.sorted_ordinals()
W = cfg.width; tiles_x = (W + 15) // 16; tiles_y = (cfg.height + 15)//16
ranges = r.tile_ranges(tiles_x * tiles_y)
f32 = np.float32
cut = f32(1) / f32(255)
for (py, px) in [(418, 68), (410, 125)]:
    tile = (py // 16) * tiles_x + px // 16
    a, b = ranges[tile]
    lst = ords[a:b]
    pos = np.searchsorted(rec["ordinal"], lst)
    print("pixel", py, px, "tile", tile, "len", b - a, "gpuT", T[py, px])
    t = f32(1)
    for i in pos:
        s = rec[i]
        x0, y0, x1, y1 = s["rect"]
        if not (x0 <= px < x1 and y0 <= py < y1): continue
        dx = f32(px) + f32(0.5) - s["mean_px"][0]; dy = f32(py) + f32(0.5) - s["mean_px"][1]
        ca, cb, cc = s["conic"]
        det = s["cov_xx"] * s["cov_yy"] - s["cov_xy"] * s["cov_xy"]; inv = f32(1) / det
        ca2, cb2, cc2 = s["cov_yy"] * inv, -s["cov_xy"] * inv, s["cov_xx"] * inv
        power = f32(-0.5) * (ca * dx * dx + cc * dy * dy) - cb * dx * dy
        pf_host = libm.logf(float(cut / s["opacity"]))
        if power >= s["power_floor"] - 1 or power >= pf_host - 1:
            alpha = min(s["opacity"] * libm.expf(float(power)), 0.99)
            print(f"  ord {s['ordinal']} power {power!r} pf_gpu {s['power_floor']!r} pf_host {f32(pf_host)!r} conic_eq {(ca,cb,cc)==(ca2,cb2,cc2)} pass {power >= s['power_floor']} alpha {alpha:.5f} T {t}")
            if power >= pf_host:
                t = t * (f32(1) - f32(alpha))
    print("  replay T", t)
