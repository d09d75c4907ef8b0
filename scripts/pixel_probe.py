import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2501_17792_b200 as P
from oracle import orc
cfg, ex = P.baseline_config(2)
scene = P.Scene(cfg)
r = P.Renderer(scene)
st = P.RenderSettings(background=(0.1, 0.1, 0.15))
rgb, T = r.render_frame(0.0, st)
o = orc.from_scene(scene)
orgb, oT, ot = o.render(0.0, orc.settings(background=(0.1, 0.1, 0.15)))
d = np.abs(rgb - orgb).max(axis=2)
idx = np.argwhere(d > 1e-4)
print("pixels >1e-4:", len(idx), ">1e-3:", int((d > 1e-3).sum()))
order = np.argsort(-d[idx[:, 0], idx[:, 1]])
for (y, x) in idx[order][:15]:
    print(y, x, "err", d[y, x], "T gpu", T[y, x], "T orc", oT[y, x], "rgb", rgb[y, x], orgb[y, x])
np.save("gpurun_out/worst.npy", idx[order][:50])
