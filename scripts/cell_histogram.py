import numpy as np, sys
sys.path.insert(0, '.')
import paper_2501_17792_b200 as P
cfg, extra = P.baseline_config(3)
s = P.Scene(cfg)
r = P.Renderer(s, device_poses=True)
r.render_frame(extra["time_s"], P.RenderSettings(), forced_lod=extra["forced_lod"])
rg = r.cell_ranges()
n = (rg[:, 1].astype(np.int64) - rg[:, 0]).clip(0)
print("cells", len(n), "pairs", n.sum(), "max", n.max(), "mean", n.mean())
for lo, hi in [(0,1),(1,64),(64,256),(256,1024),(1024,2048),(2048,4096),(4096,8192),(8192,16384),(16384,1<<30)]:
    m = (n >= lo) & (n < hi)
    print(f"[{lo},{hi}) cells {m.sum()} pairs {n[m].sum()} ({n[m].sum()/n.sum():.3f})")
