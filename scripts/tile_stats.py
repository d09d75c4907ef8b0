import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2501_17792_b200 as P
for idx in (3, 4):
    cfg, ex = P.baseline_config(idx)
    s = P.Scene(cfg)
    r = P.Renderer(s)
    st = P.StageTimes()
    r.render_frame(0.0, P.RenderSettings(), times=st)
    tx, ty = (cfg.width + 15) // 16, (cfg.height + 15) // 16
    rg = r.tile_ranges(tx * ty)
    c = (rg[:, 1] - rg[:, 0]).astype(np.int64)
    print(f"config {idx}: G={st.gaussian_count} S={st.splat_count} K={st.pair_count} tiles={tx*ty} nonzero={int((c>0).sum())}")
    print("  percentiles 50/90/99/99.9/max:", [int(np.percentile(c, q)) for q in (50, 90, 99, 99.9)], int(c.max()))
    print("  tiles > 4096:", int((c > 4096).sum()), " > 8192:", int((c > 8192).sum()), " > 16384:", int((c > 16384).sum()),
          " pairs in tiles>8192:", int(c[c > 8192].sum()))
    print("  stage ms", st.update_ms, st.gather_ms, st.sort_ms, st.rasterize_ms)
