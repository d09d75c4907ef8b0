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
    rg = r.cell_ranges()
    c = (rg[:, 1] - rg[:, 0]).astype(np.int64)
    print(f"config {idx}: K={st.pair_count} cells={len(c)} nonzero={int((c>0).sum())} >2048={int((c>2048).sum())} >16384={int((c>16384).sum())} max={int(c.max())}")
    print("  pct 50/90/99/99.9:", [int(np.percentile(c[c>0], q)) for q in (50, 90, 99, 99.9)],
          " pairs in >2048:", int(c[c > 2048].sum()), " in >16384:", int(c[c > 16384].sum()))
