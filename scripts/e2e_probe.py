"""Breakdown of the end-to-end frame (public API) at config 3: wall time per call and the
stage times the API reports, blocking and pipelined."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2501_17792_b200 as P

    cfg, extra = P.baseline_config(3)
    scene = P.Scene(cfg)
    r = P.Renderer(scene, device_poses=True)
    st = P.RenderSettings()
    out = (r.alloc_frame(pinned=True)[0], None)
    for f in range(5):
        r.render_frame(f / 30.0, st, out=out)
    for label, kw in (("pinned rgb", {"out": out}), ("pinned rgb+T", {"out": r.alloc_frame(True)}),
                      ("fresh arrays", {})):
        t = []
        times = P.StageTimes()
        for f in range(30):
            t0 = time.perf_counter()
            r.render_frame(f / 30.0, st, times=times, **kw)
            t.append(time.perf_counter() - t0)
        ms = 1e3 * np.median(t)
        print(f"{label:14s} wall {ms:.3f} ms ({1e3 / ms:.1f} FPS)  pose/host {times.pose_ms:.3f}  update {times.update_ms:.3f} "
              f"gather {times.gather_ms:.3f} sort {times.sort_ms:.3f} raster+readback {times.rasterize_ms:.3f}")
    outs = [(r.alloc_frame(pinned=True)[0], None) for _ in range(2)]
    for mode in ("pipelined", "pipelined again"):
        t = []
        t_all = time.perf_counter()
        for f in range(60):
            t0 = time.perf_counter()
            r.render_frame(f / 30.0, st, out=outs[f & 1], pipelined=True)
            t.append(time.perf_counter() - t0)
        r.wait_readback(0)
        tot = time.perf_counter() - t_all
        print(f"{mode:14s} per call median {1e3 * np.median(t):.3f} ms  loop {1e3 * tot / 60:.3f} ms/frame")


if __name__ == "__main__":
    main()
