"""Minimal profiling target: N config-3 frames through gscg_render_frame with device-resident
inputs (no e2e / CPU legs), for ncu captures of the frame's kernels.

  python scripts/profile_frame.py --frames 3 [--config 3] [--warmup 2]

Warm-up frames (which grow the buffers to their high-water mark) run outside the profiler
range (cudaProfilerStart/Stop): capture with ncu --profile-from-start off to see one
clean launch of every kernel per frame.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import gscg_settings

    cfg, extra = P.baseline_config(args.config)
    scene = P.Scene(cfg)
    if extra["origin_instance"]:
        P.place_origin_instance(scene)
    r = P.Renderer(scene, device=0, device_poses=True)
    r.prepare()  # templates + motion tables
    n = scene.counts()[2]
    dev = torch.device("cuda", 0)
    rec = r.instance_records()
    d_tids = torch.from_numpy(rec["template_ids"].view(np.int32)).to(dev)
    d_place = torch.from_numpy(rec["placement"]).to(dev)
    d_mid = torch.from_numpy(rec["motion_ids"].view(np.int32)).to(dev)
    d_phase = torch.from_numpy(rec["phase_offsets"]).to(dev)
    d_lods = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
    cam = scene.camera_basis()
    rs = gscg_settings(P.RenderSettings())
    lp = N.GscgLodPolicy()
    lp.threshold_count = len(cfg.lod_thresholds)
    for i, v in enumerate(cfg.lod_thresholds):
        lp.thresholds_m[i] = v
    fd = N.GscgFrameDesc()
    fd.instance_count = n
    fd.joint_stride = r.joint_stride
    fd.template_ids, fd.placement = d_tids.data_ptr(), d_place.data_ptr()
    fd.active_lod = d_lods.data_ptr()
    fd.forced_lod = -1 if extra["forced_lod"] is None else extra["forced_lod"]
    fd.memory = N.GSCG_MEM_DEVICE
    fd.pose_source = N.GSCG_POSES_SAMPLED  # poses sampled on the device, as bench.py
    fd.motion_ids, fd.phase_offsets = d_mid.data_ptr(), d_phase.data_ptr()
    lib = N.gscg()
    for f in range(args.warmup + args.frames):
        if f == args.warmup:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        fd.time_s = extra["time_s"] + f / 30.0
        st = N.GscgStageTimes()
        N.check_gscg(lib.gscg_render_frame(r.gpu, C.byref(fd), C.byref(cam), C.byref(rs), C.byref(lp), None, None,
                                           C.byref(st)), r.gpu)
        print(f"frame {f}: update {st.update_ms:.3f} gather {st.gather_ms:.3f} sort {st.sort_ms:.3f} "
              f"raster {st.rasterize_ms:.3f} S={st.splat_count} K={st.pair_count} launches={st.kernel_launches}")
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
