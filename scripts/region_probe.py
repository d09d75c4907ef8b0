"""Probe: one column region of the 8-GPU region split (config 3, cols [800, 992), the
slowest region of profiles/r02f_bench.log's band_split_estimate) rendered alone: frame
interval on the device, host time per gscg_render_frame call, and with the whole frame
for comparison. Run under ncu for the region's kernel list."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_17792_b200 as P
from paper_2501_17792_b200 import native as N
from paper_2501_17792_b200.multigpu import gscg_settings

cfg, extra = P.baseline_config(3)
scene = P.Scene(cfg)
if extra["origin_instance"]:
    P.place_origin_instance(scene)
dev = torch.device("cuda", 0)
rends = [P.Renderer(scene, device=0, device_poses=True)]
st = P.RenderSettings()
for r in rends:
    r.render_frame(extra["time_s"], st)
tids, place, _ = rends[0].sample_crowd(extra["time_s"])
inst = scene.instances
n = len(inst)
d_tids = torch.from_numpy(tids.view(np.int32)).to(dev)
d_place = torch.from_numpy(place).to(dev)
d_mid = torch.from_numpy(np.ascontiguousarray(inst["motion_id"]).astype(np.int32)).to(dev)
d_phase = torch.from_numpy(np.ascontiguousarray(inst["phase_offset_s"]).astype(np.float32)).to(dev)
d_lods = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
cam = scene.camera_basis()
rs = gscg_settings(st)
lp = N.GscgLodPolicy()
lp.threshold_count = len(cfg.lod_thresholds)
for i, v in enumerate(cfg.lod_thresholds):
    lp.thresholds_m[i] = v
lp.hysteresis_band_m = cfg.lod_hysteresis
lib = N.gscg()


def fd_for(t):
    fd = N.GscgFrameDesc()
    fd.instance_count = n
    fd.joint_stride = rends[0].joint_stride
    fd.template_ids = d_tids.data_ptr()
    fd.placement = d_place.data_ptr()
    fd.active_lod = d_lods.data_ptr()
    fd.forced_lod = -1
    fd.memory = N.GSCG_MEM_DEVICE
    fd.pose_source = N.GSCG_POSES_SAMPLED
    fd.time_s = t
    fd.motion_ids = d_mid.data_ptr()
    fd.phase_offsets = d_phase.data_ptr()
    return fd




def run(region, frames=60):
    c = rends[0].gpu
    N.check_gscg(lib.gscg_set_region(c, *region), c)
    ts = [extra["time_s"] + f / 30.0 for f in range(frames + 5)]
    for f in range(5):
        N.check_gscg(lib.gscg_render_frame(c, C.byref(fd_for(ts[f])), C.byref(cam), C.byref(rs), C.byref(lp),
                                           None, None, None), c)
    lib.gscg_synchronize(c)
    host = []
    t0 = time.perf_counter()
    for f in range(5, frames + 5):
        h0 = time.perf_counter()
        N.check_gscg(lib.gscg_render_frame(c, C.byref(fd_for(ts[f])), C.byref(cam), C.byref(rs), C.byref(lp),
                                           None, None, None), c)
        host.append(time.perf_counter() - h0)
    lib.gscg_synchronize(c)
    wall = (time.perf_counter() - t0) / frames
    N.check_gscg(lib.gscg_set_region(c, 0, 0, 0, 0), c)
    return wall * 1e3, float(np.median(host)) * 1e3


frames = int(sys.argv[1]) if len(sys.argv) > 1 else 60
for name, region in (("whole frame", (0, 0, 0, 0)), ("cols 800-992", (800, 0, 992, 0))):
    wall, host = run(region, frames)
    print(f"{name}: {wall:.3f} ms per frame (wall), host call median {host:.3f} ms")
