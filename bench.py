"""Headline benchmark: FPS of the crowd render path at BASELINE config 3 (14 templates x
3,500 animated characters, 3-level distance LoD, SH-3 colour, 1920x1080) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one full render_frame (LoD + FK + skinning + projection + sort + raster) of a
distinct animation time t = f/30 s. `value` times K steps with every input already in HBM
(poses sampled and uploaded before the timed region) using CUDA events on the render
stream; `e2e` times the public API (host pose sampling, pinned H2D, kernels, D2H of the
framebuffer) per step. `--impl reference` times the CPU oracle (the reference's render
path restated in C++, reference/oracle "port") on the host cores. Multi-GPU runs split the
instances across ranks (each rank renders its shard's frame; no data-path collective yet,
see DESIGN.md "Multi-GPU"), timing max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FPS at 3,500 chars 1080p (1/2/4/8 B200); splats/sec vs HBM roofline"
PROFILE_SUMMARY = ROOT / "profiles" / "ncu_summary.json"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def build_scene(config: int, rank: int, world: int):
    import paper_2501_17792_b200 as P

    cfg, extra = P.baseline_config(config)
    scene = P.Scene(cfg)
    if extra["origin_instance"]:
        P.place_origin_instance(scene)
    if world > 1:
        inst = scene.instances
        lo = len(inst) * rank // world
        hi = len(inst) * (rank + 1) // world
        scene.instances = inst[lo:hi]
    return P, cfg, extra, scene


def roofline_bytes(cfg, counts, lods, scene, sh: bool) -> dict:
    """Algorithmic bytes (SURVEY.md §8d / DESIGN.md) for the frame and its two big kernels."""
    G, S, K = counts
    a = 256 if sh else 76
    inst = scene.instances
    resident = set(zip(inst["template_id"].tolist(), lods.tolist()))
    A = sum(cfg.level_counts[l] for _, l in resident) * a
    n = len(inst)
    M = n * 24 * 48
    R = 48
    W, H = cfg.width, cfg.height
    tiles = ((W + 15) // 16) * ((H + 15) // 16)
    P = 6
    frame = A + M + 2 * S * R + K * (12 + 24 * P + 4) + 16 * W * H
    project = A + M + S * (R + 4) + K * 12          # template stream + matrices + records/ordinals + pairs
    raster = K * (4 + R) + 16 * W * H + tiles * 8  # sorted values + record gathers + framebuffer
    return {"frame": frame, "project": project, "raster": raster, "A": A, "M": M}


def run_ours(args, rank, world, local_rank) -> dict | None:
    import torch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    P, cfg, extra, scene = build_scene(args.config, rank, world)
    from paper_2501_17792_b200 import native as N

    r = P.Renderer(scene, device=local_rank)
    settings = P.RenderSettings()
    n = scene.counts()[2]
    js = r.joint_stride
    forced = extra["forced_lod"]
    frames = args.warmup + args.steps
    t0 = extra["time_s"]
    times_s = [t0 + f / 30.0 for f in range(frames)]

    # ---- device-resident inputs: sample all poses on the host up front, upload once ----
    tids, place, _ = r.sample_crowd(times_s[0])
    poses_host = np.stack([r.sample_crowd(t)[2] for t in times_s])
    dev = torch.device("cuda", local_rank)
    d_tids = torch.from_numpy(tids.view(np.int32)).to(dev)
    d_place = torch.from_numpy(place).to(dev)
    d_poses = torch.from_numpy(poses_host).to(dev)
    d_lods = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
    cam = scene.camera_basis()
    rs = N.GscgRenderSettings()
    rs.tile_size = settings.tile_size
    rs.alpha_max, rs.alpha_cutoff, rs.transmittance_floor = settings.alpha_max, settings.alpha_cutoff, settings.transmittance_floor
    rs.sh_enabled = 1
    lp = N.GscgLodPolicy()
    lp.threshold_count = len(cfg.lod_thresholds)
    for i, v in enumerate(cfg.lod_thresholds):
        lp.thresholds_m[i] = v
    lp.hysteresis_band_m = cfg.lod_hysteresis
    lib = N.gscg()
    ctx = r.gpu
    stream_ptr = C.c_void_p()
    N.check_gscg(lib.gscg_stream(ctx, C.byref(stream_ptr)), ctx)
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=dev)

    def frame(f: int, st: N.GscgStageTimes):
        fd = N.GscgFrameDesc()
        fd.instance_count = n
        fd.joint_stride = js
        fd.template_ids = d_tids.data_ptr()
        fd.placement = d_place.data_ptr()
        fd.poses = d_poses[f].data_ptr()
        fd.active_lod = d_lods.data_ptr()
        fd.forced_lod = -1 if forced is None else forced
        fd.memory = N.GSCG_MEM_DEVICE
        N.check_gscg(lib.gscg_render_frame(ctx, C.byref(fd), C.byref(cam), C.byref(rs), C.byref(lp), None, None,
                                           C.byref(st)), ctx)

    stage = []
    for f in range(args.warmup):
        st = N.GscgStageTimes()
        frame(f, st)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for f in range(args.warmup, frames):
            st = N.GscgStageTimes()
            frame(f, st)
            stage.append(st)
            launches += st.kernel_launches
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    if dist:
        dist.barrier()
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    counts = (stage[-1].gaussian_count, stage[-1].splat_count, stage[-1].pair_count)
    lods = d_lods[:n].cpu().numpy().astype(np.uint32)

    # ---- end-to-end through the public API (host poses + pinned H2D + kernels + D2H) ----
    e2e_times = []
    for f in range(min(args.warmup, 2)):
        r.render_frame(times_s[f], settings, forced_lod=forced)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t_start = time.perf_counter()
    for f in range(args.warmup, frames):
        r.render_frame(times_s[f], settings, forced_lod=forced)
    e2e_s = time.perf_counter() - t_start
    if dist:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_fps = args.steps / e2e_s
    h2d = n * 4 + n * 16 + n * (4 + 4 * js) * 4 + n * 4
    d2h = cfg.width * cfg.height * 16 + n * 4

    if dist:
        tot = torch.tensor(list(counts), dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        counts = tuple(int(x) for x in tot.tolist())
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    peaks = _peaks()
    med = lambda attr: float(np.median([getattr(s, attr) for s in stage]))
    stage_ms = {k: med(k + "_ms") for k in ("update", "gather", "sort", "rasterize")}
    rb = roofline_bytes(cfg, counts, lods, scene, sh=True)
    dom = "rasterize" if stage_ms["rasterize"] >= stage_ms["gather"] else "gather"
    kernel = {"rasterize": "k_raster16q", "gather": "k_project"}[dom]
    kbytes = rb["raster"] if dom == "rasterize" else rb["project"]
    achieved = kbytes / (stage_ms[dom] * 1e-3) / 1e9
    traffic = None
    if PROFILE_SUMMARY.exists():
        try:
            prof = json.loads(PROFILE_SUMMARY.read_text())
            traffic = prof.get("kernels", {}).get(kernel, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    fps = 1000.0 / ms_step
    frame_roofline_ms = rb["frame"] / (peaks["hbm_gbs"] * 1e9) * 1e3
    out = {
        "metric": METRIC, "value": round(fps, 3), "unit": "FPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"BASELINE config {args.config}: 14 synthetic templates (202738/12661/3176 G, SH deg 3) x "
                               f"{cfg.crowd_count} animated characters, distance LoD 5/10 m, {cfg.width}x{cfg.height}, tile 16",
                   "instances": cfg.crowd_count, "resolution": [cfg.width, cfg.height],
                   "gaussians": counts[0], "splats": counts[1], "pairs": counts[2],
                   "l2": "per-frame working set (templates ~0.5 GB + records/pairs ~0.8 GB) exceeds the 126 MB L2",
                   "parallelism": f"instance shards x{world}" if world > 1 else "single GPU"},
        "splats_per_s": round(counts[1] * fps, 1),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "frame_roofline": {"bytes": rb["frame"], "ms": round(frame_roofline_ms, 4),
                           "frac": round(frame_roofline_ms / ms_step, 4), "peak_gbs": peaks["hbm_gbs"]},
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
                     "algorithmic_bytes": kbytes, "peak_source": peaks["source"]},
        "e2e": {"value": round(e2e_fps, 3), "unit": "FPS", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(scene, args.config, frames_sample=args.cpu_frames)
    if dist:
        dist.destroy_process_group()
    return out


def cpu_baseline(scene, config: int, frames_sample: int = 2, threads: int = 0) -> dict:
    """The reference render path restated in C++ (oracle/), timed on this host's cores."""
    from oracle import orc

    P_cfg = scene.cfg
    o = orc.from_scene(scene)
    st = orc.settings(sh_colour=True)
    cores = threads or (os.cpu_count() or 1)
    o.render(0.0, st, threads=cores)  # warm-up frame
    t0 = time.perf_counter()
    for f in range(frames_sample):
        o.render((f + 1) / 30.0, st, threads=cores)
    dt = (time.perf_counter() - t0) / frames_sample
    return {"value": round(1.0 / dt, 4), "unit": "FPS", "cores": cores, "kind": "port",
            "sample": f"{frames_sample} full frames of config {config} ({P_cfg.crowd_count} chars, "
                      f"{P_cfg.width}x{P_cfg.height}) after 1 warm-up frame, std::thread static partition as "
                      f"parallel.hpp, single-threaded sort/bin as renderer.cpp"}


def run_reference(args, rank, world) -> dict | None:
    if rank != 0:
        return None
    import paper_2501_17792_b200 as P
    from oracle import orc

    cfg, extra = P.baseline_config(args.config)
    scene = P.Scene(cfg)
    if extra["origin_instance"]:
        P.place_origin_instance(scene)
    o = orc.from_scene(scene)
    st = orc.settings(sh_colour=True)
    cores = os.cpu_count() or 1
    forced = extra["forced_lod"]
    # Bounded: at most 2 warm-up frames, and the timed steps capped so the run stays in minutes.
    for f in range(min(args.warmup, 2)):
        o.render(extra["time_s"] + f / 30.0, st, forced_lod=forced, threads=cores)
    t0 = time.perf_counter()
    per = []
    steps_run = 0
    for f in range(args.steps):
        s0 = time.perf_counter()
        _, _, times = o.render(extra["time_s"] + (args.warmup + f) / 30.0, st, forced_lod=forced, threads=cores)
        per.append(time.perf_counter() - s0)
        steps_run += 1
        if time.perf_counter() - t0 > args.reference_budget_s:
            break
    ms = float(np.mean(per)) * 1e3
    fps = 1000.0 / ms
    return {"metric": METRIC, "value": round(fps, 4), "unit": "FPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"BASELINE config {args.config} ({cfg.crowd_count} chars, {cfg.width}x{cfg.height})",
                       "splats": int(times.splat_count), "pairs": int(times.pair_count)},
            "cpu_baseline": {"value": round(fps, 4), "unit": "FPS", "cores": cores, "kind": "port",
                             "sample": f"{steps_run} of {args.steps} requested full frames (time budget "
                                       f"{args.reference_budget_s:.0f} s) on {cores} host threads"},
            "e2e": {"value": round(fps, 4), "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-frames", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reference-budget-s", type=float, default=150.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local_rank = dist_env()
    out = run_reference(args, rank, world) if args.impl == "reference" else run_ours(args, rank, world, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
