"""Headline benchmark: FPS of the crowd render path at BASELINE config 3 (14 templates x
3,500 animated characters, 3-level distance LoD, SH-3 colour, 1920x1080) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one full render_frame (LoD + FK + skinning + projection + sort + raster) of a
distinct animation time t = f/30 s. `value` times K steps with every input already in HBM
(poses sampled on the device) using CUDA events on the render stream; `median_frame_ms`
is the median of the per-frame event intervals (the reference's protocol, bench.cpp:74-93).
`e2e` times the public API (instance H2D, kernels, D2H of the framebuffer into pinned
memory) per step, streaming: frame k's read-back overlaps frame k+1; the blocking
one-call-per-frame rate is reported beside it.

`--gpus N` with no torchrun environment re-launches itself under torchrun (N ranks, one per
GPU, NCCL); each rank projects an instance shard, splats are exchanged by screen band and
each rank sorts and rasterises its band; timing is the max over ranks.

`--impl reference` times the REFERENCE's own render_frame on the host cores: its
unmodified sources built against the Eigen-subset shim (oracle/_ref, "kind": "reference";
the oracle port only if that build is missing), from its own synthetic generator and
build_crowd, on every host thread. The `cpu_baseline` of our arm is the same build,
sampled at all threads and at 1 thread.
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
    """SM clocks + clock-event (throttle) reasons sampled every 2 ms during the timed
    region through NVML (nvidia-smi's source); falls back to nvidia-smi -lms 100."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device: int, period_s: float = 0.002):
        self.device = device
        self.period = period_s
        self.sm: list[float] = []
        self.mask = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._smi = None

    def _nvml_index(self) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.device < len(ids) and ids[self.device].isdigit():
                return int(ids[self.device])
        return self.device

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self._stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        self.mask |= int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
        except Exception:
            self._start_smi()
        return self

    def _start_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.hw_power_brake_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            self._smi = subprocess.Popen(["nvidia-smi", "-i", str(self._nvml_index()), f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self._smi = None
            return
        names = list(self.REASONS)

        def read():
            for line in self._smi.stdout:
                parts = [p.strip() for p in line.split(",")]
                try:
                    self.sm.append(float(parts[0]))
                    self.max_mhz = max(self.max_mhz or 0.0, float(parts[1]))
                except (ValueError, IndexError):
                    continue
                for name, v in zip(names, parts[2:7]):
                    if v.lower() == "active":
                        self.mask |= self.REASONS[name]

        self._t = threading.Thread(target=read, daemon=True)
        self._t.start()

    def __exit__(self, *exc):
        self._stop.set()
        if self._smi:
            self._smi.terminate()
            try:
                self._smi.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._smi.kill()
        if self._t:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        reasons = sorted(n for n, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.sm)}


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def dist_env() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def build_scene(config: int):
    import paper_2501_17792_b200 as P

    cfg, extra = P.baseline_config(config)
    scene = P.Scene(cfg)
    if extra["origin_instance"]:
        P.place_origin_instance(scene)
    return P, cfg, extra, scene


def roofline_bytes(cfg, counts, tile_pairs, lods, scene) -> dict:
    """Algorithmic bytes exactly as SURVEY.md §8(d) defines them:
      A = sum over resident (template, level) of N * 256 B (SH3 attributes)
      M = instances * 24 * 48 B (3x4 skin matrices)
      frame   = A + M + 2*S*48 + K*(12 + 24*6 + 4) + 16*W*H   (K = 16x16 tile pairs)
      project = A + M + S*48                                  (k_project: stream + record write)
      raster  = K*4 + S*48 + 16*W*H                           (k_raster16q: sorted value,
                                                               each record once, framebuffer)"""
    G, S, _ = counts
    K = tile_pairs
    inst = scene.instances
    resident = set(zip(inst["template_id"].tolist(), lods.tolist()))
    A = sum(cfg.level_counts[l] for _, l in resident) * 256
    M = len(inst) * 24 * 48
    W, H = cfg.width, cfg.height
    frame = A + M + 2 * S * 48 + K * (12 + 24 * 6 + 4) + 16 * W * H
    return {"frame": frame, "project": A + M + S * 48, "raster": K * 4 + S * 48 + 16 * W * H, "A": A, "M": M,
            "K_tile": K}


def issue_roofline(kernel: str, kernel_ms: float, sm_mhz) -> dict | None:
    """Issue-slot roofline of an issue-bound kernel: warp instructions (ncu
    smsp__inst_executed.sum, profiles/ncu_summary.json) over 148 SMs x 4 schedulers x the
    SM clock measured during the timed region x the kernel's live event time."""
    if not PROFILE_SUMMARY.exists() or not sm_mhz:
        return None
    try:
        k = json.loads(PROFILE_SUMMARY.read_text())["kernels"][kernel]
        inst = float(k["warp_instructions"])
    except Exception:
        return None
    peak = 148 * 4 * sm_mhz * 1e6  # warp instructions per second
    achieved = inst / (kernel_ms * 1e-3)
    return {"warp_instructions": inst, "achieved_per_s": round(achieved, 1), "peak_per_s": peak,
            "frac": round(achieved / peak, 4), "source": str(PROFILE_SUMMARY.relative_to(ROOT))}


def memory_block(r, scene) -> dict:
    """Measured device bytes (shared template store, frame buffers) beside the reference's
    MemoryLayoutModel (crowd.cpp:142-210): the config-5 shared-attribute ablation."""
    mu = r.memory_usage()
    model = scene.memory_report()
    return {"template_store_bytes": mu["template_bytes"], "frame_buffers_bytes": mu["frame_bytes"],
            "device_used_bytes": mu["device_total_bytes"] - mu["device_free_bytes"],
            "model_shared_bytes": model["shared_bytes"], "model_naive_bytes": model["naive_bytes"],
            "model_savings_fraction": round(model["savings_fraction"], 4)}


def run_ours(args, rank, world, local_rank) -> dict | None:
    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    band_path = world > 1 or args.band_path
    if band_path:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    # Config 5's shared / naive grid first, while the device is empty (the headline frame's
    # buffers grow to ~90 GB).
    ablation = (layout_ablation(args, local_rank)
                if world == 1 and args.config == 5 and not args.no_ablation and not band_path else None)
    P, cfg, extra, scene = build_scene(args.config)
    from paper_2501_17792_b200 import native as N

    r = P.Renderer(scene, device=local_rank)
    settings = P.RenderSettings()
    n = scene.counts()[2]
    js = r.joint_stride
    forced = extra["forced_lod"]
    frames = args.warmup + args.steps
    t0 = extra["time_s"]
    times_s = [t0 + f / 30.0 for f in range(frames)]

    # ---- device-resident inputs: the crowd's placement / motion ids / phase offsets and
    # the motion clips live in HBM; every step samples all poses on the device
    # (GSCG_POSES_SAMPLED, bit-identical to host sampling) and renders the frame ----
    r.device_poses = True
    r.render_frame(times_s[0], settings, forced_lod=forced)  # uploads templates + motion tables
    tids, place, _ = r.sample_crowd(times_s[0])
    inst = scene.instances
    d_tids = torch.from_numpy(tids.view(np.int32)).to(dev)
    d_place = torch.from_numpy(place).to(dev)
    d_mid = torch.from_numpy(np.ascontiguousarray(inst["motion_id"]).astype(np.int32)).to(dev)
    d_phase = torch.from_numpy(np.ascontiguousarray(inst["phase_offset_s"]).astype(np.float32)).to(dev)
    d_lods = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
    cam = scene.camera_basis()
    from paper_2501_17792_b200.multigpu import gscg_settings
    rs = gscg_settings(settings)
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

    def frame_desc(f: int) -> N.GscgFrameDesc:
        fd = N.GscgFrameDesc()
        fd.instance_count = n
        fd.joint_stride = js
        fd.template_ids = d_tids.data_ptr()
        fd.placement = d_place.data_ptr()
        fd.active_lod = d_lods.data_ptr()
        fd.forced_lod = -1 if forced is None else forced
        fd.memory = N.GSCG_MEM_DEVICE
        fd.pose_source = N.GSCG_POSES_SAMPLED
        fd.time_s = times_s[f]
        fd.motion_ids = d_mid.data_ptr()
        fd.phase_offsets = d_phase.data_ptr()
        return fd

    if not band_path:
        def frame(f: int, timed: bool = False):
            # Timed frames pass no stage-time block: reading the stage events would make
            # every call wait for its raster, so the next frame's host work could not
            # overlap it (a real render loop does not read them either). The stage
            # breakdown comes from the same frames re-rendered after the timed region.
            if timed:
                N.check_gscg(lib.gscg_render_frame(ctx, C.byref(frame_desc(f)), C.byref(cam), C.byref(rs),
                                                   C.byref(lp), None, None, None), ctx)
                return None
            st = N.GscgStageTimes()
            N.check_gscg(lib.gscg_render_frame(ctx, C.byref(frame_desc(f)), C.byref(cam), C.byref(rs), C.byref(lp),
                                               None, None, C.byref(st)), ctx)
            return {"update": st.update_ms, "gather": st.gather_ms, "sort": st.sort_ms, "rasterize": st.rasterize_ms,
                    "launches": st.kernel_launches, "counts": (st.gaussian_count, st.splat_count, st.pair_count),
                    "tile_pairs": st.tile_pair_count}
    else:
        # Band-split frame: rank r renders screen rows [rows[r], rows[r+1]) of
        # the frame (its own instance cull + projection + sort + raster), and the bands are
        # gathered into rank 0's framebuffer in HBM, one gscg_group_render_frame per frame.
        from paper_2501_17792_b200.multigpu import BandGroup
        group = BandGroup(r, rank, world, dist, axis=args.split_axis)
        group.set_tile(settings.tile_size)

        def frame(f: int, timed: bool = False):
            # Timed frames read no stage events (as on one GPU): the frames stay in flight,
            # each rank's next update and projection under its sort, raster and gather.
            if timed:
                group.render(frame_desc(f), cam, rs, lp, stage_times=False)
                return None
            st = group.render(frame_desc(f), cam, rs, lp)
            return {"update": st.update_ms, "gather": st.gather_ms, "sort": st.sort_ms, "rasterize": st.rasterize_ms,
                    "launches": st.kernel_launches, "counts": (st.gaussian_count, st.splat_count, st.pair_count),
                    "tile_pairs": st.tile_pair_count}

        # Balance the regions on the warm-up frames: pairs per tile line over all ranks,
        # then every rank's measured region time (its stage times); the timed frames keep
        # the last cuts.
        for f in range(2):
            frame(f)
            group.rebalance()
        if world > 1:
            res = frame(2)
            group.rebalance_by_time(res["update"] + res["gather"] + res["sort"] + res["rasterize"])

    first = None
    for f in range(args.warmup):
        res = frame(f)
        first = first or res  # frame 0 (t = time_s): the config's reported counts, as the reference arm's
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    stage = []
    with ClockSampler(local_rank) as clocks:
        evs[0].record(stream)
        for f in range(args.warmup, frames):
            res = frame(f, timed=True)
            if res is not None:
                stage.append(res)
            evs[f - args.warmup + 1].record(stream)
        torch.cuda.synchronize()
    ev0, ev1 = evs[0], evs[-1]
    frame_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    median_ms = float(np.median(frame_ms))
    if dist:
        t = torch.tensor([median_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        median_ms = float(t.item())
    if not stage:  # the stage breakdown: the timed frames again, each read back (untimed)
        stage = [frame(f) for f in range(args.warmup, frames)]
    launches = sum(s["launches"] for s in stage)
    counts = stage[-1]["counts"]
    tile_pairs = stage[-1]["tile_pairs"]
    culled = r.instances_culled()
    lods = d_lods[:n].cpu().numpy().astype(np.uint32)

    # ---- end-to-end through the public API (host poses + pinned H2D + kernels + D2H) ----
    def time_e2e(e2e_frame, finish=lambda: None):
        for f in range(min(args.warmup, 2)):
            e2e_frame(f)
        finish()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t_start = time.perf_counter()
        for f in range(args.warmup, frames):
            e2e_frame(f)
        finish()  # the last frame's read-back is inside the timed region
        e2e_s = time.perf_counter() - t_start
        if dist:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        return args.steps / e2e_s

    e2e_sync_fps = None
    if not band_path:
        # The frame (the reference render_frame's Framebuffer: RGB) is read back into
        # page-locked memory every step. Streaming form (the headline): frame k's
        # read-back overlaps frame k+1 (render_frame(pipelined=True), two host buffers).
        outs = [(r.alloc_frame(pinned=True)[0], None) for _ in range(2)]

        def e2e_stream(f):
            r.render_frame(times_s[f], settings, forced_lod=forced, out=outs[f & 1], pipelined=True)

        e2e_fps = time_e2e(e2e_stream, lambda: r.wait_readback(0))

        def e2e_sync(f):  # one blocking call per frame
            r.render_frame(times_s[f], settings, forced_lod=forced, out=outs[0])

        e2e_sync_fps = time_e2e(e2e_sync)
    else:
        # Public API per step: the instance records from pinned host memory, the band
        # frame, the gather, and rank 0's read-back of the frame's colour into pinned memory.
        from paper_2501_17792_b200.api import pinned_array
        rec = r.instance_records()
        pinned = {k: pinned_array(v.shape, v.dtype) for k, v in rec.items()}
        for k, v in rec.items():
            pinned[k][...] = v
        band_outs = [pinned_array((cfg.height, cfg.width, 3)) for _ in range(2)]

        def e2e_frame(f):
            fd = N.GscgFrameDesc()
            fd.instance_count = n
            fd.joint_stride = js
            fd.template_ids = pinned["template_ids"].ctypes.data
            fd.placement = pinned["placement"].ctypes.data
            fd.active_lod = pinned["lods"].ctypes.data
            fd.forced_lod = -1 if forced is None else forced
            fd.memory = N.GSCG_MEM_HOST
            fd.pose_source = N.GSCG_POSES_SAMPLED
            fd.time_s = times_s[f]
            fd.motion_ids = pinned["motion_ids"].ctypes.data
            fd.phase_offsets = pinned["phase_offsets"].ctypes.data
            # Rank 0's read-back of frame k lands under frame k + 1 (two pinned buffers).
            group.render(fd, cam, rs, lp, band_outs[f & 1] if rank == 0 else None, stage_times=False, pipelined=True)

        e2e_fps = time_e2e(e2e_frame, group.wait_readback)
        group.close()
    h2d = n * (4 + 16 + 4 + 4 + 4)  # template id, placement, previous LoD, motion id, phase offset
    d2h = cfg.width * cfg.height * 12 + n * 4

    cfg_counts, cfg_tile_pairs = first["counts"], first["tile_pairs"]
    if dist:
        tot = torch.tensor([float(counts[1]), float(tile_pairs), float(cfg_counts[1]), float(cfg_tile_pairs)],
                           dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        counts = (counts[0], int(tot[0].item()), counts[2])
        tile_pairs = int(tot[1].item())
        cfg_counts = (cfg_counts[0], int(tot[2].item()), cfg_counts[2])
        cfg_tile_pairs = int(tot[3].item())
    if rank != 0:
        dist.destroy_process_group()
        return None

    peaks = _peaks()
    keys = [k for k in stage[0] if k not in ("launches", "counts", "tile_pairs")]
    stage_ms = {k: float(np.median([s[k] for s in stage])) for k in keys}
    rb = roofline_bytes(cfg, counts, tile_pairs, lods, scene)
    # The single longest kernel of the frame: k_project (gather) or k_raster16q (rasterize);
    # the sort stage is ~35 short launches, none longer than either.
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
    clk = clocks.summary()
    frame_roofline_ms = rb["frame"] / (peaks["hbm_gbs"] * 1e9) * 1e3
    out = {
        "metric": METRIC, "value": round(fps, 3), "unit": "FPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.config, cfg, cfg_counts, cfg_tile_pairs,
                               f"{world} screen regions ({args.split_axis}, one per GPU), NCCL gather to rank 0" if band_path else "single GPU"),
        "median_frame_ms": round(median_ms, 4), "fps_median": round(1000.0 / median_ms, 3),
        "colour": "SH degree 3 (BASELINE; the reference renders fixed RGB)",
        "instances_culled": culled,
        "l2": "no flush: the per-frame working set (templates ~0.5 GB + records/pairs ~0.8 GB) exceeds the 126 MB L2",
        "splats_per_s": round(counts[1] * fps, 1),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "frame_roofline": {"bytes": rb["frame"], "ms": round(frame_roofline_ms, 4),
                           "frac": round(frame_roofline_ms / ms_step, 4), "peak_gbs": peaks["hbm_gbs"],
                           "model": "SURVEY.md 8(d): A + M + 2*S*48 + K_tile*(12+24*6+4) + 16*W*H"},
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
                     "algorithmic_bytes": kbytes, "peak_source": peaks["source"],
                     "bytes_model": ("K_tile*4 + S*48 + 16*W*H" if kernel == "k_raster16q" else "A(256 B/G) + M + S*48"),
                     "issue": issue_roofline(kernel, stage_ms[dom], clk["sm_mhz"]),
                     "limiter": ("issue-bound on exact no-FMA FP32 + integer work; profiles/ncu_summary.json"
                                 if kernel == "k_project" else
                                 "issue-bound, per-pixel list walks (ncu DRAM < 10%); profiles/ncu_summary.json")},
        "e2e": {"value": round(e2e_fps, 3), "unit": "FPS", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": ("Renderer.render_frame(out=pinned, pipelined=True): frame k's read-back overlaps frame k+1"
                        if not band_path else ("gscg_group_render_frame_async: host instance records in, frame colour out on rank 0 into "
                              "page-locked memory, frame k's read-back under frame k+1")),
                "blocking_api_fps": None if e2e_sync_fps is None else round(e2e_sync_fps, 3)},
        "gpu_launches": int(launches),
        "clocks": clk,
        "memory": memory_block(r, scene),
    }
    if ablation is not None:
        out["layout_ablation"] = ablation
    if world == 1 and args.band_estimate and not band_path:
        out["band_split_estimate"] = band_split_estimate(r, ctx, lib, frame, stream, cfg, args)
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"], out["cpu_baseline_1t"] = cpu_baselines(args.config, args.cpu_frames)
    if dist:
        dist.destroy_process_group()
    return out


def layout_ablation(args, local_rank: int) -> dict:
    """The shared-attribute ablation of BASELINE config 5 / PAPER.md Tables 1-2 on the B200:
    one template at a forced level of 202,738 / 12,661 / 3,176 Gaussians, duplicated over
    1 / 100 / 400 / 1,000 / 5,000 characters (row-major cells of a 100 x 100 grid, camera
    over the grid centre), 1280 x 720, RGB colour, with and without motion. Each cell is
    rendered with the shared (template, level) store and with naive per-instance attribute
    copies (gscg_set_layout); device memory is measured (cudaMemGetInfo after the frame,
    and the attribute bytes each layout holds) and FPS is the median of CUDA-event frame
    times with device-resident inputs. A cell whose allocation fails is reported as out of
    memory, as the reference's run_benchmark does (bench.cpp:94-97)."""
    import torch
    import paper_2501_17792_b200 as P
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import gscg_settings

    dev = torch.device("cuda", local_rank)
    cfg = P.SceneConfig(template_count=1, template_seed_base=100, level_counts=P.api.LEVELS_PAPER, with_sh=False,
                        motion_count=15, motion_seed_base=500, motion_frames=60, grid_rows=100, grid_cols=100,
                        crowd_count=5000, crowd_seed=1, cam_pos=(49.5, 1.6, -3.0), cam_look=(49.5, 1.0, 5.0),
                        width=1280, height=720)
    scene = P.Scene(cfg)
    all_inst = scene.instances
    lib = N.gscg()
    rs = gscg_settings(P.RenderSettings(sh_colour=False))
    lp = N.GscgLodPolicy()
    lp.threshold_count = 2
    lp.thresholds_m[0], lp.thresholds_m[1] = 5.0, 10.0
    counts = (1, 100, 400, 1000, 5000)
    table = []
    for level, gauss in enumerate(P.api.LEVELS_PAPER):
        for layout in ("shared", "naive"):
            for motion in (False, True):
                row = {"gaussians": gauss, "layout": layout, "motion": motion, "cells": {}}
                for nchar in counts:
                    sub = all_inst[:nchar]
                    scene.instances = sub
                    r = frame = None
                    try:
                        r = P.Renderer(scene, device=local_rank, device_poses=True)
                        r.set_layout(layout == "naive")
                        r.render_frame(0.0, P.RenderSettings(sh_colour=False), static_pose=not motion,
                                       forced_lod=level)
                        tids = torch.from_numpy(np.ascontiguousarray(sub["template_id"]).astype(np.int32)).to(dev)
                        _, place, _ = r.sample_crowd(0.0)
                        d_place = torch.from_numpy(place).to(dev)
                        d_mid = torch.from_numpy(np.ascontiguousarray(sub["motion_id"]).astype(np.int32)).to(dev)
                        d_ph = torch.from_numpy(np.ascontiguousarray(sub["phase_offset_s"]).astype(np.float32)).to(dev)
                        d_lod = torch.full((nchar,), -1, dtype=torch.int32, device=dev)
                        cam = scene.camera_basis()
                        sp = C.c_void_p()
                        N.check_gscg(lib.gscg_stream(r.gpu, C.byref(sp)), r.gpu)
                        stream = torch.cuda.ExternalStream(sp.value, device=dev)

                        def frame(f):
                            fd = N.GscgFrameDesc()
                            fd.instance_count = nchar
                            fd.joint_stride = r.joint_stride
                            fd.template_ids = tids.data_ptr()
                            fd.placement = d_place.data_ptr()
                            fd.active_lod = d_lod.data_ptr()
                            fd.forced_lod = level
                            fd.memory = N.GSCG_MEM_DEVICE
                            fd.pose_source = N.GSCG_POSES_SAMPLED
                            fd.time_s = f / 30.0
                            fd.static_pose = 0 if motion else 1
                            fd.motion_ids = d_mid.data_ptr()
                            fd.phase_offsets = d_ph.data_ptr()
                            N.check_gscg(lib.gscg_render_frame(r.gpu, C.byref(fd), C.byref(cam), C.byref(rs),
                                                               C.byref(lp), None, None, None), r.gpu)

                        steps = 5 if gauss * nchar > 2e8 else 15
                        for f in range(2):
                            frame(f)
                        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
                        evs[0].record(stream)
                        for f in range(steps):
                            frame(2 + f)
                            evs[f + 1].record(stream)
                        torch.cuda.synchronize()
                        ms = float(np.median([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]))
                        mu = r.memory_usage()
                        row["cells"][str(nchar)] = {
                            "fps": round(1000.0 / ms, 2),
                            "device_used_mib": round((mu["device_total_bytes"] - mu["device_free_bytes"]) / 2**20, 1),
                            "attribute_mib": round((mu["template_bytes"] + mu["naive_attribute_bytes"]) / 2**20, 1),
                            "frame_buffers_mib": round(mu["frame_bytes"] / 2**20, 1)}
                    except (N.NativeError, MemoryError) as e:
                        row["cells"][str(nchar)] = {"skipped": "out of memory" if getattr(e, "status", -4) == -4
                                                    else str(e)[:80]}
                    frame = None
                    del r
                    import gc
                    gc.collect()
                    torch.cuda.synchronize()
                table.append(row)
    scene.instances = all_inst
    return {"resolution": [1280, 720], "colour": "RGB", "template": "synthetic seed 100 (one template, duplicated)",
            "note": "attribute_mib: the attribute store the layout reads (shared: one (template, level) store; naive: "
                    "+ per-instance copies of 80 B / Gaussian); device_used_mib: cudaMemGetInfo after the cell",
            "rows": table}


def band_split_estimate(r, ctx, lib, frame, stream, cfg, args) -> dict:
    """One rank's work of the P-GPU region-split frame, measured on this GPU: each of P
    regions (columns, the BandGroup default, and rows for comparison; cuts balanced by the
    frame's pairs per tile line as BandGroup.rebalance does) is rendered alone with
    gscg_set_region, K frames timed with CUDA events. The ranks of the multi-GPU frame are
    independent until the gather of finished pixels (W x H x 16 B in total), so the slowest
    region bounds the P-GPU frame time from below. Not a multi-GPU measurement."""
    import torch
    from paper_2501_17792_b200 import native as N
    from paper_2501_17792_b200.multigpu import band_rows, cuts_from_region_times

    ranges = r.cell_ranges()
    tiles, cpt = r.cell_layout()
    tx = (cfg.width + 15) // 16
    tile_pairs = (ranges[:, 1] - ranges[:, 0]).astype(np.float64).reshape(-1, cpt).sum(1).reshape(-1, tx)
    out = {"method": "each region rendered alone on one B200 (gscg_set_region), median interval of K pipelined frames"}
    for axis in ("cols", "rows"):
        line = tile_pairs.sum(0) if axis == "cols" else tile_pairs.sum(1)
        extent = cfg.width if axis == "cols" else cfg.height
        res = {}
        weights = line + 0.02 * line.mean() + 1.0

        def measure(cuts):
            region_ms = []
            for b in range(len(cuts) - 1):
                if cuts[b + 1] <= cuts[b]:
                    region_ms.append(0.0)
                    continue
                x0, y0, x1, y1 = (cuts[b], 0, cuts[b + 1], 0) if axis == "cols" else (0, cuts[b], 0, cuts[b + 1])
                N.check_gscg(lib.gscg_set_region(ctx, x0, y0, x1, y1), ctx)
                for f in range(3):
                    frame(f, timed=True)
                torch.cuda.synchronize()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
                evs[0].record(stream)
                for f in range(args.steps):  # pipelined frames, as each rank renders them
                    frame(args.warmup + f, timed=True)
                    evs[f + 1].record(stream)
                torch.cuda.synchronize()
                region_ms.append(float(np.median([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])))
            N.check_gscg(lib.gscg_set_region(ctx, 0, 0, 0, 0), ctx)
            return region_ms

        for parts in (1, 2, 4, 8):
            cuts = band_rows(extent, 16, parts, weights)
            region_ms = measure(cuts)
            res[str(parts)] = {"cuts": cuts, "region_ms": [round(x, 4) for x in region_ms],
                               "max_ms": round(max(region_ms), 4)}
            if parts > 1:  # BandGroup.rebalance_by_time: cuts re-weighted by the measured region times
                tcuts = cuts_from_region_times(weights, extent, 16, cuts, region_ms)
                tms = measure(tcuts)
                res[str(parts)]["time_balanced"] = {"cuts": tcuts, "region_ms": [round(x, 4) for x in tms],
                                                    "max_ms": round(max(tms), 4)}
        for parts in (2, 4, 8):
            res[str(parts)]["speedup_vs_1"] = round(res["1"]["max_ms"] / res[str(parts)]["max_ms"], 3)
            tb = res[str(parts)]["time_balanced"]
            tb["speedup_vs_1"] = round(res["1"]["max_ms"] / tb["max_ms"], 3)
        out[axis] = res
    return out


def bench_config(config: int, cfg, counts, tile_pairs: int, parallelism: str) -> dict:
    """Identical keys and values in both arms (the driver compares them)."""
    return {"workload": f"BASELINE config {config}: 14 synthetic templates (202738/12661/3176 G) x "
                        f"{cfg.crowd_count} animated characters, distance LoD 5/10 m, {cfg.width}x{cfg.height}, tile 16"
                        if config != 1 else
                        f"BASELINE config 1: 1 synthetic template (100000 G) x 1 character, {cfg.width}x{cfg.height}",
            "instances": cfg.crowd_count, "resolution": [cfg.width, cfg.height],
            "gaussians": int(counts[0]), "splats": int(counts[1]), "tile_pairs": int(tile_pairs),
            "parallelism": parallelism}


def reference_scene(config: int):
    """The reference's own scene for a BASELINE config: its synthetic generator and
    build_crowd (oracle/_ref), or the oracle port fed by the product scene if the
    reference build is missing. Returns (scene, kind, extra)."""
    from oracle import ref

    if ref.LIB_PATH.exists():
        rc, extra = ref.baseline(config)
        return ref.RefScene(rc, extra["origin_instance"]), "reference", extra
    P, cfg, extra, scene = build_scene(config)
    from oracle import orc
    return orc.from_scene(scene), "port", extra


def _ref_render(rs, kind: str, time_s: float, forced, threads: int):
    from oracle import orc, ref

    st = ref.settings() if kind == "reference" else orc.settings(sh_colour=True)
    return rs.render(time_s, st, forced_lod=forced, threads=threads)


def cpu_baselines(config: int, frames_sample: int) -> tuple[dict, dict]:
    """The reference's render_frame timed on this host (rank 0, N=1): all host threads over
    `frames_sample` frames, then one frame at 1 thread."""
    rs, kind, extra = reference_scene(config)
    cores = os.cpu_count() or 1
    forced, t0 = extra["forced_lod"], extra["time_s"]
    _ref_render(rs, kind, t0, forced, cores)  # warm-up frame
    out = []
    for threads, frames in ((cores, frames_sample), (1, 1)):
        per = []
        for f in range(frames):
            s0 = time.perf_counter()
            _ref_render(rs, kind, t0 + (f + 1) / 30.0, forced, threads)
            per.append(time.perf_counter() - s0)
        ms = float(np.median(per)) * 1e3
        out.append({"value": round(1000.0 / ms, 4), "unit": "FPS", "cores": threads, "kind": kind,
                    "median_frame_ms": round(ms, 1),
                    "sample": f"{frames} full frame(s) of BASELINE config {config} after 1 warm-up frame; "
                              f"{'the reference render_frame (oracle/_ref: its own sources + Eigen-subset shim, RGB colour)' if kind == 'reference' else 'the oracle port (SH colour)'}"
                              f"; thread_count = {threads} (parallel.hpp static partition; its sort and binning are single-threaded)"})
    return out[0], out[1]


def run_reference(args, rank, world) -> dict | None:
    """The reference arm: the reference's own CPU render_frame, rank 0 only."""
    if rank != 0:
        return None
    rs, kind, extra = reference_scene(args.config)
    cores = os.cpu_count() or 1
    forced, t0 = extra["forced_lod"], extra["time_s"]
    _, _, times0 = _ref_render(rs, kind, t0, forced, cores)  # frame 0: the config's counts + warm-up
    for f in range(1, min(args.warmup, 2)):
        _ref_render(rs, kind, t0 + f / 30.0, forced, cores)
    per = []
    budget_t0 = time.perf_counter()
    for f in range(args.steps):
        s0 = time.perf_counter()
        _ref_render(rs, kind, t0 + (args.warmup + f) / 30.0, forced, cores)
        per.append(time.perf_counter() - s0)
        if time.perf_counter() - budget_t0 > args.reference_budget_s:
            break
    ms = float(np.mean(per)) * 1e3
    med = float(np.median(per)) * 1e3
    fps = 1000.0 / ms
    if kind == "reference":
        from oracle import ref
        cfg = ref.baseline(args.config)[0]
    else:
        cfg = build_scene(args.config)[1]
    tile_pairs = int(times0.pair_count)
    return {"metric": METRIC, "value": round(fps, 4), "unit": "FPS", "n_gpus": world, "steps": len(per),
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": bench_config(args.config, cfg, (times0.gaussian_count, times0.splat_count, 0), tile_pairs,
                                   "single GPU" if world == 1 else
                                   f"{world} screen regions ({args.split_axis}, one per GPU), NCCL gather to rank 0"),
            "median_frame_ms": round(med, 3), "fps_median": round(1000.0 / med, 4),
            "colour": ("RGB: the reference has no SH (SURVEY.md 0.4); same geometry, splats and tile pairs"
                       if kind == "reference" else "SH degree 3 (oracle port)"),
            "cpu_baseline": {"value": round(fps, 4), "unit": "FPS", "cores": cores, "kind": kind,
                             "sample": f"{len(per)} of {args.steps} requested full frames (time budget "
                                       f"{args.reference_budget_s:.0f} s) on {cores} host threads"
                                       + (" through the reference's own render_frame (oracle/_ref)"
                                          if kind == "reference" else " through the oracle port")},
            "e2e": {"value": round(fps, 4), "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_dry(args, rank, world) -> dict | None:
    """The multi-rank plumbing of run_ours on CPU (gloo): rendezvous, barrier, per-rank
    timing reduced by MAX, rank 0 alone prints. Used by tests/test_bench.py."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
        dist.barrier()
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3])
    ranks = torch.tensor([1.0])
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(ranks)
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return None
    return {"metric": METRIC, "value": None, "unit": "FPS", "n_gpus": world, "ranks_seen": int(ranks.item()),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(ms.item()), "dry_run": True}


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: one rank per GPU via torchrun (the
    driver's own launch form); rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-frames", type=int, default=2)  # ~5 s of host work at config 3, plus one 1-thread frame
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--band-path", action="store_true",
                    help="use the multi-GPU band path (shard -> NCCL exchange -> band) even on one GPU")
    ap.add_argument("--reference-budget-s", type=float, default=150.0)
    ap.add_argument("--no-ablation", action="store_true", help="config 5: skip the shared/naive layout grid")
    ap.add_argument("--split-axis", default="cols", choices=["cols", "rows"],
                    help="multi-GPU frame: screen columns (default) or rows per GPU")
    ap.add_argument("--band-estimate", action="store_true",
                    help="also time each band of a 2/4/8-way split alone on this GPU (one rank's work)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/plumbing check without a GPU: gloo ranks, max-over-ranks timing, one JSON line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    rank, world, local_rank = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    # NCCL's communicator INIT lines (rank count, transports) go to stderr; stdout stays the
    # one JSON line.
    if os.environ.get("NCCL_DEBUG") is None:
        os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.dry_run:
        out = run_dry(args, rank, world)
    else:
        out = run_reference(args, rank, world) if args.impl == "reference" else run_ours(args, rank, world, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
