"""Python mirror of the reference's host API for the crowd render path.

Names follow /root/reference/proj/include/gsc: ``SceneConfig`` (scene.hpp:33-43),
``RenderSettings`` (renderer.hpp:15-22), ``StageTimes`` (renderer.hpp:105-112) and
``render_frame`` (renderer.hpp:114-123). Everything below calls the in-tree native
libraries; the render itself runs only on the B200 through include/gscg.h.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import native as N

K_ALPHA_MAX = 0.99
K_ALPHA_CUTOFF = np.float32(1.0) / np.float32(255.0)


@dataclass
class SceneConfig:
    template_count: int = 1
    template_seed_base: int = 100
    level_counts: Sequence[int] = (60, 24, 8)
    joint_count: int = 24
    with_sh: bool = False
    motion_count: int = 1
    motion_seed_base: int = 500
    motion_fps: float = 30.0
    motion_frames: int = 24
    grid_rows: int = 1
    grid_cols: int = 1
    grid_spacing: float = 1.0
    crowd_count: int = 1
    crowd_seed: int = 1
    cam_pos: Sequence[float] = (0.0, 1.6, -3.0)
    cam_look: Sequence[float] = (0.0, 1.0, 5.0)
    fov_y_deg: float = 50.0
    width: int = 160
    height: int = 90
    near_m: float = 0.1
    lod_thresholds: Sequence[float] = (5.0, 10.0)
    lod_hysteresis: float = 0.0

    def native(self) -> N.GschSceneConfig:
        c = N.GschSceneConfig()
        c.template_count = self.template_count
        c.template_seed_base = self.template_seed_base
        c.level_count = len(self.level_counts)
        for i, v in enumerate(self.level_counts):
            c.level_counts[i] = int(v)
        c.joint_count = self.joint_count
        c.with_sh = int(bool(self.with_sh))
        c.motion_count = self.motion_count
        c.motion_seed_base = self.motion_seed_base
        c.motion_fps = self.motion_fps
        c.motion_frames = self.motion_frames
        c.grid_rows, c.grid_cols = self.grid_rows, self.grid_cols
        c.grid_spacing = self.grid_spacing
        c.crowd_count = self.crowd_count
        c.crowd_seed = self.crowd_seed
        for i in range(3):
            c.cam_pos[i] = self.cam_pos[i]
            c.cam_look[i] = self.cam_look[i]
        c.fov_y_deg = self.fov_y_deg
        c.width, c.height = self.width, self.height
        c.near_m = self.near_m
        c.lod_threshold_count = len(self.lod_thresholds)
        for i, v in enumerate(self.lod_thresholds):
            c.lod_thresholds[i] = v
        c.lod_hysteresis = self.lod_hysteresis
        return c


@dataclass
class RenderSettings:
    tile_size: int = 16
    background: Sequence[float] = (0.0, 0.0, 0.0)
    alpha_max: float = K_ALPHA_MAX
    alpha_cutoff: float = float(K_ALPHA_CUTOFF)
    transmittance_floor: float = 1e-4
    thread_count: int = 0
    sh_colour: bool = True

    def native(self) -> N.GschRenderSettings:
        s = N.GschRenderSettings()
        s.tile_size = self.tile_size
        for i in range(3):
            s.background[i] = self.background[i]
        s.alpha_max = self.alpha_max
        s.alpha_cutoff = self.alpha_cutoff
        s.transmittance_floor = self.transmittance_floor
        s.thread_count = self.thread_count
        s.sh_colour = int(bool(self.sh_colour))
        return s


@dataclass
class StageTimes:
    update_ms: float = 0.0
    gather_ms: float = 0.0
    sort_ms: float = 0.0
    rasterize_ms: float = 0.0
    pose_ms: float = 0.0
    splat_count: int = 0
    pair_count: int = 0
    gaussian_count: int = 0
    tile_pair_count: int = 0  # the reference's per-tile bin entries (pair_count: the GPU's binning cells)

    @property
    def total_ms(self) -> float:
        return self.update_ms + self.gather_ms + self.sort_ms + self.rasterize_ms


INSTANCE_DTYPE = np.dtype([("instance_id", "<u4"), ("template_id", "<u4"), ("motion_id", "<u4"), ("x", "<f4"),
                           ("z", "<f4"), ("yaw", "<f4"), ("phase_offset_s", "<f4"), ("active_lod", "<u4")])


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Scene:
    """Synthetic templates + motions + crowd (build_crowd) + camera, held by the host lib."""

    def __init__(self, cfg: SceneConfig, threads: int = 0):
        self.cfg = cfg
        h = C.c_void_p()
        N.check_gsch(N.gsch().gsch_scene_create(C.byref(cfg.native()), threads, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                N.gsch().gsch_scene_destroy(self._h)
            except TypeError:  # interpreter shutdown: the module's globals are already gone
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def counts(self) -> tuple[int, int, int]:
        t, m, n = C.c_uint32(), C.c_uint32(), C.c_uint32()
        N.check_gsch(N.gsch().gsch_scene_counts(self._h, C.byref(t), C.byref(m), C.byref(n)))
        return t.value, m.value, n.value

    @property
    def instances(self) -> np.ndarray:
        n = self.counts()[2]
        out = np.zeros(n, dtype=INSTANCE_DTYPE)
        if n:
            N.check_gsch(N.gsch().gsch_scene_get_instances(self._h, _ptr(out), n))
        return out

    @instances.setter
    def instances(self, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr, dtype=INSTANCE_DTYPE)
        N.check_gsch(N.gsch().gsch_scene_set_instances(self._h, _ptr(arr) if len(arr) else None, len(arr)))

    def set_camera(self, pos, look, fov_y_deg=50.0, width=None, height=None, near_m=0.1) -> None:
        p = np.asarray(pos, dtype=np.float32)
        l = np.asarray(look, dtype=np.float32)
        w = width if width is not None else self.cfg.width
        hgt = height if height is not None else self.cfg.height
        N.check_gsch(N.gsch().gsch_scene_set_camera(self._h, _ptr(p), _ptr(l), fov_y_deg, w, hgt, near_m))
        self.cfg.cam_pos, self.cfg.cam_look, self.cfg.fov_y_deg = tuple(pos), tuple(look), fov_y_deg
        self.cfg.width, self.cfg.height, self.cfg.near_m = w, hgt, near_m

    def camera_basis(self) -> N.GscgCamera:
        cam = N.GscgCamera()
        N.check_gsch(N.gsch().gsch_scene_camera_basis(self._h, C.byref(cam)))
        return cam

    def set_lod_policy(self, thresholds: Sequence[float], hysteresis: float = 0.0) -> None:
        th = np.asarray(thresholds, dtype=np.float32)
        N.check_gsch(N.gsch().gsch_scene_set_lod_policy(self._h, _ptr(th) if len(th) else None, len(th), hysteresis))
        self.cfg.lod_thresholds, self.cfg.lod_hysteresis = tuple(thresholds), hysteresis

    def level_count(self, t: int) -> int:
        out = C.c_uint32()
        N.check_gsch(N.gsch().gsch_scene_level_count(self._h, t, C.byref(out)))
        return out.value

    def level_view(self, t: int, l: int) -> dict[str, np.ndarray]:
        v = N.GschLevelView()
        N.check_gsch(N.gsch().gsch_scene_level_view(self._h, t, l, C.byref(v)))
        n = v.count

        def arr(ptr, ctype, shape):
            if not ptr:
                return None
            size = int(np.prod(shape))
            buf = (ctype * size).from_address(ptr)
            return np.ctypeslib.as_array(buf).reshape(shape).copy()

        return {
            "count": n,
            "means": arr(v.means, C.c_float, (n, 3)),
            "rotations": arr(v.rotations, C.c_float, (n, 4)),
            "scales": arr(v.scales, C.c_float, (n, 3)),
            "opacities": arr(v.opacities, C.c_float, (n,)),
            "colors": arr(v.colors, C.c_float, (n, 3)),
            "skin_indices": arr(v.skin_indices, C.c_uint16, (n, 4)),
            "skin_weights": arr(v.skin_weights, C.c_float, (n, 4)),
            "sh": arr(v.sh, C.c_float, (n, 45)),
            "cov6": arr(v.cov6, C.c_float, (n, 6)),
        }

    def skeleton(self, t: int) -> dict[str, np.ndarray]:
        j = C.c_uint32()
        par, ib = C.c_void_p(), C.c_void_p()
        N.check_gsch(N.gsch().gsch_scene_skeleton(self._h, t, C.byref(j), C.byref(par), C.byref(ib)))
        J = j.value
        parents = np.ctypeslib.as_array((C.c_int16 * J).from_address(par.value)).copy()
        inv = np.ctypeslib.as_array((C.c_float * (16 * J)).from_address(ib.value)).reshape(J, 16).copy()
        return {"joint_count": J, "parents": parents, "inverse_bind": inv}

    def sample_crowd(self, time_s: float, static_pose: bool = False, threads: int = 0, joint_stride: int = 24):
        """Host pose records (no GPU needed): template ids, placement, poses."""
        n = self.counts()[2]
        tids = np.zeros(max(n, 1), dtype=np.uint32)
        place = np.zeros((max(n, 1), 4), dtype=np.float32)
        poses = np.zeros((max(n, 1), 4 + 4 * joint_stride), dtype=np.float32)
        N.check_gsch(N.gsch().gsch_scene_sample_crowd(self._h, time_s, int(static_pose), threads, joint_stride,
                                                      _ptr(tids), _ptr(place), _ptr(poses)))
        return tids[:n], place[:n], poses[:n]

    def set_motion(self, m: int, fps: float, data: np.ndarray, joints: int) -> None:
        data = np.ascontiguousarray(data, dtype=np.float32)
        N.check_gsch(N.gsch().gsch_scene_set_motion(self._h, m, fps, data.shape[0], joints, _ptr(data)))

    def update_crowd(self, forced_lod: Optional[int] = None) -> None:
        """update_crowd's LoD step on the host (crowd.cpp:86-110): instances' active_lod."""
        N.check_gsch(N.gsch().gsch_scene_update_crowd(self._h, -1 if forced_lod is None else forced_lod))

    # ---- asset files (GSAT templates, GSMO motions; reference io.hpp:38-43) ----
    def save_template(self, t: int, path) -> None:
        N.check_gsch(N.gsch().gsch_scene_save_template(self._h, t, str(path).encode()))

    def load_template(self, path, t: Optional[int] = None) -> int:
        """Loads a GSAT file into template slot t (default: append); returns the slot."""
        t = self.counts()[0] if t is None else t
        N.check_gsch(N.gsch().gsch_scene_load_template(self._h, t, str(path).encode()))
        return t

    def save_motion(self, m: int, path) -> None:
        N.check_gsch(N.gsch().gsch_scene_save_motion(self._h, m, str(path).encode()))

    def load_motion(self, path, m: Optional[int] = None) -> int:
        m = self.counts()[1] if m is None else m
        N.check_gsch(N.gsch().gsch_scene_load_motion(self._h, m, str(path).encode()))
        return m

    def lod_quality_sweep(self, template_id: int, distances, settings: Optional[RenderSettings] = None,
                          device: int = 0) -> list[dict]:
        """PSNR of every LoD level against level 0 for one bind-posed character at each
        distance (reference lod_quality_sweep, metrics.cpp:25-75), rendered and scored on GPU."""
        settings = settings or RenderSettings()
        d = np.ascontiguousarray(distances, dtype=np.float32)
        n = C.c_uint32()
        st = settings.native()
        N.check_gsch(N.gsch().gsch_lod_quality_sweep(self._h, template_id, _ptr(d), d.size, C.byref(st), device,
                                                     None, 0, C.byref(n)))
        rows = (N.GschQualityRow * max(n.value, 1))()
        N.check_gsch(N.gsch().gsch_lod_quality_sweep(self._h, template_id, _ptr(d), d.size, C.byref(st), device,
                                                     rows, n.value, C.byref(n)))
        return [{"distance_m": r.distance_m, "level": r.level, "gaussian_count": r.gaussian_count,
                 "psnr_db": r.psnr_db} for r in rows[:n.value]]

    def memory_report(self) -> dict:
        r = N.GschMemoryReport()
        N.check_gsch(N.gsch().gsch_scene_memory_report(self._h, C.byref(r)))
        return _report(r)

    def motion(self, m: int) -> dict:
        fps, frames, joints = C.c_float(), C.c_uint32(), C.c_uint32()
        N.check_gsch(N.gsch().gsch_scene_motion(self._h, m, C.byref(fps), C.byref(frames), C.byref(joints), None))
        data = np.zeros((frames.value, 4 + 4 * joints.value), dtype=np.float32)
        N.check_gsch(N.gsch().gsch_scene_motion(self._h, m, None, None, None, _ptr(data)))
        return {"fps": fps.value, "frames": frames.value, "joints": joints.value, "data": data}


def _report(r: N.GschMemoryReport) -> dict:
    return {f: getattr(r, f) for f, _ in r._fields_}


def memory_report_cell(instances: int, gaussians: int, fixed_overhead: int = 0) -> dict:
    """MemoryLayoutModel accounting for one table cell (crowd.cpp:205-210)."""
    r = N.GschMemoryReport()
    N.check_gsch(N.gsch().gsch_memory_report_cell(instances, gaussians, fixed_overhead, C.byref(r)))
    return _report(r)


# FrameSplat (reference renderer.hpp:39-44) = gscg_frame_splat, 64 bytes
FRAME_SPLAT_DTYPE = np.dtype([("mean_px", "<f4", (2,)), ("cov_xx", "<f4"), ("cov_xy", "<f4"), ("cov_yy", "<f4"),
                              ("depth", "<f4"), ("color", "<f4", (3,)), ("opacity", "<f4"), ("instance_id", "<u4"),
                              ("gaussian_index", "<u4"), ("rect", "<i4", (4,))])
assert FRAME_SPLAT_DTYPE.itemsize == 64


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """The reference's PSNR (metrics.cpp:8-23) on the host: two H x W x 3 float images."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("psnr: dimension mismatch")
    out = C.c_float()
    N.check_gsch(N.gsch().gsch_psnr(_ptr(a), _ptr(b), a.shape[1], a.shape[0], C.byref(out)))
    return out.value


def pinned_array(shape, dtype=np.float32) -> np.ndarray:
    """A numpy array in page-locked host memory (freed with the array)."""
    import weakref

    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    ptr = C.c_void_p()
    N.check_gscg(N.gscg().gscg_host_alloc(nbytes, C.byref(ptr)), None)
    raw = (C.c_uint8 * max(nbytes, 1)).from_address(ptr.value)
    weakref.finalize(raw, N.gscg().gscg_host_free, ptr.value)
    return np.frombuffer(raw, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


class Renderer:
    """FrameContext on a B200: owns the gscg context and the uploaded template store."""

    def __init__(self, scene: Scene, device: int = 0, device_poses: bool = False):
        self.scene = scene
        h = C.c_void_p()
        N.check_gsch(N.gsch().gsch_renderer_create(scene.handle, device, C.byref(h)))
        self._h = h
        self.gpu = C.c_void_p(N.gsch().gsch_renderer_gpu(h))
        self._device_poses = False
        self.device_poses = device_poses

    @property
    def device_poses(self) -> bool:
        """Sample poses on the GPU (bit-identical to host sampling; uploads no pose records)."""
        return self._device_poses

    @device_poses.setter
    def device_poses(self, on: bool) -> None:
        N.check_gsch(N.gsch().gsch_renderer_set_device_poses(self._h, int(bool(on))))
        self._device_poses = bool(on)

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                N.gsch().gsch_renderer_destroy(self._h)
            except TypeError:  # interpreter shutdown: the module's globals are already gone
                pass
            self._h = None

    @property
    def joint_stride(self) -> int:
        return int(N.gsch().gsch_renderer_joint_stride(self._h))

    # ---- stage functions (reference renderer.hpp:81-103) ----
    def gather_splats(self, time_s: float, settings: Optional[RenderSettings] = None, static_pose: bool = False,
                      forced_lod: Optional[int] = None) -> np.ndarray:
        """update + projection at time_s: the surviving splats (FRAME_SPLAT_DTYPE) in
        (instance, gaussian) order, as the reference's gather_splats concatenates them."""
        settings = settings or RenderSettings()
        st = settings.native()
        n = C.c_uint64()
        fl = -1 if forced_lod is None else forced_lod
        N.check_gsch(N.gsch().gsch_gather_splats(self._h, time_s, int(static_pose), fl, C.byref(st), None, 0,
                                                 C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=FRAME_SPLAT_DTYPE)
        N.check_gsch(N.gsch().gsch_gather_splats(self._h, time_s, int(static_pose), fl, C.byref(st), _ptr(out),
                                                 out.size, C.byref(n)))
        return out[:n.value]

    def sort_splats(self, splats: np.ndarray) -> np.ndarray:
        """Sorted copy by (depth bits, instance, gaussian) (reference sort_splats)."""
        a = np.ascontiguousarray(splats, dtype=FRAME_SPLAT_DTYPE).copy()
        N.check_gsch(N.gsch().gsch_sort_splats(self._h, _ptr(a) if a.size else None, a.size))
        return a

    def rasterize_full(self, splats: np.ndarray, width: int, height: int,
                       settings: Optional[RenderSettings] = None):
        """(rgb, T) of the splats binned and blended in the given order (reference
        rasterize_full)."""
        settings = settings or RenderSettings()
        a = np.ascontiguousarray(splats, dtype=FRAME_SPLAT_DTYPE)
        rgb = np.empty((height, width, 3), dtype=np.float32)
        T = np.empty((height, width), dtype=np.float32)
        N.check_gsch(N.gsch().gsch_rasterize_splats(self._h, _ptr(a) if a.size else None, a.size, width, height,
                                                    C.byref(settings.native()), _ptr(rgb), _ptr(T)))
        return rgb, T

    def alloc_frame(self, pinned: bool = True):
        """(rgb HxWx3, T HxW) float32 output arrays; pinned ones take the direct DMA path."""
        W, H = self.scene.cfg.width, self.scene.cfg.height
        if not pinned:
            return np.empty((H, W, 3), dtype=np.float32), np.empty((H, W), dtype=np.float32)
        return pinned_array((H, W, 3)), pinned_array((H, W))

    def render_frame(self, time_s: float, settings: Optional[RenderSettings] = None, static_pose: bool = False,
                     forced_lod: Optional[int] = None, times: Optional[StageTimes] = None, out=None,
                     pipelined: bool = False):
        """Renders one frame; returns (rgb, T). `out` = (rgb, T) arrays to fill (e.g. from
        alloc_frame(pinned=True)), else fresh arrays are returned. With out = (rgb, None)
        only the colour is read back (the reference render_frame returns just the
        Framebuffer; T is rasterize_full's extra output) and T is returned as None.

        pipelined=True (gsch_render_async): returns once the frame is rendered while its
        read-back into `out` continues, overlapped with the next frame; the arrays are
        valid after wait_readback(). Streaming callers alternate two `out` pairs. The
        read-back lands after this call returns, so `out` is required (ideally pinned
        arrays from alloc_frame) and the Renderer keeps it alive until it has landed."""
        settings = settings or RenderSettings()
        W, H = self.scene.cfg.width, self.scene.cfg.height
        region = getattr(self, "_region", None)
        if region is not None:
            x0, y0, x1, y1 = region
            if y1 > y0:
                H = min(y1, H) - y0
            if x1 > x0:
                W = min(x1, W) - x0
        if pipelined and out is None:
            raise ValueError("render_frame(pipelined=True) needs `out` arrays: the read-back completes after the call")
        if out is None:
            rgb = np.empty((H, W, 3), dtype=np.float32)
            T = np.empty((H, W), dtype=np.float32)
        else:
            rgb, T = out
            if rgb.shape != (H, W, 3) or rgb.dtype != np.float32 or not rgb.flags.c_contiguous or (
                    T is not None and (T.shape != (H, W) or T.dtype != np.float32 or not T.flags.c_contiguous)):
                raise ValueError("out must be C-contiguous float32 arrays of shape (H, W, 3) and (H, W)")
        st = N.GschStageTimes()
        fn = N.gsch().gsch_render_async if pipelined else N.gsch().gsch_render
        N.check_gsch(fn(self._h, time_s, int(static_pose), -1 if forced_lod is None else forced_lod,
                        C.byref(settings.native()), _ptr(rgb), None if T is None else _ptr(T), C.byref(st)))
        # A pipelined frame's destination is written until a later call or wait_readback:
        # hold the arrays of the last two pipelined submissions (older ones are complete).
        if pipelined:
            self._inflight = (getattr(self, "_inflight", []) + [(rgb, T)])[-2:]
        self.last_times = StageTimes(**{f: getattr(st, f) for f in StageTimes.__dataclass_fields__})
        if times is not None:
            for f in StageTimes.__dataclass_fields__:
                setattr(times, f, getattr(st, f))
        return rgb, T

    def set_layout(self, naive: bool) -> None:
        """Attribute layout of the projection (gscg_set_layout): the shared (template,
        level) store, or naive per-instance copies (the config-5 memory / FPS ablation;
        RGB colour)."""
        N.check_gscg(N.gscg().gscg_set_layout(self.gpu, N.GSCG_LAYOUT_NAIVE if naive else N.GSCG_LAYOUT_SHARED),
                     self.gpu)

    def set_band(self, row_begin: int = 0, row_end: int = 0) -> None:
        """Render only screen rows [row_begin, row_end) (tile-aligned; gscg_set_band):
        render_frame then returns the band's rows, bit-identical to the same rows of the
        whole frame. (0, 0) = the whole frame."""
        self.set_region(0, row_begin, 0, row_end)

    def set_region(self, x0: int, y0: int, x1: int, y1: int) -> None:
        """Render only the region [x0, x1) x [y0, y1) (tile-aligned; gscg_set_region; an
        empty range = the whole axis): render_frame returns those pixels, bit-identical to
        the same pixels of the whole frame."""
        N.check_gscg(N.gscg().gscg_set_region(self.gpu, x0, y0, x1, y1), self.gpu)
        self._region = (x0, y0, x1, y1) if (x1 > x0 or y1 > y0) else None

    def wait_readback(self, frames_back: int = 0) -> None:
        """Blocks until the read-back of the pipelined frame submitted `frames_back`
        frames ago (0 = the last) has landed in its `out` arrays."""
        N.check_gsch(N.gsch().gsch_wait_readback(self._h, frames_back))

    def memory_usage(self) -> dict:
        """Device bytes of the shared template store and the per-frame buffers (gscg_memory_usage)."""
        m = N.GscgMemoryUsage()
        N.check_gscg(N.gscg().gscg_memory_usage(self.gpu, C.byref(m)), self.gpu)
        return {f: getattr(m, f) for f, _ in m._fields_}

    def prepare(self) -> None:
        """Upload the scene's templates and motion clips now (else on the first render)."""
        N.check_gsch(N.gsch().gsch_renderer_prepare(self._h))

    def instance_records(self, static_pose: bool = False) -> dict:
        """Per-instance records of a device-sampled frame: template_ids, placement (n x 4),
        motion_ids, phase_offsets, lods."""
        n = self.scene.counts()[2]
        out = {"template_ids": np.zeros(n, np.uint32), "placement": np.zeros((n, 4), np.float32),
               "motion_ids": np.zeros(n, np.uint32), "phase_offsets": np.zeros(n, np.float32),
               "lods": np.zeros(n, np.uint32)}
        N.check_gsch(N.gsch().gsch_fill_instances(
            self._h, int(static_pose), _ptr(out["template_ids"]), _ptr(out["placement"]), _ptr(out["motion_ids"]),
            _ptr(out["phase_offsets"]), _ptr(out["lods"])))
        return out

    def sample_crowd(self, time_s: float, static_pose: bool = False, threads: int = 0):
        n = self.scene.counts()[2]
        js = self.joint_stride
        tids = np.zeros(n, dtype=np.uint32)
        place = np.zeros((n, 4), dtype=np.float32)
        poses = np.zeros((n, 4 + 4 * js), dtype=np.float32)
        N.check_gsch(N.gsch().gsch_sample_crowd(self._h, time_s, int(static_pose), threads, _ptr(tids), _ptr(place),
                                                _ptr(poses)))
        return tids, place, poses

    # ---- parity / debug exports (include/gscg.h) ----
    def set_debug(self, flags: int) -> None:
        N.check_gscg(N.gscg().gscg_set_debug(self.gpu, flags), self.gpu)

    def counts(self) -> tuple[int, int, int]:
        g, s, k = C.c_uint64(), C.c_uint64(), C.c_uint64()
        N.check_gscg(N.gscg().gscg_get_counts(self.gpu, C.byref(g), C.byref(s), C.byref(k)), self.gpu)
        return g.value, s.value, k.value

    def instances_culled(self) -> int:
        """Instances of the last frame left out by the instance frustum cull."""
        v = C.c_uint32()
        N.check_gscg(N.gscg().gscg_get_instances_culled(self.gpu, C.byref(v)), self.gpu)
        return v.value

    def lods(self) -> np.ndarray:
        n = self.scene.counts()[2]
        out = np.zeros(n, dtype=np.uint32)
        N.check_gscg(N.gscg().gscg_get_lod(self.gpu, _ptr(out), n), self.gpu)
        return out

    def instance_base(self) -> np.ndarray:
        n = self.scene.counts()[2]
        out = np.zeros(n, dtype=np.uint32)
        N.check_gscg(N.gscg().gscg_get_instance_base(self.gpu, _ptr(out), n), self.gpu)
        return out

    def posed_means(self) -> np.ndarray:
        g = self.counts()[0]
        out = np.zeros((g, 3), dtype=np.float32)
        N.check_gscg(N.gscg().gscg_get_posed_means(self.gpu, _ptr(out), g), self.gpu)
        return out

    def splat_records(self) -> np.ndarray:
        s = self.counts()[1]
        out = (N.GscgSplatRecord * max(s, 1))()
        N.check_gscg(N.gscg().gscg_get_splat_records(self.gpu, C.addressof(out), s), self.gpu)
        return np.ctypeslib.as_array(out)[:s].copy() if s else np.zeros(0, dtype=np.ctypeslib.as_array(out).dtype)

    def cell_layout(self) -> tuple[int, int]:
        """(tiles, cells per tile) of the last frame's binning (see gscg_get_cell_layout)."""
        t, c = C.c_uint32(), C.c_uint32()
        N.check_gscg(N.gscg().gscg_get_cell_layout(self.gpu, C.byref(t), C.byref(c)), self.gpu)
        return t.value, c.value

    def cell_ranges(self) -> np.ndarray:
        """[start, end) into the sorted pairs for every binning cell (tiles x cells_per_tile)."""
        tiles, cpt = self.cell_layout()
        out = np.zeros((tiles * cpt, 2), dtype=np.uint32)
        N.check_gscg(N.gscg().gscg_get_tile_ranges(self.gpu, _ptr(out), tiles * cpt), self.gpu)
        return out

    def tile_lists(self, depth_of_ordinal=None) -> tuple[np.ndarray, np.ndarray]:
        """The reference's per-tile lists (bins) as (counts per tile, concatenated splat
        ordinals): each tile's cell lists merged in (depth, ordinal) order, duplicates of a
        splat spanning several cells kept once. depth_of_ordinal maps ordinal -> depth bits
        (from splat_records); needed only when cells_per_tile > 1."""
        tiles, cpt = self.cell_layout()
        ranges = self.cell_ranges()
        ords = self.sorted_ordinals().astype(np.int64)
        counts = np.zeros(tiles, dtype=np.int64)
        items = []
        for t in range(tiles):
            segs = [ords[ranges[t * cpt + q, 0]:ranges[t * cpt + q, 1]] for q in range(cpt)]
            lst = np.concatenate(segs) if cpt > 1 else segs[0]
            if cpt > 1 and len(lst):
                lst = np.unique(lst)
                keys = depth_of_ordinal(lst)
                lst = lst[np.lexsort((lst, keys))]
            counts[t] = len(lst)
            items.append(lst)
        return counts, (np.concatenate(items) if items else np.zeros(0, np.int64))

    def sorted_ordinals(self) -> np.ndarray:
        k = self.counts()[2]
        out = np.zeros(max(k, 1), dtype=np.uint32)
        N.check_gscg(N.gscg().gscg_get_sorted_ordinals(self.gpu, _ptr(out), k), self.gpu)
        return out[:k]


def render_frame(renderer: Renderer, time_s: float, settings: Optional[RenderSettings] = None,
                 static_pose: bool = False, forced_lod: Optional[int] = None,
                 times: Optional[StageTimes] = None) -> np.ndarray:
    """render_frame(crowd, camera, time_s, settings, static_pose, forced_lod, times, ctx) -> Framebuffer."""
    rgb, _ = renderer.render_frame(time_s, settings, static_pose, forced_lod, times)
    return rgb


# ---------------------------------------------------------------- BASELINE configs
LEVELS_PAPER = (202738, 12661, 3176)


def baseline_config(index: int) -> tuple[SceneConfig, dict]:
    """Scene for BASELINE.json configs[index-1]; extra dict: time_s, forced_lod, instance override."""
    if index == 1:
        cfg = SceneConfig(template_count=1, template_seed_base=42, level_counts=(100000,), with_sh=True,
                          motion_count=1, motion_seed_base=500, motion_frames=60, grid_rows=1, grid_cols=1,
                          crowd_count=1, crowd_seed=1, cam_pos=(0.0, 0.95, -2.2), cam_look=(0.0, 0.95, 0.0),
                          width=512, height=512)
        return cfg, {"time_s": 0.5, "forced_lod": None, "origin_instance": True}
    grids = {2: (10, 10, 100, 1920, 1080), 3: (59, 60, 3500, 1920, 1080), 4: (100, 100, 10000, 3840, 2160),
             5: (59, 60, 3500, 1920, 1080)}
    rows, cols, count, w, h = grids[index]
    cx = (cols - 1) / 2.0
    cfg = SceneConfig(template_count=14, template_seed_base=100, level_counts=LEVELS_PAPER, with_sh=True,
                      motion_count=15, motion_seed_base=500, motion_frames=60, grid_rows=rows, grid_cols=cols,
                      crowd_count=count, crowd_seed=1, cam_pos=(cx, 1.6, -3.0), cam_look=(cx, 1.0, 5.0),
                      width=w, height=h)
    return cfg, {"time_s": 0.0, "forced_lod": 0 if index == 5 else None, "origin_instance": False}


def place_origin_instance(scene: Scene) -> None:
    inst = scene.instances
    inst["x"] = 0.0
    inst["z"] = 0.0
    inst["yaw"] = 0.0
    inst["phase_offset_s"] = 0.0
    inst["template_id"] = 0
    inst["motion_id"] = 0
    scene.instances = inst
