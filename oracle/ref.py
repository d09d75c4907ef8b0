"""ctypes face of oracle/_ref/libgsc_ref.so: the REFERENCE's own render path (its
unmodified src/{math,avatar,synthetic,lod,crowd,renderer,metrics,bench}.cpp compiled
against oracle/eigen_shim; see oracle/Makefile and ref_driver.cpp) — TEST INFRASTRUCTURE
ONLY. tests/, tests/golden/make_golden.py and bench.py's reference arm may load it; the
product never does. It depends on nothing in paper_2501_17792_b200/.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

_DIR = Path(__file__).resolve().parent
LIB_PATH = _DIR / "_ref" / "libgsc_ref.so"
REFERENCE_SRC = Path("/root/reference/proj")


class RefSceneDesc(C.Structure):
    _fields_ = [("template_count", C.c_uint32), ("template_seed_base", C.c_uint32), ("level_count", C.c_uint32),
                ("level_counts", C.c_uint32 * 8), ("joint_count", C.c_uint32), ("motion_count", C.c_uint32),
                ("motion_seed_base", C.c_uint32), ("motion_frames", C.c_uint32), ("motion_fps", C.c_float),
                ("grid_rows", C.c_uint32), ("grid_cols", C.c_uint32), ("grid_spacing", C.c_float),
                ("crowd_count", C.c_uint32), ("crowd_seed", C.c_uint64), ("cam_pos", C.c_float * 3),
                ("cam_look", C.c_float * 3), ("fov_y_deg", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("near_m", C.c_float), ("threshold_count", C.c_uint32), ("thresholds", C.c_float * 8),
                ("hysteresis", C.c_float)]


class RefSettings(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("background", C.c_float * 3), ("alpha_max", C.c_float),
                ("alpha_cutoff", C.c_float), ("transmittance_floor", C.c_float), ("pad", C.c_int32)]


class RefTimes(C.Structure):
    _fields_ = [("update_ms", C.c_double), ("gather_ms", C.c_double), ("sort_ms", C.c_double),
                ("rasterize_ms", C.c_double), ("splat_count", C.c_uint64), ("pair_count", C.c_uint64),
                ("gaussian_count", C.c_uint64)]


INSTANCE_DTYPE = np.dtype([("instance_id", "<u4"), ("template_id", "<u4"), ("motion_id", "<u4"), ("x", "<f4"),
                           ("z", "<f4"), ("yaw", "<f4"), ("phase_offset_s", "<f4"), ("active_lod", "<u4")])
SPLAT_DTYPE = np.dtype([("mean_px", "<f4", (2,)), ("cov_xx", "<f4"), ("cov_xy", "<f4"), ("cov_yy", "<f4"),
                        ("depth", "<f4"), ("color", "<f4", (3,)), ("opacity", "<f4"), ("instance_id", "<u4"),
                        ("gaussian_index", "<u4"), ("rect", "<i4", (4,))])

_P = C.c_void_p
_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_scene_new": (_P, [C.POINTER(RefSceneDesc)]),
    "ref_scene_free": (None, [_P]),
    "ref_scene_counts": (C.c_int, [_P, _P, _P, _P]),
    "ref_get_instances": (C.c_int, [_P, _P]),
    "ref_set_instances": (C.c_int, [_P, C.c_uint32, _P]),
    "ref_level_size": (C.c_uint32, [_P, C.c_uint32, C.c_uint32]),
    "ref_get_level": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ref_get_skeleton": (C.c_int, [_P, C.c_uint32, _P, _P, _P]),
    "ref_get_motion": (C.c_int, [_P, C.c_uint32, _P, _P, _P, _P]),
    "ref_render": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, C.POINTER(RefSettings), C.c_int32, _P, _P,
                             C.POINTER(RefTimes)]),
    "ref_get_lods": (C.c_int, [_P, _P]),
    "ref_gaussian_count": (C.c_uint64, [_P]),
    "ref_get_posed": (C.c_int, [_P, _P]),
    "ref_splat_count": (C.c_uint64, [_P]),
    "ref_get_splats": (C.c_int, [_P, _P]),
    "ref_pair_count": (C.c_uint64, [_P]),
    "ref_get_bins": (C.c_int, [_P, _P, _P]),
    "ref_psnr": (C.c_float, [_P, _P, C.c_int32, C.c_int32]),
}

_lib = None


def available() -> bool:
    return LIB_PATH.exists() or (REFERENCE_SRC / "src" / "renderer.cpp").exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import subprocess
            subprocess.run(["make", "-C", str(_DIR), "ref"], check=True, capture_output=True)
        _lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


@dataclass
class RefConfig:
    """The reference's scene inputs (SceneConfig scene.hpp:33-43 + the synthetic asset
    seeds); field names follow paper_2501_17792_b200.SceneConfig so one can be read as
    the other, but nothing here imports the product."""
    template_count: int = 1
    template_seed_base: int = 100
    level_counts: Sequence[int] = (60, 24, 8)
    joint_count: int = 24
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

    @classmethod
    def like(cls, cfg) -> "RefConfig":
        return cls(**{f: getattr(cfg, f) for f in cls.__dataclass_fields__})

    def desc(self) -> RefSceneDesc:
        d = RefSceneDesc()
        d.template_count, d.template_seed_base = self.template_count, self.template_seed_base
        d.level_count = len(self.level_counts)
        for i, v in enumerate(self.level_counts):
            d.level_counts[i] = int(v)
        d.joint_count = self.joint_count
        d.motion_count, d.motion_seed_base = self.motion_count, self.motion_seed_base
        d.motion_frames, d.motion_fps = self.motion_frames, self.motion_fps
        d.grid_rows, d.grid_cols, d.grid_spacing = self.grid_rows, self.grid_cols, self.grid_spacing
        d.crowd_count, d.crowd_seed = self.crowd_count, self.crowd_seed
        for i in range(3):
            d.cam_pos[i] = self.cam_pos[i]
            d.cam_look[i] = self.cam_look[i]
        d.fov_y_deg, d.width, d.height, d.near_m = self.fov_y_deg, self.width, self.height, self.near_m
        d.threshold_count = len(self.lod_thresholds)
        for i, v in enumerate(self.lod_thresholds):
            d.thresholds[i] = v
        d.hysteresis = self.lod_hysteresis
        return d


def settings(tile_size=16, background=(0, 0, 0), alpha_max=0.99, alpha_cutoff=None,
             transmittance_floor=1e-4) -> RefSettings:
    s = RefSettings()
    s.tile_size = tile_size
    for i in range(3):
        s.background[i] = background[i]
    s.alpha_max = alpha_max
    s.alpha_cutoff = float(np.float32(1.0) / np.float32(255.0)) if alpha_cutoff is None else alpha_cutoff
    s.transmittance_floor = transmittance_floor
    return s


# BASELINE.json configs[0..4] as the reference's inputs; the same
# scenes the product's baseline_config builds.
LEVELS_PAPER = (202738, 12661, 3176)


def baseline(index: int) -> tuple[RefConfig, dict]:
    if index == 1:
        cfg = RefConfig(template_count=1, template_seed_base=42, level_counts=(100000,), motion_count=1,
                        motion_seed_base=500, motion_frames=60, crowd_count=1, cam_pos=(0.0, 0.95, -2.2),
                        cam_look=(0.0, 0.95, 0.0), width=512, height=512)
        return cfg, {"time_s": 0.5, "forced_lod": None, "origin_instance": True}
    rows, cols, count, w, h = {2: (10, 10, 100, 1920, 1080), 3: (59, 60, 3500, 1920, 1080),
                               4: (100, 100, 10000, 3840, 2160), 5: (59, 60, 3500, 1920, 1080)}[index]
    cx = (cols - 1) / 2.0
    cfg = RefConfig(template_count=14, template_seed_base=100, level_counts=LEVELS_PAPER, motion_count=15,
                    motion_seed_base=500, motion_frames=60, grid_rows=rows, grid_cols=cols, crowd_count=count,
                    crowd_seed=1, cam_pos=(cx, 1.6, -3.0), cam_look=(cx, 1.0, 5.0), width=w, height=h)
    return cfg, {"time_s": 0.0, "forced_lod": 0 if index == 5 else None, "origin_instance": False}


class RefScene:
    """Templates, motions and crowd built by the reference's own generator and
    build_crowd; frames rendered by its own render_frame."""

    def __init__(self, cfg: RefConfig, origin_instance: bool = False):
        self.cfg = cfg
        h = lib().ref_scene_new(C.byref(cfg.desc()))
        if not h:
            raise RuntimeError(lib().ref_last_error().decode())
        self._h = C.c_void_p(h)
        if origin_instance:  # config 1: one character at the origin, clip 0, no phase (metrics.cpp:43-49)
            inst = self.instances
            inst["x"] = inst["z"] = inst["yaw"] = inst["phase_offset_s"] = 0.0
            inst["template_id"] = inst["motion_id"] = 0
            self.instances = inst

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_scene_free(self._h)
            self._h = None

    def counts(self) -> tuple[int, int, int]:
        t, m, n = C.c_uint32(), C.c_uint32(), C.c_uint32()
        lib().ref_scene_counts(self._h, C.byref(t), C.byref(m), C.byref(n))
        return t.value, m.value, n.value

    @property
    def instances(self) -> np.ndarray:
        out = np.zeros(self.counts()[2], INSTANCE_DTYPE)
        if len(out):
            lib().ref_get_instances(self._h, _p(out))
        return out

    @instances.setter
    def instances(self, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, dtype=INSTANCE_DTYPE)
        _check(lib().ref_set_instances(self._h, len(a), _p(a) if len(a) else None))

    def level(self, t: int, l: int) -> dict:
        n = lib().ref_level_size(self._h, t, l)
        out = {"count": n, "means": np.zeros((n, 3), np.float32), "rotations": np.zeros((n, 4), np.float32),
               "scales": np.zeros((n, 3), np.float32), "opacities": np.zeros(n, np.float32),
               "colors": np.zeros((n, 3), np.float32), "skin_indices": np.zeros((n, 4), np.uint16),
               "skin_weights": np.zeros((n, 4), np.float32), "cov6": np.zeros((n, 6), np.float32)}
        _check(lib().ref_get_level(self._h, t, l, *(_p(out[k]) for k in (
            "means", "rotations", "scales", "opacities", "colors", "skin_indices", "skin_weights", "cov6"))))
        return out

    def skeleton(self, t: int) -> dict:
        j = C.c_uint32()
        lib().ref_get_skeleton(self._h, t, C.byref(j), None, None)
        parents = np.zeros(j.value, np.int16)
        ib = np.zeros((j.value, 16), np.float32)
        lib().ref_get_skeleton(self._h, t, C.byref(j), _p(parents), _p(ib))
        return {"joint_count": j.value, "parents": parents, "inverse_bind": ib}

    def motion(self, m: int) -> dict:
        fps, frames, joints = C.c_float(), C.c_uint32(), C.c_uint32()
        lib().ref_get_motion(self._h, m, C.byref(fps), C.byref(frames), C.byref(joints), None)
        data = np.zeros((frames.value, 4 + 4 * joints.value), np.float32)
        lib().ref_get_motion(self._h, m, None, None, None, _p(data))
        return {"fps": fps.value, "frames": frames.value, "joints": joints.value, "data": data}

    def render(self, time_s: float, st: Optional[RefSettings] = None, static_pose=False, forced_lod=None,
               threads=0):
        st = st or settings()
        rgb = np.empty((self.cfg.height, self.cfg.width, 3), np.float32)
        T = np.empty((self.cfg.height, self.cfg.width), np.float32)
        times = RefTimes()
        _check(lib().ref_render(self._h, time_s, int(static_pose), -1 if forced_lod is None else forced_lod,
                                C.byref(st), threads, _p(rgb), _p(T), C.byref(times)))
        return rgb, T, times

    def lods(self, n: Optional[int] = None) -> np.ndarray:
        out = np.zeros(self.counts()[2], np.uint32)
        assert n is None or n == len(out)
        if len(out):
            lib().ref_get_lods(self._h, _p(out))
        return out

    def posed(self) -> np.ndarray:
        out = np.zeros((lib().ref_gaussian_count(self._h), 3), np.float32)
        if len(out):
            lib().ref_get_posed(self._h, _p(out))
        return out

    def splats(self) -> np.ndarray:
        out = np.zeros(lib().ref_splat_count(self._h), SPLAT_DTYPE)
        if len(out):
            lib().ref_get_splats(self._h, _p(out))
        return out

    def bins(self, tiles: int):
        k = lib().ref_pair_count(self._h)
        counts = np.zeros(tiles, np.uint32)
        items = np.zeros(max(k, 1), np.uint32)
        lib().ref_get_bins(self._h, _p(counts), _p(items))
        return counts, items[:k]


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return float(lib().ref_psnr(_p(a), _p(b), a.shape[1], a.shape[0]))
