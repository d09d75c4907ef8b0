"""ctypes face of the CPU ORACLE (oracle/orc.cpp) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this
module; the product path never does. See orc.h for what the oracle restates and how it
is pinned ("parity unpinned" against a real Eigen build of the reference).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_LIB_PATH = _DIR / "_build" / "liborc.so"


class OrcInstance(C.Structure):
    _fields_ = [("instance_id", C.c_uint32), ("template_id", C.c_uint32), ("motion_id", C.c_uint32),
                ("x", C.c_float), ("z", C.c_float), ("yaw", C.c_float), ("phase_offset_s", C.c_float),
                ("active_lod", C.c_uint32)]


class OrcSplat(C.Structure):
    _fields_ = [("mean_px", C.c_float * 2), ("cov_xx", C.c_float), ("cov_xy", C.c_float), ("cov_yy", C.c_float),
                ("depth", C.c_float), ("color", C.c_float * 3), ("opacity", C.c_float),
                ("instance_id", C.c_uint32), ("gaussian_index", C.c_uint32), ("rect", C.c_int32 * 4)]


class OrcSettings(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("background", C.c_float * 3), ("alpha_max", C.c_float),
                ("alpha_cutoff", C.c_float), ("transmittance_floor", C.c_float), ("sh_colour", C.c_int32)]


class OrcTimes(C.Structure):
    _fields_ = [("update_ms", C.c_double), ("gather_ms", C.c_double), ("sort_ms", C.c_double),
                ("rasterize_ms", C.c_double), ("splat_count", C.c_uint64), ("pair_count", C.c_uint64),
                ("gaussian_count", C.c_uint64)]


SPLAT_DTYPE = np.dtype([("mean_px", "<f4", (2,)), ("cov_xx", "<f4"), ("cov_xy", "<f4"), ("cov_yy", "<f4"),
                        ("depth", "<f4"), ("color", "<f4", (3,)), ("opacity", "<f4"), ("instance_id", "<u4"),
                        ("gaussian_index", "<u4"), ("rect", "<i4", (4,))])
assert SPLAT_DTYPE.itemsize == C.sizeof(OrcSplat)

_P = C.c_void_p
_SIGS = {
    "orc_scene_new": (_P, []),
    "orc_scene_free": (None, [_P]),
    "orc_last_error": (C.c_char_p, []),
    "orc_add_template": (C.c_int, [_P, C.c_uint32, _P, _P]),
    "orc_add_level": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "orc_add_motion": (C.c_int, [_P, C.c_float, C.c_uint32, C.c_uint32, _P]),
    "orc_set_instances": (C.c_int, [_P, C.c_uint32, _P]),
    "orc_get_instances": (C.c_int, [_P, C.c_uint32, _P]),
    "orc_set_camera": (C.c_int, [_P, _P, _P, C.c_float, C.c_int32, C.c_int32, C.c_float]),
    "orc_set_lod": (C.c_int, [_P, _P, C.c_uint32, C.c_float]),
    "orc_render": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, C.POINTER(OrcSettings), C.c_int32, _P, _P,
                             C.POINTER(OrcTimes)]),
    "orc_get_lods": (C.c_int, [_P, _P]),
    "orc_gaussian_count": (C.c_uint64, [_P]),
    "orc_get_posed": (C.c_int, [_P, _P]),
    "orc_splat_count": (C.c_uint64, [_P]),
    "orc_get_splats": (C.c_int, [_P, _P]),
    "orc_pair_count": (C.c_uint64, [_P]),
    "orc_get_bins": (C.c_int, [_P, _P, _P]),
    "orc_get_level_cov": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P]),
    "orc_libm_sinf": (None, [_P, _P, C.c_uint64]),
    "orc_libm_expf_range": (None, [C.c_uint32, C.c_uint64, _P]),
    "orc_build_covariance": (C.c_int, [_P, _P, _P]),
    "orc_camera": (C.c_int, [_P, _P, C.c_float, C.c_int32, C.c_int32, C.c_float, _P, _P, _P]),
    "orc_project": (C.c_int, [_P, _P, _P, C.c_float, _P, _P, C.c_float, C.c_int32, C.c_int32, C.c_float, _P]),
    "orc_select_lod": (C.c_uint32, [_P, C.c_uint32, C.c_float, C.c_float, C.c_int64]),
    "orc_sort_splats": (C.c_int, [_P, C.c_uint32]),
    "orc_rasterize": (C.c_int, [_P, C.c_uint32, C.c_int32, C.c_int32, C.POINTER(OrcSettings), C.c_int32, _P, _P]),
    "orc_naive_rasterize": (C.c_int, [_P, C.c_uint32, C.c_int32, C.c_int32, C.POINTER(OrcSettings), _P, _P]),
    "orc_sample_pose": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_float, C.c_float, C.c_int32, _P]),
    "orc_forward_kinematics": (C.c_int, [_P, C.c_uint32, _P, _P, _P]),
    "orc_skin_means": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            import subprocess
            subprocess.run(["make", "-C", str(_DIR)], check=True, capture_output=True)
        _lib = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(lib().orc_last_error().decode())


def settings(tile_size=16, background=(0, 0, 0), alpha_max=0.99, alpha_cutoff=None, transmittance_floor=1e-4,
             sh_colour=True) -> OrcSettings:
    s = OrcSettings()
    s.tile_size = tile_size
    for i in range(3):
        s.background[i] = background[i]
    s.alpha_max = alpha_max
    s.alpha_cutoff = float(np.float32(1.0) / np.float32(255.0)) if alpha_cutoff is None else alpha_cutoff
    s.transmittance_floor = transmittance_floor
    s.sh_colour = int(bool(sh_colour))
    return s


class OracleScene:
    """CPU restatement of a crowd scene; fed the identical host arrays as the GPU path."""

    def __init__(self):
        self._h = C.c_void_p(lib().orc_scene_new())
        self.width = self.height = 0

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_scene_free(self._h)
            self._h = None

    def add_template(self, parents: np.ndarray, inverse_bind: np.ndarray) -> None:
        parents = np.ascontiguousarray(parents, dtype=np.int16)
        ib = np.ascontiguousarray(inverse_bind, dtype=np.float32)
        _check(lib().orc_add_template(self._h, len(parents), _p(parents), _p(ib)))

    def add_level(self, t: int, lv: dict) -> None:
        a = {k: (np.ascontiguousarray(v) if isinstance(v, np.ndarray) else v) for k, v in lv.items()}
        _check(lib().orc_add_level(self._h, t, a["count"], _p(a["means"]), _p(a["rotations"]), _p(a["scales"]),
                                   _p(a["opacities"]), _p(a["colors"]), _p(a["skin_indices"]), _p(a["skin_weights"]),
                                   _p(a.get("sh"))))

    def add_motion(self, fps: float, data: np.ndarray, joints: int) -> None:
        data = np.ascontiguousarray(data, dtype=np.float32)
        _check(lib().orc_add_motion(self._h, fps, data.shape[0], joints, _p(data)))

    def set_instances(self, inst: np.ndarray) -> None:
        arr = np.ascontiguousarray(inst)
        _check(lib().orc_set_instances(self._h, len(arr), _p(arr) if len(arr) else None))

    def instances(self, like: np.ndarray) -> np.ndarray:
        out = np.zeros_like(like)
        _check(lib().orc_get_instances(self._h, len(out), _p(out) if len(out) else None))
        return out

    def set_camera(self, eye, target, fov, w, h, near_m=0.1) -> None:
        e = np.asarray(eye, dtype=np.float32)
        t = np.asarray(target, dtype=np.float32)
        _check(lib().orc_set_camera(self._h, _p(e), _p(t), fov, w, h, near_m))
        self.width, self.height = w, h

    def set_lod(self, thresholds, hysteresis=0.0) -> None:
        th = np.asarray(thresholds, dtype=np.float32)
        _check(lib().orc_set_lod(self._h, _p(th) if len(th) else None, len(th), hysteresis))

    def render(self, time_s: float, st: OrcSettings, static_pose=False, forced_lod=None, threads=0):
        rgb = np.empty((self.height, self.width, 3), dtype=np.float32)
        T = np.empty((self.height, self.width), dtype=np.float32)
        times = OrcTimes()
        _check(lib().orc_render(self._h, time_s, int(static_pose), -1 if forced_lod is None else forced_lod,
                                C.byref(st), threads, _p(rgb), _p(T), C.byref(times)))
        return rgb, T, times

    def lods(self, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint32)
        if n:
            lib().orc_get_lods(self._h, _p(out))
        return out

    def posed(self) -> np.ndarray:
        g = lib().orc_gaussian_count(self._h)
        out = np.zeros((g, 3), dtype=np.float32)
        if g:
            lib().orc_get_posed(self._h, _p(out))
        return out

    def splats(self) -> np.ndarray:
        s = lib().orc_splat_count(self._h)
        out = np.zeros(s, dtype=SPLAT_DTYPE)
        if s:
            lib().orc_get_splats(self._h, _p(out))
        return out

    def bins(self, tiles: int):
        k = lib().orc_pair_count(self._h)
        counts = np.zeros(tiles, dtype=np.uint32)
        items = np.zeros(max(k, 1), dtype=np.uint32)
        lib().orc_get_bins(self._h, _p(counts), _p(items))
        return counts, items[:k]

    def level_cov(self, t: int, l: int, n: int) -> np.ndarray:
        out = np.zeros((n, 6), dtype=np.float32)
        _check(lib().orc_get_level_cov(self._h, t, l, _p(out)))
        return out


def from_scene(scene, with_instances: bool = True) -> OracleScene:
    """Mirror a paper_2501_17792_b200.Scene (same host arrays) into the oracle."""
    o = OracleScene()
    nt, nm, _ = scene.counts()
    for t in range(nt):
        sk = scene.skeleton(t)
        o.add_template(sk["parents"], sk["inverse_bind"])
        for l in range(scene.level_count(t)):
            o.add_level(t, scene.level_view(t, l))
    for m in range(nm):
        mo = scene.motion(m)
        o.add_motion(mo["fps"], mo["data"], mo["joints"])
    if with_instances:
        o.set_instances(scene.instances)
    c = scene.cfg
    o.set_camera(c.cam_pos, c.cam_look, c.fov_y_deg, c.width, c.height, c.near_m)
    o.set_lod(c.lod_thresholds, c.lod_hysteresis)
    return o


def libm_sinf(x: np.ndarray) -> np.ndarray:
    """The host libm's sinf, elementwise (checker for the device sinf replica)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    lib().orc_libm_sinf(_p(x), _p(out), x.size)
    return out


def libm_expf_range(first_bits: int, n: int) -> np.ndarray:
    """The host libm's expf over n consecutive float bit patterns (checker for the
    rasteriser's device expf replica)."""
    out = np.empty(n, dtype=np.float32)
    lib().orc_libm_expf_range(first_bits, n, _p(out))
    return out
