"""ctypes bindings of the two in-tree native libraries.

  lib/libgscg.so      include/gscg.h  — the B200 render path (CUDA, sm_100a)
  lib/libgsc_host.so  include/gsch.h  — host scene layer (gsc API) over libgscg

Loading fails loudly when the libraries are missing: there is no CPU fallback for the
render path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
if os.environ.get("GSCG_LIB_DIR"):  # e.g. lib_checked/ (device bounds checks)
    LIB_DIR = Path(os.environ["GSCG_LIB_DIR"]).resolve()

GSCG_OK = 0
GSCG_ERR_INVALID_ARGUMENT = -1
GSCG_ERR_CUDA = -2
GSCG_ERR_NCCL = -3
GSCG_ERR_OOM = -4
GSCG_ERR_STATE = -5
GSCG_UNIQUE_ID_BYTES = 128
GSCG_LOD_GIVEN = -2
GSCG_SPLIT_ROWS = 0
GSCG_SPLIT_COLS = 1
GSCG_LAYOUT_SHARED = 0
GSCG_LAYOUT_NAIVE = 1
GSCG_MEM_HOST = 0
GSCG_MEM_DEVICE = 1
GSCG_DEBUG_POSED = 1
GSCG_DEBUG_RECORDS = 2
GSCG_DEBUG_NO_CULL = 4
GSCG_MAX_BANDS = 64
GSCG_BAND_SPLAT_BYTES = 64
MAX_LOD_THRESHOLDS = 8


class GscgCamera(C.Structure):
    _fields_ = [("world_to_view", C.c_float * 9), ("position", C.c_float * 3), ("focal", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("near_m", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32)]


class GscgRenderSettings(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("background", C.c_float * 3), ("alpha_max", C.c_float),
                ("alpha_cutoff", C.c_float), ("transmittance_floor", C.c_float), ("sh_enabled", C.c_int32)]


class GscgLodPolicy(C.Structure):
    _fields_ = [("threshold_count", C.c_uint32), ("thresholds_m", C.c_float * MAX_LOD_THRESHOLDS),
                ("hysteresis_band_m", C.c_float)]


GSCG_POSES_GIVEN = 0
GSCG_POSES_SAMPLED = 1


class GscgFrameDesc(C.Structure):
    _fields_ = [("instance_count", C.c_uint32), ("joint_stride", C.c_uint32), ("template_ids", C.c_void_p),
                ("placement", C.c_void_p), ("poses", C.c_void_p), ("active_lod", C.c_void_p),
                ("forced_lod", C.c_int32), ("memory", C.c_int32), ("pose_source", C.c_int32),
                ("time_s", C.c_float), ("static_pose", C.c_int32), ("motion_ids", C.c_void_p),
                ("phase_offsets", C.c_void_p)]


class GscgMotionDesc(C.Structure):
    _fields_ = [("fps", C.c_float), ("frame_count", C.c_uint32), ("joint_count", C.c_uint32),
                ("frames", C.c_void_p)]


class GscgStageTimes(C.Structure):
    _fields_ = [("update_ms", C.c_double), ("gather_ms", C.c_double), ("sort_ms", C.c_double),
                ("rasterize_ms", C.c_double), ("h2d_ms", C.c_double), ("d2h_ms", C.c_double),
                ("splat_count", C.c_uint64), ("pair_count", C.c_uint64), ("gaussian_count", C.c_uint64),
                ("sort_passes", C.c_uint32), ("kernel_launches", C.c_uint32), ("tile_pair_count", C.c_uint64)]


class GscgMemoryUsage(C.Structure):
    _fields_ = [("template_bytes", C.c_uint64), ("frame_bytes", C.c_uint64), ("pinned_bytes", C.c_uint64),
                ("device_free_bytes", C.c_uint64), ("device_total_bytes", C.c_uint64),
                ("naive_attribute_bytes", C.c_uint64)]


class GscgSplatRecord(C.Structure):
    _fields_ = [("ordinal", C.c_uint32), ("instance_id", C.c_uint32), ("gaussian_index", C.c_uint32),
                ("depth", C.c_float), ("mean_px", C.c_float * 2), ("cov_xx", C.c_float), ("cov_xy", C.c_float),
                ("cov_yy", C.c_float), ("conic", C.c_float * 3), ("power_floor", C.c_float), ("opacity", C.c_float),
                ("color", C.c_float * 3), ("rect", C.c_int32 * 4)]


class GschSceneConfig(C.Structure):
    _fields_ = [("template_count", C.c_uint32), ("template_seed_base", C.c_uint64), ("level_count", C.c_uint32),
                ("level_counts", C.c_uint32 * 4), ("joint_count", C.c_uint32), ("with_sh", C.c_int32),
                ("motion_count", C.c_uint32), ("motion_seed_base", C.c_uint64), ("motion_fps", C.c_float),
                ("motion_frames", C.c_uint32), ("grid_rows", C.c_uint32), ("grid_cols", C.c_uint32),
                ("grid_spacing", C.c_float), ("crowd_count", C.c_uint32), ("crowd_seed", C.c_uint64),
                ("cam_pos", C.c_float * 3), ("cam_look", C.c_float * 3), ("fov_y_deg", C.c_float),
                ("width", C.c_uint32), ("height", C.c_uint32), ("near_m", C.c_float),
                ("lod_threshold_count", C.c_uint32), ("lod_thresholds", C.c_float * 8),
                ("lod_hysteresis", C.c_float)]


class GschInstance(C.Structure):
    _fields_ = [("instance_id", C.c_uint32), ("template_id", C.c_uint32), ("motion_id", C.c_uint32),
                ("x", C.c_float), ("z", C.c_float), ("yaw", C.c_float), ("phase_offset_s", C.c_float),
                ("active_lod", C.c_uint32)]


class GschLevelView(C.Structure):
    _fields_ = [("count", C.c_uint32), ("means", C.c_void_p), ("rotations", C.c_void_p), ("scales", C.c_void_p),
                ("opacities", C.c_void_p), ("colors", C.c_void_p), ("skin_indices", C.c_void_p),
                ("skin_weights", C.c_void_p), ("sh", C.c_void_p), ("cov6", C.c_void_p)]


class GschRenderSettings(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("background", C.c_float * 3), ("alpha_max", C.c_float),
                ("alpha_cutoff", C.c_float), ("transmittance_floor", C.c_float), ("thread_count", C.c_int32),
                ("sh_colour", C.c_int32)]


class GschMemoryReport(C.Structure):
    _fields_ = [("naive_bytes", C.c_uint64), ("shared_bytes", C.c_uint64), ("savings_fraction", C.c_double),
                ("naive_marginal_bytes_per_instance", C.c_double), ("shared_marginal_bytes_per_instance", C.c_double),
                ("resident_template_bytes", C.c_uint64), ("posed_mean_bytes", C.c_uint64),
                ("instance_count", C.c_uint64)]


class GschStageTimes(C.Structure):
    _fields_ = [("update_ms", C.c_double), ("gather_ms", C.c_double), ("sort_ms", C.c_double),
                ("rasterize_ms", C.c_double), ("pose_ms", C.c_double), ("total_ms", C.c_double),
                ("splat_count", C.c_uint64), ("pair_count", C.c_uint64), ("gaussian_count", C.c_uint64),
                ("tile_pair_count", C.c_uint64)]


_P = C.c_void_p
GSCG_SYMBOLS = {
    "gscg_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "gscg_destroy": (C.c_int, [_P]),
    "gscg_last_error": (C.c_char_p, [_P]),
    "gscg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "gscg_upload_skeleton": (C.c_int, [_P, C.c_uint32, _P]),
    "gscg_upload_level": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P]),
    "gscg_upload_template": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P]),
    "gscg_template_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "gscg_upload_motion": (C.c_int, [_P, C.c_uint32, C.POINTER(GscgMotionDesc)]),
    "gscg_eval_sinf": (C.c_int, [_P, _P, _P, C.c_uint32]),
    "gscg_eval_expf": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P]),
    "gscg_set_band": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "gscg_set_layout": (C.c_int, [_P, C.c_int32]),
    "gscg_set_region": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "gscg_group_unique_id": (C.c_int, [_P]),
    "gscg_group_create": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "gscg_create_group": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "gscg_group_destroy": (C.c_int, [_P]),
    "gscg_group_render_frame": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera),
                                          C.POINTER(GscgRenderSettings), C.POINTER(GscgLodPolicy), C.c_int32, _P,
                                          _P, _P, C.POINTER(GscgStageTimes)]),
    "gscg_group_render_frame_async": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera),
                                                C.POINTER(GscgRenderSettings), C.POINTER(GscgLodPolicy), C.c_int32,
                                                _P, _P, _P, C.POINTER(GscgStageTimes)]),
    "gscg_group_wait_readback": (C.c_int, [_P]),
    "gscg_group_framebuffer_device": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P)]),
    "gscg_group_tile_costs": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P]),
    "gscg_gather_splats": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera),
                                     C.POINTER(GscgRenderSettings), C.POINTER(GscgLodPolicy), _P, C.c_uint64,
                                     C.POINTER(C.c_uint64)]),
    "gscg_sort_splats": (C.c_int, [_P, _P, C.c_uint64]),
    "gscg_skin_means": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera), C.POINTER(GscgLodPolicy), _P,
                                  C.c_uint64, C.POINTER(C.c_uint64)]),
    "gscg_gather_posed": (C.c_int, [_P, C.POINTER(GscgFrameDesc), _P, C.c_uint64, _P, C.POINTER(GscgCamera),
                                    C.POINTER(GscgRenderSettings), _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    "gscg_rasterize_splats": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(GscgRenderSettings),
                                        _P, _P]),
    "gscg_set_debug": (C.c_int, [_P, C.c_uint32]),
    "gscg_render_frame": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera),
                                    C.POINTER(GscgRenderSettings), C.POINTER(GscgLodPolicy), _P, _P,
                                    C.POINTER(GscgStageTimes)]),
    "gscg_render_frame_async": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera),
                                          C.POINTER(GscgRenderSettings), C.POINTER(GscgLodPolicy), _P, _P,
                                          C.POINTER(GscgStageTimes)]),
    "gscg_wait_readback": (C.c_int, [_P, C.c_uint32]),
    "gscg_memory_usage": (C.c_int, [_P, C.POINTER(GscgMemoryUsage)]),
    "gscg_device_alloc": (C.c_int, [_P, C.c_uint64, C.POINTER(_P)]),
    "gscg_device_free": (C.c_int, [_P, _P]),
    "gscg_psnr": (C.c_int, [_P, _P, _P, C.c_uint64, C.POINTER(C.c_float)]),
    "gscg_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(_P)]),
    "gscg_host_free": (C.c_int, [_P]),
    "gscg_framebuffer_device": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P)]),
    "gscg_synchronize": (C.c_int, [_P]),
    "gscg_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "gscg_get_counts": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "gscg_get_instances_culled": (C.c_int, [_P, C.POINTER(C.c_uint32)]),
    "gscg_get_lod": (C.c_int, [_P, _P, C.c_uint32]),
    "gscg_get_instance_base": (C.c_int, [_P, _P, C.c_uint32]),
    "gscg_get_posed_means": (C.c_int, [_P, _P, C.c_uint64]),
    "gscg_get_splat_records": (C.c_int, [_P, _P, C.c_uint64]),
    "gscg_get_cell_layout": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "gscg_get_tile_ranges": (C.c_int, [_P, _P, C.c_uint32]),
    "gscg_get_sorted_ordinals": (C.c_int, [_P, _P, C.c_uint64]),
    "gscg_get_sorted_values": (C.c_int, [_P, _P, C.c_uint64]),
    "gscg_project_shard": (C.c_int, [_P, C.POINTER(GscgFrameDesc), C.POINTER(GscgCamera),
                                     C.POINTER(GscgRenderSettings), C.POINTER(GscgLodPolicy), C.c_uint32,
                                     C.c_uint32, C.c_uint32, _P, _P, C.POINTER(GscgStageTimes)]),
    "gscg_pack_bands": (C.c_int, [_P, _P]),
    "gscg_render_band": (C.c_int, [_P, _P, C.c_uint64, C.c_uint32, C.c_uint32, _P, _P, C.c_int32,
                                   C.POINTER(GscgStageTimes)]),
}

GSCH_ERR_FORMAT = -6


class GschQualityRow(C.Structure):
    _fields_ = [("distance_m", C.c_float), ("level", C.c_uint32), ("gaussian_count", C.c_uint32),
                ("psnr_db", C.c_float)]


GSCH_SYMBOLS = {
    "gsch_psnr": (C.c_int, [_P, _P, C.c_uint32, C.c_uint32, C.POINTER(C.c_float)]),
    "gsch_lod_quality_sweep": (C.c_int, [_P, C.c_uint32, _P, C.c_uint32, _P, C.c_int, _P, C.c_uint32,
                                         C.POINTER(C.c_uint32)]),
    "gsch_scene_update_crowd": (C.c_int, [_P, C.c_int32]),
    "gsch_scene_save_template": (C.c_int, [_P, C.c_uint32, C.c_char_p]),
    "gsch_scene_load_template": (C.c_int, [_P, C.c_uint32, C.c_char_p]),
    "gsch_scene_save_motion": (C.c_int, [_P, C.c_uint32, C.c_char_p]),
    "gsch_scene_load_motion": (C.c_int, [_P, C.c_uint32, C.c_char_p]),
    "gsch_last_error": (C.c_char_p, []),
    "gsch_scene_create": (C.c_int, [C.POINTER(GschSceneConfig), C.c_int, C.POINTER(_P)]),
    "gsch_scene_destroy": (C.c_int, [_P]),
    "gsch_scene_counts": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "gsch_scene_get_instances": (C.c_int, [_P, _P, C.c_uint32]),
    "gsch_scene_set_instances": (C.c_int, [_P, _P, C.c_uint32]),
    "gsch_scene_set_camera": (C.c_int, [_P, _P, _P, C.c_float, C.c_uint32, C.c_uint32, C.c_float]),
    "gsch_scene_camera_basis": (C.c_int, [_P, C.POINTER(GscgCamera)]),
    "gsch_scene_set_lod_policy": (C.c_int, [_P, _P, C.c_uint32, C.c_float]),
    "gsch_scene_level_count": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_uint32)]),
    "gsch_scene_level_view": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.POINTER(GschLevelView)]),
    "gsch_scene_skeleton": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(_P), C.POINTER(_P)]),
    "gsch_scene_motion": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_float), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32), _P]),
    "gsch_scene_sample_crowd": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, C.c_uint32, _P, _P, _P]),
    "gsch_scene_set_motion": (C.c_int, [_P, C.c_uint32, C.c_float, C.c_uint32, C.c_uint32, _P]),
    "gsch_memory_report_cell": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(GschMemoryReport)]),
    "gsch_scene_memory_report": (C.c_int, [_P, C.POINTER(GschMemoryReport)]),
    "gsch_renderer_set_device_poses": (C.c_int, [_P, C.c_int32]),
    "gsch_gather_splats": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, _P, _P, C.c_uint64,
                                     C.POINTER(C.c_uint64)]),
    "gsch_sort_splats": (C.c_int, [_P, _P, C.c_uint64]),
    "gsch_rasterize_splats": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_int32, _P, _P, _P]),
    "gsch_renderer_prepare": (C.c_int, [_P]),
    "gsch_fill_instances": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, _P]),
    "gsch_renderer_create": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "gsch_renderer_destroy": (C.c_int, [_P]),
    "gsch_renderer_gpu": (_P, [_P]),
    "gsch_renderer_joint_stride": (C.c_uint32, [_P]),
    "gsch_render": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, C.POINTER(GschRenderSettings), _P, _P,
                              C.POINTER(GschStageTimes)]),
    "gsch_render_async": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, C.POINTER(GschRenderSettings), _P, _P,
                                    C.POINTER(GschStageTimes)]),
    "gsch_wait_readback": (C.c_int, [_P, C.c_uint32]),
    "gsch_sample_crowd": (C.c_int, [_P, C.c_float, C.c_int32, C.c_int32, _P, _P, _P]),
}

_libs: dict[str, C.CDLL] = {}


def _load(name: str, symbols: dict) -> C.CDLL:
    if name in _libs:
        return _libs[name]
    path = LIB_DIR / name
    if not path.exists():
        raise RuntimeError(f"{path} is missing: build the native libraries first "
                           "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
    for sym, (res, args) in symbols.items():
        fn = getattr(lib, sym)
        fn.restype = res
        fn.argtypes = args
    _libs[name] = lib
    return lib


def gscg() -> C.CDLL:
    return _load("libgscg.so", GSCG_SYMBOLS)


def gsch() -> C.CDLL:
    gscg()
    return _load("libgsc_host.so", GSCH_SYMBOLS)


class NativeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[status {status}] {message}")
        self.status = status


class FormatError(NativeError):
    """Typed asset-file failure (reference io.hpp FormatError); .kind is one of IoError,
    BadMagic, VersionMismatch, Truncated, InvariantViolation."""

    def __init__(self, message: str):
        kind, _, rest = message.partition("] ")
        self.kind = kind.lstrip("[") if rest else "Unknown"
        super().__init__(GSCH_ERR_FORMAT, rest or message)


def check_gsch(status: int) -> None:
    if status != 0:
        msg = gsch().gsch_last_error().decode(errors="replace")
        if status == GSCG_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if status == GSCH_ERR_FORMAT:
            raise FormatError(msg)
        raise NativeError(status, msg)


def check_gscg(status: int, ctx) -> None:
    if status != 0:
        msg = gscg().gscg_last_error(ctx).decode(errors="replace")
        if status == GSCG_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        raise NativeError(status, msg)
