"""B200-native CrowdSplat crowd-render path (arXiv 2501.17792).

The per-frame path of the reference's ``gsc::render_frame`` — distance LoD, instanced
LBS of shared template Gaussians, EWA projection with SH colour, tile|depth sort and
per-tile blending — runs in hand-written sm_100a CUDA kernels behind the C-ABI in
include/gscg.h. The C++ host API (host/gsc, C-ABI include/gsch.h) keeps the reference's
template / instance / camera interface; this package is its Python face.
"""
from .api import (RenderSettings, Renderer, Scene, SceneConfig, StageTimes, baseline_config,  # noqa: F401
                  place_origin_instance, psnr, render_frame)
from .native import FormatError, NativeError  # noqa: F401

__all__ = ["RenderSettings", "Renderer", "Scene", "SceneConfig", "StageTimes", "baseline_config",
           "place_origin_instance", "psnr", "render_frame", "NativeError", "FormatError"]
