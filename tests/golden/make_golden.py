"""Regenerates tests/golden/*.npz: small crowd frames with their full parity state.

The reference ships no golden images. RGB fixtures ("source":
"reference") are rendered by the REFERENCE's own code: oracle/_ref/libgsc_ref.so, its
unmodified src/*.cpp compiled against the Eigen-subset shim (oracle/Makefile), from its
own synthetic generator and build_crowd. The SH fixture ("source": "oracle") exercises
the SH-deg-3 colour extension, which the reference does not have,
so it comes from the oracle restatement, itself bit-identical to the reference on RGB
frames (tests/test_reference_pin.py). CPU tests check both still reproduce them; the GPU
tests check the CUDA path against them without running either (-m gpu).

Run from the repo root after building:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

# (name, SceneConfig kwargs, render kwargs); sh=False cases come from the reference build.
CASES = [
    ("crowd6_sh_t16",
     dict(template_count=2, template_seed_base=100, level_counts=(1500, 400, 100), with_sh=True,
          motion_count=2, motion_frames=60, grid_rows=2, grid_cols=3, crowd_count=6, crowd_seed=11,
          cam_pos=(1.0, 1.4, -2.5), cam_look=(1.0, 1.0, 3.0), width=160, height=120,
          lod_thresholds=(3.0, 4.5)),
     dict(time_s=0.41, tile_size=16, background=(0.05, 0.1, 0.2), sh=True)),
    ("crowd4_rgb_t8_static",
     dict(template_count=1, template_seed_base=300, level_counts=(1200, 300), with_sh=False,
          motion_count=1, motion_frames=30, grid_rows=2, grid_cols=2, crowd_count=4, crowd_seed=5,
          cam_pos=(0.5, 1.2, -2.0), cam_look=(0.5, 0.9, 2.0), width=96, height=80,
          lod_thresholds=(3.0,)),
     dict(time_s=0.0, tile_size=8, background=(0.0, 0.0, 0.0), sh=False, static_pose=True)),
    ("crowd12_rgb_t16_hyst",
     dict(template_count=3, template_seed_base=104, level_counts=(2500, 600, 140), with_sh=False,
          motion_count=3, motion_frames=60, grid_rows=3, grid_cols=4, crowd_count=12, crowd_seed=9,
          cam_pos=(1.5, 1.5, -2.5), cam_look=(1.5, 1.0, 4.0), width=200, height=112,
          lod_thresholds=(2.5, 4.0), lod_hysteresis=0.5),
     dict(time_s=0.73, tile_size=16, background=(0.1, 0.05, 0.0), sh=False, forced_lod=None)),
]


def render_case(cfg_kw: dict, r_kw: dict, source: str | None = None):
    """source: "reference" (oracle/_ref, RGB only) or "oracle" (orc.cpp from the product
    scene); default: the reference for RGB cases, the oracle for SH ones."""
    source = source or ("oracle" if r_kw["sh"] else "reference")
    if source == "reference":
        from oracle import ref

        o = ref.RefScene(ref.RefConfig(**{k: v for k, v in cfg_kw.items() if k != "with_sh"}))
        st = ref.settings(tile_size=r_kw["tile_size"], background=r_kw["background"])
        n = o.counts()[2]
    else:
        import paper_2501_17792_b200 as P
        from oracle import orc

        scene = P.Scene(P.SceneConfig(**cfg_kw))
        o = orc.from_scene(scene)
        st = orc.settings(tile_size=r_kw["tile_size"], background=r_kw["background"], sh_colour=r_kw["sh"])
        n = scene.counts()[2]
    rgb, T, times = o.render(r_kw["time_s"], st, r_kw.get("static_pose", False), r_kw.get("forced_lod"))
    lods = o.lods(n)
    sp = o.splats()
    ts = r_kw["tile_size"]
    tiles = ((cfg_kw["width"] + ts - 1) // ts) * ((cfg_kw["height"] + ts - 1) // ts)
    counts, items = o.bins(tiles)
    return dict(
        rgb=rgb, T=T, lods=lods,
        counts=np.array([times.gaussian_count, times.splat_count, times.pair_count], dtype=np.uint64),
        splats=sp, posed=o.posed(), bin_counts=counts, bin_items=items,
    )


def main() -> None:
    from paper_2501_17792_b200.build import build, build_oracle
    build()
    build_oracle()
    out = Path(__file__).resolve().parent
    for name, cfg_kw, r_kw in CASES:
        arrays = render_case(cfg_kw, r_kw)
        meta = json.dumps(dict(config=cfg_kw, render=r_kw, source="oracle" if r_kw["sh"] else "reference"))
        np.savez_compressed(out / f"{name}.npz", meta=np.array(meta), **arrays)
        c = arrays["counts"]
        print(f"{name}: G={c[0]} S={c[1]} K={c[2]} -> {name}.npz")


if __name__ == "__main__":
    main()
