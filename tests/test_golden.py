"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py).

CPU: the code each fixture came from (the reference build for RGB fixtures, the oracle for
the SH-extension one) and the oracle restatement + the product's host generator both
still reproduce every fixture bit for bit.
GPU: the CUDA path reproduces the fixtures through the C-ABI with the same bars as the
live-oracle parity tests (tests/parity.py), without running the oracle.
"""
from __future__ import annotations

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load(name: str):
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}


class GoldenOracle:
    """Read-only stand-in for oracle.orc.OracleScene backed by a fixture."""

    def __init__(self, arrays):
        self.a = arrays

    def lods(self, n):
        assert n == len(self.a["lods"])
        return self.a["lods"]

    def posed(self):
        return self.a["posed"]

    def splats(self):
        return self.a["splats"]

    def bins(self, tiles):
        assert tiles == len(self.a["bin_counts"])
        return self.a["bin_counts"], self.a["bin_items"]


def test_golden_fixtures_present():
    assert len(CASES) >= 2


@pytest.mark.parametrize("source", ["fixture", "oracle"])
@pytest.mark.parametrize("name", CASES)
def test_reproduces_golden(name, source):
    import sys
    sys.path.insert(0, str(GOLDEN))
    from make_golden import render_case
    from oracle import ref

    meta, gold = load(name)
    src = meta.get("source", "oracle") if source == "fixture" else "oracle"
    if src == "reference" and not ref.available():
        pytest.skip("reference build (oracle/_ref) unavailable")
    cfg = meta["config"]
    cfg = {k: tuple(v) if isinstance(v, list) else v for k, v in cfg.items()}
    now = render_case(cfg, meta["render"], src)
    for k, v in gold.items():
        assert now[k].dtype == v.dtype and now[k].shape == v.shape, k
        assert now[k].tobytes() == v.tobytes(), f"{name}: {k} drifted from the golden fixture ({src})"


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_matches_golden(name):
    import paper_2501_17792_b200 as P
    from tests.parity import check_frame
    from paper_2501_17792_b200 import native as N

    meta, gold = load(name)
    cfg = {k: tuple(v) if isinstance(v, list) else v for k, v in meta["config"].items()}
    r = meta["render"]
    scene = P.Scene(P.SceneConfig(**cfg))
    renderer = P.Renderer(scene, device=0)
    renderer.set_debug(N.GSCG_DEBUG_POSED | N.GSCG_DEBUG_RECORDS)
    st = P.RenderSettings(tile_size=r["tile_size"], background=tuple(r["background"]), sh_colour=r["sh"])
    rgb, T = renderer.render_frame(r["time_s"], st, r.get("static_pose", False), r.get("forced_lod"))
    c = gold["counts"]
    times = SimpleNamespace(gaussian_count=int(c[0]), splat_count=int(c[1]), pair_count=int(c[2]))
    rep = check_frame(scene, renderer, GoldenOracle(gold), (rgb, T), (gold["rgb"], gold["T"], times),
                      tile_size=r["tile_size"])
    assert rep["psnr"] >= 50.0
