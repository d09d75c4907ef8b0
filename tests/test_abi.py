"""The C-ABI libraries load and export every entry point their headers declare; without a
GPU the render path refuses to start (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2501_17792_b200 import native as N
from tests.conftest import has_gpu

ROOT = Path(__file__).resolve().parents[1]


def declared(header: str) -> list[str]:
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b((?:gscg|gsch)_\w+)\s*\(", text, flags=re.M)))


@pytest.mark.parametrize("header,loader", [("gscg.h", N.gscg), ("gsch.h", N.gsch)])
def test_every_declared_symbol_is_exported(header, loader):
    names = declared(header)
    assert len(names) >= 10
    lib = loader()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    table = N.GSCG_SYMBOLS if header == "gscg.h" else N.GSCH_SYMBOLS
    assert set(names) == set(table), set(names) ^ set(table)


def test_struct_layouts_match_headers():
    assert C.sizeof(N.GscgCamera) == 4 * (9 + 3 + 4 + 2)
    assert C.sizeof(N.GscgSplatRecord) == 4 * (3 + 1 + 2 + 3 + 3 + 1 + 1 + 3 + 4)
    assert C.sizeof(N.GscgFrameDesc) == 8 + 4 * 8 + 8 + 4 * 4 + 2 * 8


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_create_without_gpu_fails_loudly():
    ctx = C.c_void_p()
    st = N.gscg().gscg_create(0, C.byref(ctx))
    assert st == N.GSCG_ERR_CUDA
    assert b"no CUDA device" in N.gscg().gscg_last_error(ctx)
    N.gscg().gscg_destroy(ctx)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_renderer_without_gpu_raises():
    import paper_2501_17792_b200 as P

    s = P.Scene(P.SceneConfig())
    with pytest.raises(P.NativeError):
        P.Renderer(s)


def test_oracle_is_not_on_the_product_path():
    """The product package never imports or links the oracle."""
    pkg = ROOT / "paper_2501_17792_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cpp")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.h*")):
        if f.name == "build.py":
            continue  # builds the checker next to the product, never links it
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text and "liborc" not in text, f
