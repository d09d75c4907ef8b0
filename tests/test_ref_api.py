"""The reference's own unit tests for the callers of the render path, unmodified, against
this repo's drop-in C++ API (SURVEY.md §8b "signatures to keep").

oracle/_ref/ref_api_tests is /root/reference/proj/tests/test_{lod,crowd,renderer,metrics}.cpp
plus its src/bench.cpp (run_benchmark) and src/metrics.cpp (lod_quality_sweep), compiled
against paper_2501_17792_b200/host/gsc/*.hpp and linked to libgsc_host.so / libgscg.so
(oracle/Makefile; doctest and Eigen's double types for tests/oracles.hpp come from shims).
On a B200 every case runs the GPU path: update_crowd, gather_splats, sort_splats,
rasterize_full, render_frame (incl. thread-count determinism and footprint locality),
run_benchmark cells and the LoD quality sweep. Without a GPU the host-only cases must pass
and every other case must fail only with the no-CPU-fallback error.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "ref_api_tests"

pytestmark = pytest.mark.skipif(not BIN.exists(), reason="reference unit tests not built (needs /root/reference)")


def run() -> tuple[list[str], list[str], str]:
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    lines = res.stdout.splitlines()
    ok = [l for l in lines if l.startswith("ok")]
    fail = [l for l in lines if l.startswith("FAIL")]
    return ok, fail, res.stdout[-4000:]


def test_reference_unit_tests_without_gpu_fail_only_for_the_missing_device():
    from tests.conftest import has_gpu
    if has_gpu():
        pytest.skip("a GPU is present: see the gpu test")
    ok, fail, out = run()
    assert len(ok) >= 20, out
    assert all("no CUDA device" in l for l in fail), out


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_b200():
    ok, fail, out = run()
    assert not fail, out
    assert len(ok) == 47, out
