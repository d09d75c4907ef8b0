"""The parity suite's core cases again on the checked build (lib_checked/: device bounds
checks, GSCG_DCHECK in csrc/gscg_common.cuh). compute-sanitizer is closed on the GPU pool,
so out-of-range bucket, staging, rank and sort-output indices are caught by the kernels
themselves: a failed check traps and the render call returns a CUDA error."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2501_17792_b200" / "lib_checked"

CASES = ("test_fixture_scene or test_tile_sizes or test_forced_lod or test_hysteresis_across_frames "
         "or test_long_equal_depth_runs or test_truncated_depth_sort or test_lsd_depth_sort "
         "or test_bucket_sort_large_buckets or test_baseline_config or test_band_frames "
         "or test_column_regions or test_naive_layout or test_empty_crowd or test_extreme_gaussians "
         "or test_extreme_cameras")


@pytest.mark.gpu
def test_parity_cases_pass_with_device_bounds_checks():
    assert (CHECKED / "libgscg.so").exists(), "build() makes lib_checked/ next to lib/"
    env = dict(os.environ, GSCG_LIB_DIR=str(CHECKED))
    res = subprocess.run([sys.executable, "-m", "pytest", str(ROOT / "tests" / "test_gpu_parity.py"), "-m", "gpu",
                          "-q", "-x", "-p", "no:cacheprovider", "-k", CASES + " and not config3 and not config4"],
                         capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    assert "GSCG_DCHECK failed" not in res.stdout + res.stderr, tail
    assert " passed" in res.stdout, tail


def test_checked_library_is_loaded_from_gscg_lib_dir():
    """GSCG_LIB_DIR redirects the loader (CPU check: the path only, no device call)."""
    code = ("import paper_2501_17792_b200.native as N; print(N.LIB_DIR)")
    env = dict(os.environ, GSCG_LIB_DIR=str(CHECKED))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr
    assert Path(res.stdout.strip()) == CHECKED.resolve()


def test_checked_build_carries_the_device_checks_and_the_product_does_not():
    checked = (CHECKED / "libgscg.so").read_bytes()
    product = (ROOT / "paper_2501_17792_b200" / "lib" / "libgscg.so").read_bytes()
    assert b"GSCG_DCHECK failed" in checked
    assert b"GSCG_DCHECK failed" not in product
