"""The pipelined-frame parity tests again under the other stream schedules the render path
can take (csrc/gscg_api.cu): stream priorities (GSCG_STREAM_PRIO), the sort on the render
stream (GSCG_SPLIT_SORT=0), the front half not overlapped (GSCG_OVERLAP_UPDATE=0). The
frames must not depend on how the three streams interleave, so each schedule reproduces
the oracle's frames and the synchronous render's. Each runs in its own process (the
settings are read once per process)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

CASES = ("pipelined or hysteresis or (baseline_config and not config3 and not config4) "
         "or (gpu_matches_reference_build and not config3)")

SCHEDULES = {
    "equal-priorities": {"GSCG_STREAM_PRIO": "0"},
    "front-first": {"GSCG_STREAM_PRIO": "1"},
    "sort-above-raster": {"GSCG_STREAM_PRIO": "2"},
    "one-stream": {"GSCG_SPLIT_SORT": "0", "GSCG_OVERLAP_UPDATE": "0"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SCHEDULES))
def test_pipelined_frames_under_each_stream_schedule(name):
    env = dict(os.environ, **SCHEDULES[name])
    res = subprocess.run([sys.executable, "-m", "pytest", str(ROOT / "tests" / "test_gpu_parity.py"), "-m", "gpu",
                          "-q", "-x", "-p", "no:cacheprovider", "-k", CASES],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    tail = (res.stdout + res.stderr)[-3000:]
    assert res.returncode == 0, tail
    assert " passed" in res.stdout and " failed" not in res.stdout, tail
