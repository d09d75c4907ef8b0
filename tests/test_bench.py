"""bench.py contract on CPU: the --gpus N launcher (torchrun re-exec, one JSON line from
rank 0, max over ranks), and a reference arm that never loads the product libraries."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_gpus_flag_launches_that_many_ranks():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, res.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["ranks_seen"] == 2 and out["ms_per_step"] >= 20.0  # max over ranks (rank 1 sleeps 20 ms)


def test_gpus_mismatch_with_world_size_is_an_error():
    import os
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT, env=env)
    assert res.returncode == 2


def test_reference_arm_is_independent_of_the_product():
    """The reference arm renders through oracle/_ref (the reference's own sources); the
    product's libgscg.so / libgsc_host.so must not be mapped into that process."""
    from oracle import ref
    if not ref.available():
        pytest.skip("reference build unavailable")
    code = (
        "import sys, json; sys.argv=['bench.py','--impl','reference','--config','1','--steps','2','--warmup','3'];"
        f"sys.path.insert(0, {str(ROOT)!r}); import bench; bench.main();"
        "maps = open('/proc/self/maps').read();"
        "print(json.dumps({'product_module': 'paper_2501_17792_b200' in sys.modules,"
        " 'gscg': 'libgscg.so' in maps, 'host': 'libgsc_host.so' in maps, 'ref': 'libgsc_ref.so' in maps}))")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr
    line, probe = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["splats"] == 100000 and line["config"]["instances"] == 1
    assert probe == {"product_module": False, "gscg": False, "host": False, "ref": True}
