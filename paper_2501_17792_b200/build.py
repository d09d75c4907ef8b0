"""Build recipe for the B200 crowd renderer's native libraries (in-tree).

  lib/libgscg.so      CUDA kernels + C-ABI (include/gscg.h), sm_100a only
  lib/libgsc_host.so  C++ host API (namespace gsc) + C-ABI for Python (include/gsch.h)
  lib_checked/        both again with device bounds checks (-DGSCG_DEVICE_CHECKS)

Parity-critical translation units (update, project) are compiled with --fmad=false so
no multiply-add is contracted; host code uses -ffp-contract=off and no -march, the
reference's Release floating-point contract.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
LIB = PKG / "lib"
OBJ = PKG / "_obj"
LIB_CHECKED = PKG / "lib_checked"
OBJ_CHECKED = PKG / "_obj_checked"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
              "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}"] + ARCH
EXACT_TUS = {"gscg_update.cu", "gscg_project.cu", "gscg_pose.cu"}
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
             f"-I{INCLUDE}", f"-I{HOST}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 path cannot be built")


def _cxx() -> str:
    return os.environ.get("CXX") or shutil.which("g++") or "g++"


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], log: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build step failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}{res.stderr}")


def build(verbose: bool = False, force: bool = False) -> dict[str, Path]:
    out = _build_variant(LIB, OBJ, [], verbose, force)
    # lib_checked/: the same sources with device bounds checks (GSCG_DCHECK, gscg_common.cuh),
    # loaded by the checked-build GPU test through GSCG_LIB_DIR (compute-sanitizer is closed
    # on the GPU pool).
    _build_variant(LIB_CHECKED, OBJ_CHECKED, ["-DGSCG_DEVICE_CHECKS"], verbose, force)
    return out


def _build_variant(LIB: Path, OBJ: Path, defines: list[str], verbose: bool, force: bool) -> dict[str, Path]:
    LIB.mkdir(exist_ok=True)
    OBJ.mkdir(exist_ok=True)
    nvcc = _nvcc()
    log: list[str] = []
    headers = sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    cu = sorted(CSRC.glob("*.cu"))
    objs = []
    jobs = []
    for src in cu:
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            flags = list(NVCC_FLAGS) + defines + (["--fmad=false"] if src.name in EXACT_TUS else [])
            jobs.append([nvcc, "-c", str(src), "-o", str(obj)] + flags)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for f in [ex.submit(_run, j, log) for j in jobs]:
            f.result()
    gscg = LIB / "libgscg.so"
    if force or jobs or _stale(gscg, objs):
        _run([nvcc, "-shared", "-o", str(gscg)] + [str(o) for o in objs] + ARCH + ["-lcudart_static", "-lrt", "-lpthread", "-ldl"], log)

    host_src = sorted((HOST / "gsc").glob("*.cpp")) + [HOST / "gsch_capi.cpp"]
    host_hdr = sorted((HOST / "gsc").glob("*.hpp")) + sorted(INCLUDE.glob("*.h"))
    host_lib = LIB / "libgsc_host.so"
    if force or _stale(host_lib, host_src + host_hdr + [gscg]):
        _run([_cxx(), "-shared", "-o", str(host_lib)] + CXX_FLAGS + [str(s) for s in host_src]
             + [f"-L{LIB}", "-lgscg", "-Wl,-rpath,$ORIGIN", "-lpthread"], log)
    if verbose:
        print("\n".join(log))
    return {"gscg": gscg, "host": host_lib}


def build_oracle(verbose: bool = False) -> Path:
    oracle = ROOT / "oracle"
    res = subprocess.run(["make", "-C", str(oracle)], capture_output=True, text=True)
    if verbose:
        print(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + res.stdout + res.stderr)
    # oracle/_ref: the reference's own sources (read in place under /root/reference,
    # which exists only in the build container) + the Eigen-subset shim. The built .so
    # travels to the GPU box with the repo; there it is used prebuilt.
    if Path("/root/reference/proj/src/renderer.cpp").exists():
        res = subprocess.run(["make", "-C", str(oracle), "ref"], capture_output=True, text=True)
        if verbose:
            print(res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError("reference build (oracle/_ref) failed:\n" + res.stdout + res.stderr)
    return oracle / "_build" / "liborc.so"


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    build_oracle(verbose="-v" in sys.argv)
