"""Builds the in-tree native library `libflexmoe_b200.so` for sm_100a.

Plain nvcc, no torch extension machinery: every `.cu` / `.cpp` under
`csrc/` is compiled to an object under `build/` (incremental, parallel) and
linked into `paper_2304_03946_b200/libflexmoe_b200.so`, which travels to the
GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "flexmoe_b200"
LIB = PKG / "libflexmoe_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
CU_FLAGS = ARCH + COMMON + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
# extra nvcc flags for A/B builds (e.g. NVCC_EXTRA=-DFM_GEMM_DIRECT_STORE)
CU_FLAGS += os.environ.get("NVCC_EXTRA", "").split()


def _deps_newer(src: Path, obj: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
    return any(p.stat().st_mtime > t for p in [src, *headers])


def _compile(src: Path, verbose: bool) -> tuple[Path, str]:
    obj = BUILD / (src.name + ".o")
    if not _deps_newer(src, obj):
        return obj, ""
    flags = CU_FLAGS if src.suffix == ".cu" else ARCH + COMMON + os.environ.get("NVCC_EXTRA", "").split()
    cmd = [NVCC, *flags, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
    return obj, res.stderr if verbose else ""


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    sources = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), sources))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            print(log, file=sys.stderr)
    if not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
