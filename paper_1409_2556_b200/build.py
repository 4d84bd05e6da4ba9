"""Build the in-tree sm_100a library `_lib/liblaptomo_gpu.so` with nvcc.

Every translation unit is compiled for `-gencode arch=compute_100a,code=sm_100a`
with `-lineinfo` (ncu source view); objects go to build/, the shared library
stays in-tree so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "liblaptomo_gpu.so"
OBJ_DIR = ROOT / "build" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          f"-I{ROOT / 'include'}", f"-I{CSRC}", "--expt-relaxed-constexpr"]


def sources():
    return sorted([p for p in CSRC.iterdir() if p.suffix in (".cu", ".cpp")])


def headers():
    hs = [p for p in CSRC.iterdir() if p.suffix in (".cuh", ".hpp", ".h")]
    hs += list((ROOT / "include").glob("*.h"))
    return hs


def _needs(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, verbose: bool, defines=(), tag: str = "") -> Path:
    obj = OBJ_DIR / (src.name + tag + ".o")
    if _needs(obj, [src] + headers()):
        cmd = [NVCC, *ARCH, *COMMON, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr:
            print(res.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, defines=(), variant: str = "") -> Path:
    """variant != "": an experiment build with extra -D defines into liblaptomo_gpu_<variant>.so."""
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    lib = LIB if not variant else OUT_DIR / f"liblaptomo_gpu_{variant}.so"
    tag = f".{variant}" if variant else ""
    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, defines, tag), srcs))
    if _needs(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs), "-lcufft", "-lcublas", "-lcusolver"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
