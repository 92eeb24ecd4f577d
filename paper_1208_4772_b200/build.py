"""In-tree build of the sm_100a extension (nvcc) and the oracle checkers.

    python -m paper_1208_4772_b200.build          # libcdg_gpu.so (+ oracle when present)

The product library is ``paper_1208_4772_b200/libcdg_gpu.so`` (C ABI,
include/cdg_gpu.h). Compiled for sm_100a only; -lineinfo for ncu source maps.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libcdg_gpu.so"


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    raise FileNotFoundError("nvcc not found")


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_gpu(force: bool = False, verbose: bool = False) -> Path:
    """Compile every translation unit (cdg_gpu.cu + the kernel-set TUs
    sets_*.cu) to an object in parallel, then link libcdg_gpu.so."""
    headers = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "cdg_gpu.h"]
    units = sorted(CSRC.glob("*.cu"))
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    comp = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-ccbin", "/usr/bin/g++", "-I", str(ROOT / "include")]
    procs, objs = [], []
    for cu in units:
        obj = objdir / (cu.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [cu] + headers):
            cmd = comp + ["-c", "-o", str(obj), str(cu)]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((cu, subprocess.Popen(cmd)))
    for cu, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, f"nvcc {cu.name}")
    if force or procs or _stale(LIB, objs):
        cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", "/usr/bin/g++",
               "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


def build_variant(tag: str, defines, units=("sets_p4",), verbose: bool = False) -> Path:
    """Tuning experiments only (not the product): recompile the kernel-set TUs
    `units` with extra -D`defines` into build/<tag>/ and link
    variants/libcdg_gpu_<tag>.so with the product objects of every other TU.
    scripts/tune_p4.py times such libraries side by side (gpu.use_library)."""
    build_gpu()
    headers = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "cdg_gpu.h"]
    objdir = PKG / "build" / tag
    objdir.mkdir(parents=True, exist_ok=True)
    out = PKG / "variants" / f"libcdg_gpu_{tag}.so"
    out.parent.mkdir(exist_ok=True)
    comp = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-ccbin", "/usr/bin/g++", "-I", str(ROOT / "include")]
    comp += [f"-D{d}" for d in defines]
    objs = []
    for cu in sorted(CSRC.glob("*.cu")):
        if cu.stem in units:
            obj = objdir / (cu.stem + ".o")
            if _stale(obj, [cu] + headers) or not (objdir / "defines").exists() or \
                    (objdir / "defines").read_text() != " ".join(defines):
                cmd = comp + ["-c", "-o", str(obj), str(cu)]
                if verbose:
                    print(" ".join(cmd), flush=True)
                subprocess.run(cmd, check=True)
            objs.append(obj)
        else:
            objs.append(PKG / "build" / (cu.stem + ".o"))
    (objdir / "defines").write_text(" ".join(defines))
    subprocess.run([_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", "/usr/bin/g++",
                    "-o", str(out), *map(str, objs)], check=True)
    return out


def build_oracle(verbose: bool = False) -> None:
    """oracle/: the C restatement always; oracle/_ref when /root/reference exists."""
    env = dict(os.environ)
    env.pop("CXX", None)
    env.pop("CC", None)
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8", "port"], check=True, env=env)
    if Path("/root/reference/proj/core/src/solver.cpp").exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8", "ref"], check=True, env=env)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    build_gpu(force="--force" in argv, verbose=True)
    if "--no-oracle" not in argv:
        build_oracle()
    print(f"built {LIB}")


if __name__ == "__main__":
    main()
