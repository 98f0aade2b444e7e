"""Build libkvt.so in-tree: every CUDA source compiled for sm_100a only (no other arch, no PTX JIT).

    python paper_2502_04420_b200/build.py [--force] [--verbose] [--variant NAME -D MACRO=VALUE ...]

Object files go to paper_2502_04420_b200/build/ and are compiled in parallel; the shared library
is linked with the static CUDA runtime.  ptxas resource usage (-Xptxas -v) is written to
build/ptxas.log for inspection (registers, spills, shared memory).
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "libkvt.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I", str(INCLUDE), "-I", str(CSRC)]


def sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def headers():
    return sorted(list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")))


def _compile(src: Path, force: bool, defines=(), bdir: Path = BUILD) -> tuple[Path, str]:
    obj = bdir / (src.name + ".o")
    dep_mtime = max([src.stat().st_mtime] + [h.stat().st_mtime for h in headers()])
    if not force and obj.exists() and obj.stat().st_mtime >= dep_mtime:
        return obj, ""
    lang = ["-x", "cu"]
    cmd = [NVCC, *ARCH, *CFLAGS, *[f"-D{d}" for d in defines], *lang, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, defines=(), variant: str = "") -> Path:
    """Build libkvt.so (or, for kernel A/B experiments, libkvt_<variant>.so with extra -D defines)."""
    bdir = BUILD / variant if variant else BUILD
    lib = LIB.with_name(f"libkvt_{variant}.so") if variant else LIB
    bdir.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, defines, bdir), srcs))
    logs = [log for _, log in results if log]
    if logs:
        (bdir / "ptxas.log").write_text("\n".join(logs))
    objs = [o for o, _ in results]
    newest = max(o.stat().st_mtime for o in objs)
    if force or not lib.exists() or lib.stat().st_mtime < newest:
        tmp = lib.with_name(f"{lib.name}.tmp{os.getpid()}")
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    _stamp(lib)
    if verbose:
        print(f"built {lib}")
    return lib


def _stamp(lib: Path):
    """BUILD_INFO.json next to the library: the git SHA of the sources it was built from (bench.py reports it;
    the GPU box's copy of the repo has no .git).  Git-ignored."""
    import json

    info = {"git_sha": None, "dirty": None, "lib": lib.name}
    try:
        r = subprocess.run(["git", "rev-parse", "HEAD"], cwd=PKG.parent, capture_output=True, text=True, timeout=10)
        if r.returncode == 0:
            info["git_sha"] = r.stdout.strip()
            st = subprocess.run(["git", "status", "--porcelain", "--untracked-files=no"], cwd=PKG.parent,
                                capture_output=True, text=True, timeout=10)
            info["dirty"] = st.stdout.strip() != ""
    except (OSError, subprocess.SubprocessError):
        pass
    (PKG / "BUILD_INFO.json").write_text(json.dumps(info) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    try:
        build(a.force, a.verbose or True, a.defines, a.variant)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        sys.exit(1)
