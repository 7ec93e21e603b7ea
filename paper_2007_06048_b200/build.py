"""In-tree build of libminimod_b200.so (the C-ABI CUDA library) for sm_100a.

    python -m paper_2007_06048_b200.build [--force]

Compiles every source under csrc/ with nvcc (-gencode arch=compute_100a,
code=sm_100a -lineinfo) into build/ and links
paper_2007_06048_b200/libminimod_b200.so.  Host code is compiled with
-ffp-contract=off so the setup numerics stay bit-identical to the reference.
nvcc cross-compiles without a GPU, so this runs in the CPU container too.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "minimod_b200"
LIB = PKG / "libminimod_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
          "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
# per-file extra flags
EXTRA = {
    # strict kernels: reference operation order, never contract to FMA
    "kernels_strict.cu": ["-fmad=false"],
    "vd_engine.cu": ["-fmad=false"],
    "kernels_fast.cu": ["-Xptxas", "-v"] if os.environ.get("MM_PTXAS_VERBOSE") else [],
}


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: cannot build the CUDA library")
    return cand


def _sources():
    return sorted([p for p in CSRC.iterdir() if p.suffix in (".cu", ".cpp")])


def _headers_mtime() -> float:
    hs = (list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) +
          list((ROOT / "include").glob("*.h")))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, force: bool, bdir: Path = BUILD, defines=()) -> Path:
    obj = bdir / (src.name + ".o")
    if (not force and obj.exists() and obj.stat().st_mtime >= src.stat().st_mtime
            and obj.stat().st_mtime >= _headers_mtime()):
        return obj
    cmd = [nvcc(), *ARCH, *COMMON, *EXTRA.get(src.name, []), *[f"-D{d}" for d in defines],
           "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if res.stderr.strip() and os.environ.get("MM_BUILD_VERBOSE"):
        print(res.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> Path:
    """Build the library.  `variant` + `defines` build an experiment copy
    (libminimod_b200_<variant>.so, loaded when MM_LIB_VARIANT=<variant>)."""
    bdir = BUILD.with_name(BUILD.name + (f"_{variant}" if variant else ""))
    lib = LIB.with_name(f"libminimod_b200_{variant}.so") if variant else LIB
    bdir.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, bdir, defines), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not lib.exists() or lib.stat().st_mtime < newest:
        tmp = lib.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}")
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    build(force=a.force, verbose=True, variant=a.variant, defines=a.defines)
