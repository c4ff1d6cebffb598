"""Build liblinkcert_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

Usage: python -m paper_2106_12655_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "liblinkcert_b200.so"
SOURCES = ["abi.cu", "pipeline.cu", "gauss.cu", "pls.cu", "discretize.cu", "bh.cu", "probe.cu", "comm.cu", "digest.cpp"]
# bh.cu reproduces the reference numba arithmetic (no FMA contraction) operation by operation
EXTRA_FLAGS = {"bh.cu": ["-fmad=false"]}
HEADERS = ["common.cuh", "gauss.cuh", "pipeline.cuh", "pls.cuh", "discretize.cuh", "geom.cuh", "scan.cuh", "bh.cuh",
           "comm.cuh", "pass1.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]

CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O3", "-std=c++17", "-g", "-fPIC", "-fvisibility=hidden", "-pthread"]


def _fmt_include() -> str:
    """Header-only fmt (Dragonbox shortest float digits) vendored with PyTorch."""
    import importlib.util

    spec = importlib.util.find_spec("torch")
    for loc in (spec.submodule_search_locations or []) if spec else []:
        inc = Path(loc) / "include"
        if (inc / "fmt" / "format.h").exists():
            return str(inc)
    raise RuntimeError("fmt headers not found (expected under torch/include/fmt)")


def _sources():
    return [CSRC / s for s in SOURCES if (CSRC / s).exists()]


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = _sources() + [CSRC / h for h in HEADERS if (CSRC / h).exists()]
    deps.append(ROOT / "include" / "linkcert_b200.h")
    deps.append(Path(__file__))
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> Path:
    """variant/defines: an A/B build (e.g. -DLC_ROWS=3) into _build_<variant>/, leaving the product .so alone."""
    lib = PKG / f"_build_{variant}" / "liblinkcert_b200.so" if variant else LIB
    if not variant and not force and not _stale():
        return LIB
    objs = []
    build_dir = PKG / (f"_build_{variant}" if variant else "_build")
    build_dir.mkdir(exist_ok=True)
    procs = []
    for src in _sources():
        obj = build_dir / (src.stem + ".o")
        if src.suffix == ".cpp":     # host-only code: the host compiler directly
            cmd = [CXX, *CXX_FLAGS, "-I", _fmt_include(), "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        else:
            # LC_NVCC_EXTRA: extra nvcc flags for A/B variant builds only (e.g. "-Xptxas -regUsageLevel=8")
            extra = os.environ.get("LC_NVCC_EXTRA", "").split() if variant else []
            cmd = [NVCC, *NVCC_FLAGS, *EXTRA_FLAGS.get(src.name, []), *extra, *[f"-D{d}" for d in defines], "-I",
                   str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode(errors="replace")))
        elif verbose and out:
            print(out.decode(errors="replace"), file=sys.stderr)
    if failed:
        msg = "\n".join(f"--- {s.name}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           *map(str, objs), "-ldl", "-o", str(tmp)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else ""
    defs = [args[k + 1] for k, a in enumerate(args) if a == "-D"]
    print(build(force="--force" in args, verbose="-v" in args, variant=var, defines=defs))
