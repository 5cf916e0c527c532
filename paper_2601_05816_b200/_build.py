"""Build libb200wd.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box.  ``python -m paper_2601_05816_b200._build``.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libb200wd.so"
SOURCES = ["capi.cu", "layout.cu", "dirac.cu", "dirac_c128.cu", "dirac_c64.cu", "blas.cu"] + [
    f"dirac_{d}_{g}.cu" for d in ("c128", "c64") for g in ("b0", "b4", "b8", "b16", "b24")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "b200wd.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: Path | None = None,
          only: tuple = ()) -> Path:
    """only: (variant builds) translation units compiled with `defines`; the
    others are taken from the default build's objects."""
    lib = Path(out) if out else LIB
    if not force and out is None and not needs_build():
        return LIB
    objs = []
    tmp = PKG / "build" / ("_".join(defines) or "default")
    tmp.mkdir(parents=True, exist_ok=True)
    logs = []
    procs = []
    for src in SOURCES:  # translation units compile in parallel
        obj = tmp / (Path(src).stem + ".o")
        if only and Path(src).stem not in only:
            objs.append(str(PKG / "build" / "default" / (Path(src).stem + ".o")))
            continue
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", str(ROOT / "include"), "-I", str(CSRC),
               "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(str(obj))
    for src, pr in procs:
        _, err = pr.communicate()
        logs.append(err)
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{err}")
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
           *objs, "-o", str(lib) + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(str(lib) + ".tmp", lib)
    (tmp / "ptxas.log").write_text("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    only = tuple(x for a in sys.argv[1:] if a.startswith("--only=") for x in a.split("=", 1)[1].split(","))
    print(build(force="--force" in sys.argv, verbose="--quiet" not in sys.argv, defines=defs,
                out=Path(outs[0]) if outs else None, only=only))
