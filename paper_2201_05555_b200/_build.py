"""In-tree build of the sm_100a C-ABI library (nvcc, no torch extension machinery).

The library is a plain shared object exporting the `extern "C"` entry points of
include/picrom_b200.h; it links the CUDA runtime statically so it has no
dependency on torch's own libcudart.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_NAME = "libpicrom_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale():
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG_DIR.parent / "include" / "picrom_b200.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force=False, verbose=False):
    """Compile csrc/*.cu into LIB_PATH (skipped when up to date)."""
    if not force and not _stale():
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not Path(nvcc).exists():
        nvcc = "nvcc"
    tmp = LIB_PATH.with_suffix(".so.tmp")
    # one nvcc per translation unit, in parallel, then a host link
    objs, procs = [], []
    for src in sources():
        obj = PKG_DIR / f"build_{src.stem}.o"
        cmd = [nvcc, *NVCC_FLAGS, "-c", "-o", str(obj), str(src)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
        objs.append(obj)
    log = []
    for cmd, pr in procs:
        out, err = pr.communicate()
        log.append(err)
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed ({pr.returncode}): {' '.join(cmd)}")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
           *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc link failed ({res.returncode}): {' '.join(cmd)}")
    for o in objs:
        o.unlink(missing_ok=True)
    if verbose:
        sys.stderr.write("".join(log))
    (PKG_DIR / "build_ptxas.log").write_text("".join(log))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB_PATH)
