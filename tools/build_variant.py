"""Build a variant of the library with extra nvcc defines (dev tool):
    python tools/build_variant.py NAME [--only=fom] -DPICROM_FIX_U=2 ...
Output: paper_2201_05555_b200/variants/libpicrom_NAME.so (select with PICROM_LIB=...).
--only=STEM compiles only csrc/STEM.cu with the defines; the other translation
units come from a cache of default-flag objects (rebuilt when their source changes)."""
import hashlib
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import _build  # noqa: E402

args = sys.argv[1:]
name = args[0]
only = [a.split("=", 1)[1] for a in args[1:] if a.startswith("--only=")]
defs = [a for a in args[1:] if not a.startswith("--")]
out = _build.PKG_DIR / "variants"
out.mkdir(exist_ok=True)
cache = out / "cache"
cache.mkdir(exist_ok=True)
deps = b"".join(p.read_bytes() for p in sorted(_build.CSRC.glob("*.cuh")))
deps += (_build.PKG_DIR.parent / "include" / "picrom_b200.h").read_bytes()
objs, procs = [], []
for src in _build.sources():
    if only and src.stem not in only:
        key = hashlib.sha1(src.read_bytes() + deps + " ".join(_build.NVCC_FLAGS).encode()).hexdigest()[:16]
        obj = cache / f"{src.stem}_{key}.o"
        objs.append(obj)
        if obj.exists():
            continue
        cmd = ["nvcc", *_build.NVCC_FLAGS, "-c", "-o", str(obj), str(src)]
    else:
        obj = out / f"{name}_{src.stem}.o"
        objs.append(obj)
        cmd = ["nvcc", *_build.NVCC_FLAGS, *defs, "-c", "-o", str(obj), str(src)]
    procs.append(subprocess.Popen(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.PIPE, text=True))
for pr in procs:
    _, err = pr.communicate()
    if pr.returncode:
        sys.exit(err)
    with (out / f"{name}.ptxas.log").open("a") as f:
        f.write(err)
lib = out / f"libpicrom_{name}.so"
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib),
                       *map(str, objs)])
for o in out.glob(f"{name}_*.o"):
    o.unlink()
print(lib)
