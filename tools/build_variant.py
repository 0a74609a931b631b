"""Build a variant of the library with extra nvcc defines (dev tool):
    python tools/build_variant.py NAME -DPICROM_STEP_U=8 ...
Output: paper_2201_05555_b200/variants/libpicrom_NAME.so (select with PICROM_LIB=...)."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_05555_b200 import _build  # noqa: E402

name, defs = sys.argv[1], [a for a in sys.argv[2:] if not a.startswith("--swap=")]
# --swap=STEM=PATH compiles PATH (copied next to csrc/STEM.cu) instead of csrc/STEM.cu
swaps = dict(a[len("--swap="):].split("=", 1) for a in sys.argv[2:] if a.startswith("--swap="))
out = _build.PKG_DIR / "variants"
out.mkdir(exist_ok=True)
objs, procs = [], []
for src in _build.sources():
    obj = out / f"{name}_{src.stem}.o"
    if src.stem in swaps:
        tmp = src.with_name(f"_swap_{name}_{src.stem}.cuv")
        tmp.write_text(Path(swaps[src.stem]).read_text())
        src = tmp
    cmd = ["nvcc", *_build.NVCC_FLAGS, *defs, "-x", "cu", "-c", "-o", str(obj), str(src)]
    procs.append(subprocess.Popen(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.PIPE, text=True))
    objs.append(obj)
for pr in procs:
    _, err = pr.communicate()
    if pr.returncode:
        sys.exit(err)
lib = out / f"libpicrom_{name}.so"
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib), *map(str, objs)])
for o in objs:
    o.unlink()
for t in _build.CSRC.glob(f"_swap_{name}_*.cuv"):
    t.unlink()
print(lib)
