"""ctypes binding of the C-ABI library (include/picrom_b200.h).

There is no CPU fallback: importing the compute path without the built
library, or calling it without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from ._build import LIB_PATH
from .errors import ConfigurationError

HEADER = Path(__file__).resolve().parent.parent / "include" / "picrom_b200.h"

_vp, _i, _ll, _d, _sz = C.c_void_p, C.c_int, C.c_longlong, C.c_double, C.c_size_t

# name -> (restype, argtypes); must match include/picrom_b200.h exactly
SIGNATURES = {
    "picrom_version": (_i, []),
    "picrom_last_error": (C.c_char_p, []),
    "picrom_device_info": (_i, [_vp, _vp, _vp]),
    "picrom_fom_workspace_bytes": (_sz, [_ll, _i, _i, _i]),
    "picrom_locate": (_i, [_vp, _ll, _i, _ll, _vp, _i, _vp, _vp, _ll, _vp, _vp]),
    "picrom_basis_table": (_i, [_vp, _ll, _i, _ll, _vp, _i, _i, _i, _vp, _vp, _ll, _vp, _vp]),
    "picrom_deposit": (_i, [_vp, _ll, _i, _ll, _vp, _i, _i, _vp, _vp, _vp, _vp]),
    "picrom_rmatvec": (_i, [_vp, _vp, _ll, _i, _ll, _vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "picrom_poisson": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "picrom_field_energy": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "picrom_gather": (_i, [_vp, _ll, _i, _ll, _vp, _i, _i, _vp, _i, _vp, _ll, _vp, _vp]),
    "picrom_pic_step": (_i, [_vp, _vp, _ll, _i, _ll, _vp, _i, _i, _vp, _vp, _vp,
                             _d, _d, _d, _ll, _vp, _ll, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                             _vp]),
    "picrom_timestamp": (_i, [_vp, _vp]),
    "picrom_pic_push": (_i, [_vp, _vp, _ll, _i, _ll, _vp, _i, _i, _vp, _d, _d, _d, _ll, _vp,
                             _vp, _vp, _vp]),
    "picrom_pic_solve": (_i, [_ll, _i, _i, _i, _vp, _vp, _vp, _vp, _ll, _vp, _ll, _vp, _vp, _vp,
                              _vp, _vp, _vp]),
    "picrom_verlet_drift": (_i, [_vp, _vp, _vp, _ll, _i, _ll, _vp, _i, _i, _vp, _vp,
                                 _d, _ll, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "picrom_verlet_kick": (_i, [_vp, _vp, _vp, _ll, _i, _ll, _vp, _i, _i, _vp, _d, _vp, _vp, _vp]),
    "picrom_half_sumsq": (_i, [_vp, _ll, _i, _ll, _vp, _vp, _vp]),
    "picrom_transpose": (_i, [_vp, _ll, _ll, _vp, _vp]),
    "picrom_rom_workspace_bytes": (_sz, [_ll, _i, _i, _i]),
    "picrom_rom_field": (_i, [_vp, _ll, _i, _vp, _i, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp, _vp]),
    "picrom_rom_gather": (_i, [_vp, _ll, _i, _vp, _i, _i, _vp, _vp, _i, _i, _vp, _i, _vp, _i,
                               _vp, _vp, _ll, _vp, _vp, _vp, _vp]),
    "picrom_rom_gather_uv": (_i, [_vp, _ll, _i, _vp, _i, _i, _vp, _vp, _i, _i, _vp, _i, _vp, _vp,
                                  _i, _vp, _vp, _ll, _vp, _vp, _vp]),
    "picrom_paired_gram": (_i, [_i, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp]),
    "picrom_gram_tasks": (_i, [_i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _ll, _vp, _vp, _vp]),
    "picrom_cross_gram": (_i, [_i, _i, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp]),
    "picrom_tall_atb_workspace_bytes": (_sz, [_ll, _i, _i]),
    "picrom_tall_atb": (_i, [_vp, _i, _i, _vp, _i, _i, _ll, _vp, _vp, _vp]),
    "picrom_small_cholinv": (_i, [_vp, _i, _vp, _vp, _vp]),
    "picrom_small_rmul": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp]),
    "picrom_argmax_abs": (_i, [_vp, _ll, _ll, _vp, _i, _vp, _vp, _vp, _vp]),
    "picrom_deim_workspace_bytes": (_sz, [_ll, _i]),
    "picrom_diff_sumsq": (_i, [_vp, _vp, _ll, _vp, _vp, _vp]),
    "picrom_deim_greedy": (_i, [_vp, _i, _ll, _i, _vp, _vp, _vp, _vp, _vp]),
    "picrom_combine": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _ll, _vp, _i, _i, _i, _vp]),
    "picrom_dmd_extrapolate": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "picrom_deim_gather": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp, _i,
                                _vp, _vp, _vp]),
    "picrom_fp_update": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _d, _d, _i, _vp, _vp, _vp]),
    "picrom_rows_gather": (_i, [_vp, _i, _vp, _i, _i, _vp, _vp]),
    "picrom_transpose_i64": (_i, [_vp, _ll, _ll, _vp, _vp]),
}

_lib = None


def header_symbols():
    """Function names declared in include/picrom_b200.h."""
    return sorted(header_arity())


def header_arity():
    """{name: number of parameters} parsed from the header's declarations."""
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*(?:int|size_t|const char\*)\s+(picrom_\w+)\s*\(([^)]*)\)\s*;",
                         text, re.M):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def load():
    """Load (not build) the library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2201_05555_b200._build` "
            "(there is no CPU fallback for the hot path)")
    import os
    lib = C.CDLL(os.environ.get("PICROM_LIB", str(LIB_PATH)))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name, *args):
    """Invoke a C-ABI entry point; nonzero status -> exception with the library message."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.picrom_last_error().decode(errors="replace")
        if rc == 1:
            raise ConfigurationError(f"{name}: {msg}")
        raise RuntimeError(f"{name} failed ({rc}): {msg}")
    return rc


def query(name, *args):
    return getattr(load(), name)(*args)
