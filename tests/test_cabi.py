"""The C-ABI library builds, loads, and exports every symbol the header declares.

No compute calls (no GPU in the build container)."""

import ctypes
import subprocess

from paper_2201_05555_b200 import _lib


def test_header_and_bindings_agree():
    declared = set(_lib.header_symbols())
    assert declared, "no picrom_* declarations parsed from include/picrom_b200.h"
    assert declared == set(_lib.SIGNATURES), (declared ^ set(_lib.SIGNATURES))


def test_binding_arity_matches_header():
    arity = _lib.header_arity()
    for name, (_, args) in _lib.SIGNATURES.items():
        assert len(args) == arity[name], (name, len(args), arity[name])


def test_library_exports_every_declared_symbol(lib_built):
    for name in _lib.header_symbols():
        assert hasattr(lib_built, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = set(_lib.header_symbols()) - exported
    assert not missing, missing


def test_host_only_queries(lib_built):
    assert lib_built.picrom_version() >= 1
    nbytes = lib_built.picrom_fom_workspace_bytes(1000, 4, 64, 3)
    assert nbytes > 0


def test_sm100a_code_in_library(lib_built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    import pytest
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "nope.so")
    with pytest.raises(ImportError):
        _lib.load()
