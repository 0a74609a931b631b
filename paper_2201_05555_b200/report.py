"""Run-report serialization -- the reference's output formats (report.py:57-246).

The reference assembles a `RunReport` in its CLI driver (driver.py:277-499,
out of scope here) and writes one directory per run: energies.csv,
errors.csv, ranks.csv, hamiltonian.csv, structure.csv, timings.csv,
config.json, rates.json, summary.json.  This module writes the same files
with the same headers, row order and number formatting (shortest round-trip
repr), so downstream tooling reading a picrom report directory reads these
unchanged.  `report_from_records` fills a RunReport from this package's own
FullOrderRecord / RomRecord; compare-mode error series (diagnostics.py) and
rate fits can be attached to the fields directly.  Figures (matplotlib) are
not rendered.
"""

from __future__ import annotations

import csv
import json
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["RunReport", "report_from_records", "serialize", "build_summary", "parse_summary",
           "load_summary", "write_report"]

RATE_CONVENTION = ("field-amplitude exponential rate: half the log-slope of the "
                   "electric-energy peaks")


@dataclass
class RunReport:
    """The fields serialization reads (diagnostics.py:198-237)."""

    config: dict
    mode: str
    params: np.ndarray
    times: np.ndarray = None
    energy_fom: np.ndarray = None
    energy_rom: np.ndarray = None
    hamiltonian_fom: np.ndarray = None
    hamiltonian_rom: np.ndarray = None
    error_times: np.ndarray = None
    eps_x: np.ndarray = None
    eps_v: np.ndarray = None
    target_x: np.ndarray = None
    target_v: np.ndarray = None
    eps_total: np.ndarray = None
    target_total: np.ndarray = None
    ham_error_times: np.ndarray = None
    ham_rel_error: np.ndarray = None
    dh_total: np.ndarray = None
    dh_coeff: np.ndarray = None
    dh_coeff_dd: np.ndarray = None
    rank_times: np.ndarray = None
    rank_potential: np.ndarray = None
    rank_x: np.ndarray = None
    rank_v: np.ndarray = None
    ortho_residuals: np.ndarray = None
    sympl_residuals: np.ndarray = None
    fp_iterations: np.ndarray = None
    dmd_ranks: np.ndarray = None
    s_conds: np.ndarray = None
    dmd_imag_defect: float = 0.0
    phase_totals: dict = field(default_factory=dict)
    phase_series: dict = field(default_factory=dict)
    fom_step_seconds: np.ndarray = None
    rates: dict = field(default_factory=dict)
    warnings: list = field(default_factory=list)
    notes: dict = field(default_factory=dict)


def report_from_records(config, params, fom=None, rom=None):
    """RunReport of a full ("full"), reduced ("rom") or side-by-side ("compare")
    run from fullorder.FullOrderRecord / driver.RomRecord."""
    mode = "compare" if fom is not None and rom is not None else ("full" if fom is not None else "rom")
    rep = RunReport(config=dict(config or {}), mode=mode,
                    params=None if params is None else np.asarray(params, dtype=float))
    if fom is not None:
        rep.times = np.asarray(fom.energy_times)
        rep.energy_fom = np.asarray(fom.electric_energy)
        rep.hamiltonian_fom = np.asarray(fom.hamiltonian)
        rep.fom_step_seconds = np.asarray(fom.step_seconds)
        rep.phase_totals.update(fom.phase_seconds or {})
    if rom is not None:
        if rep.times is None:
            rep.times = np.asarray(rom.energy_times)
        rep.energy_rom = np.asarray(rom.electric_energy)
        rep.hamiltonian_rom = np.asarray(rom.hamiltonian)
        for name in ("ortho_residuals", "sympl_residuals", "fp_iterations", "dmd_ranks", "s_conds",
                     "dh_total", "dh_coeff", "dh_coeff_dd"):
            setattr(rep, name, np.asarray(getattr(rom, name)))
        rep.ham_error_times = np.asarray(rom.decomp_times)
        rep.dmd_imag_defect = float(rom.dmd_imag_defect)
        rep.notes.update(rom.notes or {})
        if rom.timers is not None:
            rep.phase_totals.update(rom.timers.totals)
            rep.phase_series.update({k: np.asarray(v) for k, v in rom.timers.series.items()})
    if fom is not None and rom is not None:
        h_ref, h_rom = np.atleast_2d(rep.hamiltonian_fom), np.atleast_2d(rep.hamiltonian_rom)
        if h_ref.shape == h_rom.shape:
            rep.ham_rel_error = (np.linalg.norm(h_ref - h_rom, axis=1)
                                 / np.linalg.norm(h_ref, axis=1))
    return rep


# ------------------------------------------------------------- formatting

def _cell(v):
    """CSV cell text: shortest round-trip repr for floats, '' for None."""
    if v is None:
        return ""
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    return str(v)


def _csv(path, header, rows):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows([[_cell(v) for v in r] for r in rows])


def _plain(v):
    """JSON-safe copy (numpy scalars/arrays to Python)."""
    if isinstance(v, dict):
        return {str(k): _plain(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_plain(x) for x in v]
    if isinstance(v, np.ndarray):
        return _plain(v.tolist())
    if isinstance(v, np.bool_):
        return bool(v)
    if isinstance(v, np.integer):
        return int(v)
    if isinstance(v, np.floating):
        return float(v)
    return v


def _p(rep):
    return 0 if rep.params is None else int(np.asarray(rep.params).shape[0])


# ----------------------------------------------------------------- tables

def _energies(rep):
    p = _p(rep)
    series = []
    if rep.mode in ("full", "compare"):
        series.append(("fom", rep.energy_fom))
    if rep.mode in ("rom", "compare"):
        series.append(("rom", rep.energy_rom))
    header = ["time"] + [f"{tag}_{j}" for tag, _ in series for j in range(p)]
    if rep.times is None or not series or any(s is None for _, s in series):
        return header, []
    arrs = [np.asarray(s) for _, s in series]
    return header, [[t] + [x for a in arrs for x in a[k]] for k, t in enumerate(np.asarray(rep.times))]


def _errors(rep):
    names = ("eps_x", "eps_v", "target_x", "target_v", "eps_total", "target_total")
    header = ["time"] + list(names)
    cols = [getattr(rep, k) for k in names]
    if rep.error_times is None or any(c is None for c in cols):
        return header, []
    cols = [np.asarray(c) for c in cols]
    return header, [[t] + [float(c[k]) for c in cols] for k, t in enumerate(np.asarray(rep.error_times))]


def _ranks(rep):
    rows = []
    if rep.rank_times is not None and rep.rank_potential is not None:
        rows += [[t, "potential", int(r)] for t, r in zip(np.asarray(rep.rank_times),
                                                         np.asarray(rep.rank_potential))]
    st = (rep.notes or {}).get("state_rank_times")
    if rep.rank_x is not None and st is not None:
        rows += [[t, "state_complex", int(r)] for t, r in zip(st, np.asarray(rep.rank_x))]
    return ["time", "series", "rank"], rows


def _hamiltonian(rep):
    rows = []
    if rep.times is not None and rep.ham_rel_error is not None:
        rows += [[t, "rel_error", v] for t, v in zip(np.asarray(rep.times),
                                                    np.asarray(rep.ham_rel_error))]
    if rep.ham_error_times is not None:
        for name in ("dh_total", "dh_coeff", "dh_coeff_dd"):
            data = getattr(rep, name)
            if data is not None:
                rows += [[t, name, v] for t, v in zip(np.asarray(rep.ham_error_times),
                                                     np.asarray(data))]
    return ["time", "series", "value"], rows


def _structure(rep):
    header = ["step", "time", "ortho_residual", "sympl_residual", "fp_iterations", "dmd_rank",
              "s_cond"]
    if rep.ortho_residuals is None:
        return header, []
    ortho, sympl = np.asarray(rep.ortho_residuals), np.asarray(rep.sympl_residuals)
    dt = float((rep.config or {}).get("dt", 1.0))

    def per_step(arr, tau):
        return None if tau == 0 or arr is None else arr[tau - 1]

    return header, [[tau, tau * dt, ortho[tau], sympl[tau], per_step(rep.fp_iterations, tau),
                     per_step(rep.dmd_ranks, tau), per_step(rep.s_conds, tau)]
                    for tau in range(ortho.shape[0])]


def _timings(rep):
    rows = []
    series = rep.phase_series or {}
    for ph in sorted(rep.phase_totals or {}):
        data = series.get(ph)
        if data is not None and len(data):
            a = np.asarray(data, dtype=float)
            rows.append([ph, rep.phase_totals[ph], a.size, float(np.median(a))])
        else:
            rows.append([ph, rep.phase_totals[ph], 0, None])
    return ["phase", "total_seconds", "num_intervals", "per_interval_median_seconds"], rows


# ---------------------------------------------------------------- outputs

def build_summary(rep):
    """Acceptance scalars plus the verbatim config echo (report.py:157-190)."""
    out = {"config": _plain(rep.config), "mode": rep.mode, "num_params": _p(rep),
           "params": _plain(rep.params) if rep.params is not None else [],
           "warnings": _plain(rep.warnings or []), "notes": _plain(rep.notes or {}),
           "rates": _plain(rep.rates or {}), "phase_totals": _plain(rep.phase_totals or {}),
           "dmd_imag_defect": float(rep.dmd_imag_defect)}
    if rep.ortho_residuals is not None:
        out["max_ortho_residual"] = float(np.max(rep.ortho_residuals))
        out["max_sympl_residual"] = float(np.max(rep.sympl_residuals))
    if rep.fp_iterations is not None and np.size(rep.fp_iterations):
        out["max_fp_iterations"] = int(np.max(rep.fp_iterations))
    if rep.ham_rel_error is not None and np.size(rep.ham_rel_error):
        out["max_hamiltonian_rel_error"] = float(np.max(rep.ham_rel_error))
    if rep.eps_total is not None and np.size(rep.eps_total):
        out["final_eps_total"] = _plain(np.asarray(rep.eps_total)[-1])
        out["final_target_total"] = _plain(np.asarray(rep.target_total)[-1])
    if rep.rank_potential is not None and np.size(rep.rank_potential):
        out["max_potential_rank"] = int(np.max(rep.rank_potential))
    med = {k: float(np.median(np.asarray(v, dtype=float)))
           for k, v in (rep.phase_series or {}).items() if v is not None and len(v)}
    if med:
        out["phase_medians"] = med
    return out


def parse_summary(path):
    with open(path) as fh:
        return json.load(fh)


load_summary = parse_summary


def serialize(rep, outdir):
    """Write the delimited and JSON outputs of one run; returns {name: path}."""
    os.makedirs(outdir, exist_ok=True)
    paths = {}
    tables = (("energies.csv", _energies), ("errors.csv", _errors), ("ranks.csv", _ranks),
              ("hamiltonian.csv", _hamiltonian), ("structure.csv", _structure),
              ("timings.csv", _timings))
    try:
        for name, make in tables:
            paths[name] = os.path.join(outdir, name)
            _csv(paths[name], *make(rep))
        docs = {"config.json": _plain(rep.config),
                "rates.json": {"convention": RATE_CONVENTION, "rates": _plain(rep.rates or {})},
                "summary.json": build_summary(rep)}
        for name, doc in docs.items():
            paths[name] = os.path.join(outdir, name)
            with open(paths[name], "w") as fh:
                json.dump(doc, fh, indent=2)
    except OSError as err:
        raise OSError(f"failed writing report files under {outdir}: {err}") from err
    return paths


def write_report(rep, outdir, figures=False):
    """serialize(); figures are not rendered (no matplotlib in this build)."""
    return serialize(rep, outdir)
