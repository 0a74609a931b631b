"""Report output formats (report.py:57-246): the files this package writes are
byte-identical to the reference's serialize() on the same RunReport fields
(the reference is imported from /root/reference where it exists -- this
container; the GPU box has no /root/reference and skips)."""

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2201_05555_b200 import report

REF = Path("/root/reference/pkg/src")
FILES = ("energies.csv", "errors.csv", "ranks.csv", "hamiltonian.csv", "structure.csv",
         "timings.csv", "config.json", "rates.json", "summary.json")


def _fields(rng, mode):
    p, te, steps = 3, 6, 10
    f = dict(config={"dt": 0.05, "benchmark": "landau", "num_params": p}, mode=mode,
             params=rng.uniform(size=(p, 2)), times=np.linspace(0, 0.5, te),
             energy_fom=rng.uniform(size=(te, p)), energy_rom=rng.uniform(size=(te, p)),
             error_times=np.linspace(0, 0.5, 3), eps_x=rng.uniform(size=3),
             eps_v=rng.uniform(size=3), target_x=rng.uniform(size=3), target_v=rng.uniform(size=3),
             eps_total=rng.uniform(size=3), target_total=rng.uniform(size=3),
             ham_error_times=np.array([0.25, 0.5]), ham_rel_error=rng.uniform(size=te),
             dh_total=rng.uniform(size=2), dh_coeff=rng.uniform(size=2),
             dh_coeff_dd=rng.uniform(size=2), rank_times=np.array([0.0, 0.25]),
             rank_potential=np.array([3, 4]), ortho_residuals=rng.uniform(size=steps + 1) * 1e-15,
             sympl_residuals=rng.uniform(size=steps + 1) * 1e-15,
             fp_iterations=rng.integers(5, 9, steps), dmd_ranks=rng.integers(0, 5, steps),
             s_conds=rng.uniform(1, 10, steps), dmd_imag_defect=1e-4,
             phase_totals={"rom_basis": 1.5, "rom_coeff": 2.5, "fom_step": 0.25},
             phase_series={"rom_basis": rng.uniform(size=steps), "rom_coeff": rng.uniform(size=steps)},
             rates={"fom": -0.15}, warnings=["w"], notes={"state_rank_times": [0.0]})
    f["rank_x"] = np.array([5])
    return f


@pytest.mark.parametrize("mode", ["full", "rom", "compare"])
def test_serialize_matches_reference(tmp_path, mode):
    if not (REF / "picrom").exists():
        pytest.skip("reference package not present")
    sys.path.insert(0, str(REF))
    try:
        from picrom import diagnostics as rdiag
        from picrom import report as rrep
    finally:
        sys.path.remove(str(REF))
    f = _fields(np.random.default_rng(3), mode)
    ours = report.serialize(report.RunReport(**f), tmp_path / "ours")
    theirs = rrep.serialize(rdiag.RunReport(**f), tmp_path / "ref")
    assert set(ours) == set(theirs) == set(FILES)
    for name in FILES:
        assert Path(ours[name]).read_bytes() == Path(theirs[name]).read_bytes(), name


def test_empty_report_still_writes_headers(tmp_path):
    paths = report.serialize(report.RunReport(config={}, mode="rom", params=None), tmp_path)
    for name in FILES[:6]:
        lines = Path(paths[name]).read_text().splitlines()
        assert len(lines) == 1 and lines[0]
    assert report.parse_summary(paths["summary.json"])["mode"] == "rom"


def test_report_from_records_layout(tmp_path):
    """A compare-mode report built from (duck-typed) FOM and ROM records writes
    the per-step structure table and the energy / Hamiltonian tables."""
    from types import SimpleNamespace
    from paper_2201_05555_b200.diagnostics import PhaseTimers
    rng = np.random.default_rng(5)
    steps, te, p = 4, 3, 2
    t = PhaseTimers()
    for _ in range(steps):
        with t.phase("rom_basis"):
            pass
        t.flush_step()
    fom = SimpleNamespace(energy_times=np.array([0.0, 0.1, 0.2]), electric_energy=rng.uniform(size=(te, p)),
                          hamiltonian=rng.uniform(1, 2, size=(te, p)), step_seconds=np.full(steps, 1e-3),
                          phase_seconds={"fom_step": 4e-3})
    rom = SimpleNamespace(energy_times=fom.energy_times, electric_energy=rng.uniform(size=(te, p)),
                          hamiltonian=fom.hamiltonian * (1 + 1e-6), ortho_residuals=np.zeros(steps + 1),
                          sympl_residuals=np.zeros(steps + 1), fp_iterations=np.full(steps, 7),
                          dmd_ranks=np.zeros(steps, int), s_conds=np.ones(steps),
                          dh_total=np.array([1e-9]), dh_coeff=np.array([2e-9]), dh_coeff_dd=np.array([3e-9]),
                          decomp_times=np.array([0.2]), dmd_imag_defect=0.0, notes={}, timers=t)
    rep = report.report_from_records({"dt": 0.05}, rng.uniform(size=(p, 2)), fom=fom, rom=rom)
    assert rep.mode == "compare"
    np.testing.assert_allclose(rep.ham_rel_error, 1e-6, rtol=1e-6)
    paths = report.serialize(rep, tmp_path)
    assert Path(paths["energies.csv"]).read_text().splitlines()[0] == "time,fom_0,fom_1,rom_0,rom_1"
    assert len(Path(paths["structure.csv"]).read_text().splitlines()) == steps + 2
    ham = Path(paths["hamiltonian.csv"]).read_text().splitlines()
    assert ham[0] == "time,series,value" and len(ham) == 1 + te + 3
