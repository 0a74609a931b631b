"""Seeded input generators for C1-C5 (host logic, CPU)."""

import numpy as np
import pytest

from paper_2201_05555_b200 import workloads as wl


@pytest.mark.parametrize("name,p,nx,deg", [("C1", 1, 64, 2), ("C2", 32, 128, 3), ("C3", 128, 64, 2),
                                           ("C4", 128, 64, 2), ("C5", 64, 512, 3)])
def test_configs(name, p, nx, deg):
    w = wl.config(name)
    assert w.p == p and w.num_cells == nx and w.degree == deg


def test_generation_deterministic_and_in_domain():
    w = wl.config("C2")
    x1, v1 = wl.generate(w, num_particles=5000, instances=[0, 7, 31])
    x2, v2 = wl.generate(w, num_particles=5000, instances=[0, 7, 31])
    np.testing.assert_array_equal(x1, x2)
    np.testing.assert_array_equal(v1, v2)
    assert x1.shape == (5000, 3)
    assert (x1 >= 0).all() and (x1 < w.lengths[0]).all()
    # two-stream: bimodal at +-v0
    assert abs(np.abs(v1[:, 2]).mean() - w.vparams[31, 0]) < 0.05
    # subsetting instances gives the same columns as the full draw
    xa, _ = wl.generate(w, num_particles=5000)
    np.testing.assert_array_equal(xa[:, [0, 7, 31]], x1)


def test_density_perturbation_visible():
    w = wl.config("C5")
    x, v = wl.generate(w, num_particles=200_000, instances=[3])
    k, a = w.wavenumbers[3], w.alphas[3]
    est = 2 * np.mean(np.cos(k * x[:, 0]))
    assert abs(est - a) < 0.01
    assert abs(np.mean(v[:, 0] > 3.0) - 0.1) < 0.01
