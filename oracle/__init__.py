"""CPU oracle for the picrom hot path -- TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and the CPU-baseline leg of ``bench.py`` may import
it. The product package (``paper_2201_05555_b200``) never imports it and fails
loudly when its CUDA library is missing.

It restates, in plain numpy/scipy, the algorithm of the reference package
``picrom`` (``/root/reference/pkg/src/picrom``), generalised from P1 hat
functions to cardinal B-splines of degree 1..3 (BASELINE configs C1-C5 ask for
quadratic/cubic splines, which the reference does not have):

* ``fe_bspline``   -- fem.py (locate, basis tables, deposit, Poisson, energy, field)
* ``pic_loop``     -- fullorder.py (VlasovSystem, VerletStepper, run_full_order)
* ``manifold``     -- reduction.py (J products, cSVD, S matrix, velocity, Cayley
                      retraction, tangent transport, fixed point, PRK2 step)
* ``dmd_deim``     -- hyper.py (DMD, RBF, DEIM greedy/fit, hyper stage)
* ``rom_loop``     -- driver.py (exact_gradients, full stage, run_reduced)

Pinning: at degree 1 with one mesh, every function is checked against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``,
fixtures in ``tests/golden/*.npz``). Degree 2/3 values are pinned only by the
reference's own property tests ported to degree p (partition of unity, adjoint
vs dense, zero-mean solve vs pinv, translation equivariance, two-path
Hamiltonian, force = -grad energy) -- "parity pinned at degree 1, property-
pinned at degree 2/3".
"""
