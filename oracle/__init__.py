"""CPU oracle for the exact-projection IPG hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference (CoverBLIP,
``/root/reference/pkg/src/coverblip``) for the rows of SURVEY.md section 8:

* ``oracle.projection``  -- ``project_cone_exact`` / ``_gammas_for``
  (reference ``projection.py:38-67``) plus the top-2 near-tie classifier
  (SURVEY 8c restatement 1).
* ``oracle.operator``    -- Cartesian ``ForwardOperator.apply/adjoint``
  (reference ``forward_model.py:123-167``), ``make_epi_pattern``
  (``forward_model.py:170-187``) and the 3-D variant (SURVEY 8c restatement 2).
* ``oracle.solver``      -- ``step_shrinkage`` and ``_solve_core``
  (reference ``solver.py:116-257``).

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the real
reference in the build container and freezes its outputs to
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
restatement against those vectors (CPU, ``-m "not gpu"``).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only
as the checker or the timed CPU baseline.  The product package
``paper_1810_01967_b200`` never imports it: the CUDA path fails loudly when
its extension is missing instead of falling back here.
"""
