"""IPG loop with step-size shrinkage, restated from the reference (TEST INFRASTRUCTURE).

Reference: ``coverblip/solver.py``.
* ``step_shrinkage`` follows ``solver.py:116-144``: project ``X - mu G``,
  ``nd = ||dX||^2``; ``nd == 0`` is a fixed point; accept iff
  ``mu <= nd / ||A dX||^2`` (non-strict; zero denominator => ratio inf);
  else ``mu /= zeta`` and raise after ``max_shrink`` shrinks.
* ``solve_core``     follows ``_solve_core`` (``solver.py:155-257``) for the
  exact modes (``tm`` / ``blip_exact``): ``mu0 = n/m`` (``:192-197``),
  ``X0 = 0``, the k == 1 kappa rescale kept only when it does not worsen the
  fidelity (``:220-230``), ``carry_over`` (``:231-232``), the non-finite
  check (``:235-238``), trace records (``:239-246``) and the relative-progress
  stop rule (``:247-252``).  The cover-tree mode is out of scope.
"""

from __future__ import annotations

import numpy as np

from .projection import atoms_of, project_cone_exact


class SolverError(RuntimeError):
    pass


def step_shrinkage(X, G, mu0, project_fn, apply_diff, zeta, max_shrink,
                   fixed=False):
    mu = mu0
    shrinks = 0
    while True:
        proj = project_fn(X - mu * G)
        dX = proj.projected - X
        nd = float(np.linalg.norm(dX) ** 2)
        if nd == 0.0:
            return mu, proj, shrinks, True
        if fixed:
            return mu, proj, shrinks, False
        den = float(np.linalg.norm(apply_diff(dX)) ** 2)
        ratio = np.inf if den == 0.0 else nd / den
        if mu <= ratio:
            return mu, proj, shrinks, False
        mu /= zeta
        shrinks += 1
        if shrinks > max_shrink:
            raise SolverError(
                "step-size collapse: shrinkage exceeded "
                f"{max_shrink} sub-iterations")


def solve_core(Y, A, atoms, basis=None, *, mode="blip_exact", max_iters=50,
               zeta=2.0, rel_tol=1e-6, max_shrink=60, mu_init=None,
               fixed_step=None, step_policy="reset_each_iter", weights=None,
               lookup_table=None, on_iter=None):
    """Exact-mode IPG.  ``basis`` (L, s) selects the compressed variant
    (``solve_compressed``, ``solver.py:269-275``; compress = rows @ V,
    decompress = rows @ V^H, ``dictionary.py:116-122``).

    ``on_iter(k, X_before, G, mu_k, shrinks, proj)`` is a lockstep hook.
    Returns ``(image, indices, gammas, records)``.
    """
    Y = np.asarray(Y, dtype=complex)
    n = A.n
    if basis is None:
        compress = decompress = (lambda X: X)
        dim = atoms.shape[1]
    else:
        compress = (lambda R: R @ basis)
        decompress = (lambda Xc: Xc @ basis.conj().T)
        dim = basis.shape[1]
    w = None if weights is None else np.broadcast_to(weights, Y.shape)

    def project_fn(Z):
        return project_cone_exact(Z, atoms)

    def apply_diff(dX):
        return A.apply(decompress(dX))

    def objective(X):
        R = A.apply(decompress(X)) - Y
        if w is not None:
            return float(np.sum(w * np.abs(R) ** 2))
        return float(np.linalg.norm(R) ** 2)

    def gradient(X):
        R = A.apply(decompress(X)) - Y
        if w is not None:
            R = w * R
        return compress(A.adjoint(R))

    if fixed_step is not None:
        mu_base = fixed_step
    elif mu_init is not None:
        mu_base = mu_init
    else:
        mu_base = n / A.m

    X = np.zeros((n, dim), dtype=complex)
    obj = objective(X)
    records = []
    iters = 1 if mode == "tm" else max_iters
    gammas = np.zeros(n)
    indices = np.zeros(n, dtype=np.int64)
    for k in range(1, iters + 1):
        G = gradient(X)
        mu_k, proj, shrinks, fixed_pt = step_shrinkage(
            X, G, mu_base, project_fn, apply_diff, zeta, max_shrink,
            fixed=fixed_step is not None)
        if on_iter is not None:
            on_iter(k, X, G, mu_k, shrinks, proj)
        if fixed_pt:
            break
        X = proj.projected
        gammas, indices = proj.gammas, proj.indices
        if k == 1 and fixed_step is None:
            e = float(np.linalg.norm(A.apply(decompress(X))))
            if e > 0.0:
                kappa = float(np.linalg.norm(Y)) / e
                if objective(kappa * X) <= objective(X):
                    X = kappa * X
                    gammas = kappa * gammas
                    mu_base *= kappa
        elif step_policy == "carry_over":
            mu_base = mu_k
        new_obj = objective(X)
        if not np.isfinite(new_obj):
            raise SolverError(f"non-finite fidelity at iteration {k}: {new_obj}")
        records.append(dict(iter=k, fidelity=float(np.sqrt(new_obj)),
                            mu=mu_k, shrinks=shrinks, cost=proj.cost))
        if obj > 0.0 and (obj - new_obj) / obj < rel_tol:
            obj = new_obj
            break
        obj = new_obj
        if obj == 0.0:
            break
    return decompress(X), indices, gammas, records


__all__ = ["SolverError", "solve_core", "step_shrinkage", "atoms_of"]
