"""Darcy consumer on the GPU vs the reference's own solutions
(tests/golden/darcy.npz, made by running fieldfit.darcy.solve_darcy)."""

import numpy as np
import pytest

import paper_2605_16564_b200 as pam
from paper_2605_16564_b200 import darcy as D
from _darcy_cases import problems

pytestmark = pytest.mark.gpu


def _check(name, sol, g, tol):
    ref = g[f"{name}_values"]
    fin = np.isfinite(ref)
    np.testing.assert_array_equal(np.isfinite(sol.values), fin)  # hole nodes are NaN in both
    scale = np.abs(ref[fin]).max()
    assert np.max(np.abs(sol.values[fin] - ref[fin])) <= tol * scale, name
    A, b = sol.system
    np.testing.assert_array_equal(A.indptr, g[f"{name}_A_indptr"])
    np.testing.assert_array_equal(A.indices, g[f"{name}_A_indices"])
    np.testing.assert_allclose(A.data, g[f"{name}_A_data"], rtol=1e-14, atol=1e-14 * np.abs(A.data).max())
    np.testing.assert_array_equal(b, g[f"{name}_b"])
    assert sol.diagnostics["residual"] < 1e-9


@pytest.mark.parametrize("name", ["d1", "d3"])
def test_darcy_small_systems_match_direct_solve(cuda, golden, name):
    g = golden("darcy")
    sol = D.solve_darcy(problems()[name])
    _check(name, sol, g, 1e-9)  # reference: sparse LU; here PCG to 1e-14
    assert sol.diagnostics["method"] == "cg"


def test_darcy_cg_path_with_holes_neumann_source(cuda, golden):
    g = golden("darcy")
    sol = D.solve_darcy(problems()["d2"])
    _check("d2", sol, g, 1e-7)  # both sides stop at ||r|| < 1e-10 ||b||
    assert abs(sol.diagnostics["iterations"] - int(g["d2_iterations"])) <= 5
    ref_react = float(g["d2_reaction_left"])
    assert abs(sol.boundary_reaction("left") - ref_react) <= 1e-6 * abs(ref_react)


def test_darcy_with_surrogate_coefficient(cuda, golden):
    """The reference's fitted surrogate, loaded from its own text, as the coefficient:
    sampled at 1,800 triangle centroids by the GPU evaluation kernel."""
    g = golden("darcy")
    sur = pam.loads(str(g["d4_surrogate"]))
    sol = D.solve_darcy(problems(sur)["d4"])
    _check("d4", sol, g, 1e-9)


def test_darcy_errors(cuda):
    m = D.triangulate(4, 4, ((0, 1), (0, 1)))
    with pytest.raises(pam.NumericalError, match="triangle 3 is not positive"):
        D.solve_darcy(D.DarcyProblem(mesh=m, coefficient=lambda p: np.where(np.arange(len(p)) == 3, -1.0, 1.0),
                                     dirichlet={"left": 0.0}))
    hole = D.triangulate(6, 6, ((0, 1), (0, 1)), holes=[(0.0, 0.5, 0.7)])  # removes the whole left face
    with pytest.raises(pam.NumericalError, match="no Dirichlet nodes"):
        D.solve_darcy(D.DarcyProblem(mesh=hole, coefficient=lambda p: np.ones(len(p)), dirichlet={"left": 0.0}))
