"""Host-side Darcy logic (mesh, CSR pattern, load vector, validation) vs the reference's outputs."""

import io

import numpy as np
import pytest

from paper_2605_16564_b200 import darcy as D
from _darcy_cases import problems


def test_triangulation_layout():
    t = D.triangulate(3, 2, ((0.0, 3.0), (0.0, 2.0)))
    assert t.n_nodes == 12 and t.triangles.shape == (12, 3)
    np.testing.assert_array_equal(t.triangles[:2], [[0, 1, 5], [0, 5, 4]])
    assert np.all(t.areas() > 0)  # counterclockwise
    np.testing.assert_array_equal(t.face_nodes("left"), [0, 4, 8])
    th = D.triangulate(10, 10, ((0, 1), (0, 1)), holes=[(0.5, 0.5, 0.2)])
    assert th.triangles.shape[0] < 200 and th.tri_kept.sum() == th.triangles.shape[0]
    with pytest.raises(ValueError, match="every triangle"):
        D.triangulate(2, 2, ((0, 1), (0, 1)), holes=[(0.5, 0.5, 5.0)])
    with pytest.raises(ValueError, match="unknown face"):
        t.face_nodes("front")


def test_problem_validation():
    m = D.triangulate(2, 2, ((0, 1), (0, 1)))
    with pytest.raises(ValueError, match="at least one Dirichlet"):
        D.DarcyProblem(mesh=m, coefficient=lambda p: p[:, 0], dirichlet={})
    with pytest.raises(ValueError, match="both boundary sets"):
        D.DarcyProblem(mesh=m, coefficient=lambda p: p[:, 0], dirichlet={"left": 0}, neumann={"left": 1})
    with pytest.raises(ValueError, match="unknown face"):
        D.DarcyProblem(mesh=D.line_mesh(4, (0, 1)), coefficient=lambda p: p[:, 0], dirichlet={"top": 0})


@pytest.mark.parametrize("name", ["d1", "d2", "d3"])
def test_pattern_and_load_vector_match_reference(golden, name):
    g = golden("darcy")
    prob = problems()[name]
    elem, pts, _ = D._elements(prob.mesh)
    row_ptr, col, slot_ptr, contrib = D._csr_pattern(elem, prob.mesh.n_nodes)
    np.testing.assert_array_equal(row_ptr, g[f"{name}_A_indptr"])
    np.testing.assert_array_equal(col, g[f"{name}_A_indices"])
    # the contributions of every nonzero, summed in COO order on the host, give the reference's A
    k = prob.coefficient(pts)
    if prob.mesh.dim == 2:
        p = prob.mesh.nodes[elem]
        bv = np.stack([p[:, 1, 1] - p[:, 2, 1], p[:, 2, 1] - p[:, 0, 1], p[:, 0, 1] - p[:, 1, 1]], 1)
        cv = np.stack([p[:, 2, 0] - p[:, 1, 0], p[:, 0, 0] - p[:, 2, 0], p[:, 1, 0] - p[:, 0, 0]], 1)
        local = ((bv[:, :, None] * bv[:, None, :] + cv[:, :, None] * cv[:, None, :])
                 * (k / (4.0 * prob.mesh.areas()))[:, None, None]).ravel()
    else:
        w = k / np.diff(prob.mesh.nodes)
        local = (np.array([1.0, -1.0, -1.0, 1.0])[None, :] * w[:, None]).ravel()
    vals = np.add.reduceat(local[contrib], slot_ptr[:-1])
    np.testing.assert_allclose(vals, g[f"{name}_A_data"], rtol=1e-14, atol=1e-14 * np.abs(vals).max())
    np.testing.assert_array_equal(D._rhs(prob, prob.mesh, elem, pts), g[f"{name}_b"])


def test_pressure_text_and_interpolation():
    m = D.triangulate(2, 1, ((0.0, 2.0), (0.0, 1.0)))
    sol = D.PressureSolution(mesh=m, values=np.arange(6, dtype=float), diagnostics={})
    buf = io.StringIO()
    D.write_pressure_text(sol, buf)
    assert buf.getvalue().splitlines()[:3] == ["2 3 2", "0 2 0 1", "0"]
    np.testing.assert_allclose(sol.interpolate([[0.0, 0.0], [2.0, 1.0], [0.5, 0.25]]), [0.0, 5.0, 1.25])
    with pytest.raises(ValueError, match="outside the mesh"):
        sol.interpolate([[3.0, 0.0]])
