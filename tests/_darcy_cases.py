"""The Darcy problems of tests/golden/darcy.npz (same definitions as make_golden.py)."""

import numpy as np

from paper_2605_16564_b200 import darcy as D


def coef1(p):
    return np.exp(np.sin(3 * p[:, 0]) * np.cos(2 * p[:, 1]))


def problems(surrogate=None):
    out = {
        "d1": D.DarcyProblem(mesh=D.triangulate(40, 30, ((0.0, 2.0), (0.0, 1.0))), coefficient=coef1,
                             dirichlet={"left": 1.0, "right": 0.0}),
        "d2": D.DarcyProblem(mesh=D.triangulate(160, 140, ((0.0, 1.0), (0.0, 1.0)), holes=[(0.5, 0.5, 0.12)]),
                             coefficient=lambda p: 10.0 ** (np.where(p[:, 0] > 0.3, 1.0, -0.5)
                                                           + 0.3 * np.sin(7 * p[:, 1])),
                             dirichlet={"left": lambda p: 1.0 + p[:, 1], "right": 0.0},
                             neumann={"top": 0.3}, source=1.0),
        "d3": D.DarcyProblem(mesh=D.line_mesh(50, (0.0, 2.0)), coefficient=lambda p: np.exp(p[:, 0]),
                             dirichlet={"left": 1.0}, neumann={"right": 0.5}, source=2.0),
    }
    if surrogate is not None:
        out["d4"] = D.DarcyProblem(mesh=D.triangulate(30, 30, ((0.0, 1.0), (0.0, 1.0))),
                                   coefficient=surrogate.evaluate, dirichlet={"bottom": 0.0, "top": 1.0})
    return out
