"""Darcy pressure solve that consumes a surrogate — SURVEY §8f row 2.

Mirror of the reference's P1 solver (darcy.py): structured triangulations
with optional disk holes, named-face Dirichlet / Neumann data, coefficient
sampled at element centroids (one-point quadrature, so ``coefficient`` may be
``GlobalSurrogate.evaluate``, i.e. the K4 evaluation kernel), stiffness
assembly and a Jacobi-preconditioned CG on the device (csrc/darcy.cu).

Host side: mesh and face bookkeeping, the integer CSR pattern, the right-hand
side (source and Neumann terms are O(nodes) vectors, as in the reference) and
the result dataclasses.  Device side: stiffness values, Dirichlet lifting
(A x_D), the PCG solve and the true residual.  Differences from the
reference, all within its tolerances: systems of <= 20,000 unknowns, which the
reference factorises directly (darcy.py:266-269), are solved here by the same
PCG to ||r|| < 1e-14 ||b||; ``diagnostics["method"]`` reports ``"cg"``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Mapping

import numpy as np

from . import _native as nat
from .errors import NumericalError
from .fields import FieldData, relative_l2_error

FACES_2D = ("left", "right", "bottom", "top")
FACES_1D = ("left", "right")
DIRECT_SOLVE_LIMIT = 20_000  # reference darcy.py:26
DIRECT_EQUIVALENT_RTOL = 1e-14
CG_RTOL = 1e-10  # reference darcy.py:285


@dataclass(frozen=True)
class Triangulation:
    """Structured triangle mesh of a rectangle, possibly with disk holes (darcy.py:30-78)."""

    counts: tuple[int, int]
    bounds: tuple[tuple[float, float], tuple[float, float]]
    nodes: np.ndarray  # (n_nodes, 2)
    triangles: np.ndarray  # (n_tri, 3), counterclockwise
    tri_kept: np.ndarray  # mask into the full 2*nx*ny triangle list

    @property
    def n_nodes(self) -> int:
        return self.nodes.shape[0]

    @property
    def dim(self) -> int:
        return 2

    def centroids(self) -> np.ndarray:
        return self.nodes[self.triangles].mean(axis=1)

    def areas(self) -> np.ndarray:
        p = self.nodes[self.triangles]
        u, v = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]
        return 0.5 * (u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0])

    def face_nodes(self, face: str) -> np.ndarray:
        (x0, x1), (y0, y1) = self.bounds
        x, y = self.nodes[:, 0], self.nodes[:, 1]
        masks = {"left": x == x0, "right": x == x1, "bottom": y == y0, "top": y == y1}
        if face not in masks:
            raise ValueError(f"unknown face {face!r}; expected one of {FACES_2D}")
        return np.flatnonzero(masks[face])

    def boundary_edges(self) -> np.ndarray:
        """Edges of exactly one kept triangle, as sorted node pairs (np.unique order)."""
        t = self.triangles
        e = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
        uniq, cnt = np.unique(e, axis=0, return_counts=True)
        return uniq[cnt == 1]


@dataclass(frozen=True)
class LineMesh:
    """Uniform interval mesh (darcy.py:80-101)."""

    count: int
    bounds: tuple[float, float]
    nodes: np.ndarray  # (count + 1,)

    @property
    def n_nodes(self) -> int:
        return self.nodes.shape[0]

    @property
    def dim(self) -> int:
        return 1

    def face_nodes(self, face: str) -> np.ndarray:
        if face not in FACES_1D:
            raise ValueError(f"unknown face {face!r}; expected one of {FACES_1D}")
        return np.array([0 if face == "left" else self.count])


def line_mesh(n: int, bounds) -> LineMesh:
    if n < 1:
        raise ValueError(f"element count must be >= 1, got {n}")
    lo, hi = float(bounds[0]), float(bounds[1])
    if lo >= hi:
        raise ValueError(f"inverted bounds {bounds}")
    return LineMesh(count=n, bounds=(lo, hi), nodes=np.linspace(lo, hi, n + 1))


def triangulate(nx: int, ny: int, bounds, holes=()) -> Triangulation:
    """Rectangle grid split along each cell's lower-left/upper-right diagonal (darcy.py:113-153).

    Node (i, j) is i + j (nx+1) (x fastest); cell (i, j) gives the lower
    triangle (n00, n10, n11) then the upper (n00, n11, n01).  Triangles whose
    centroid lies strictly inside a hole disk are dropped.
    """
    if nx < 1 or ny < 1:
        raise ValueError(f"grid counts must be >= 1, got {(nx, ny)}")
    b = np.asarray(bounds, dtype=float).reshape(2, 2)
    xs = np.linspace(b[0, 0], b[0, 1], nx + 1)
    ys = np.linspace(b[1, 0], b[1, 1], ny + 1)
    nodes = np.column_stack([np.tile(xs, ny + 1), np.repeat(ys, nx + 1)])
    n00 = (np.arange(ny)[:, None] * (nx + 1) + np.arange(nx)[None, :]).ravel()
    tris = np.empty((2 * nx * ny, 3), dtype=np.int64)
    tris[0::2] = np.column_stack([n00, n00 + 1, n00 + nx + 2])
    tris[1::2] = np.column_stack([n00, n00 + nx + 2, n00 + nx + 1])
    kept = np.ones(tris.shape[0], dtype=bool)
    if holes:
        cent = nodes[tris].mean(axis=1)
        for cx, cy, r in holes:
            kept &= (cent[:, 0] - cx) ** 2 + (cent[:, 1] - cy) ** 2 > r ** 2
        if not kept.any():
            raise ValueError("holes remove every triangle")
    return Triangulation(counts=(nx, ny), bounds=((b[0, 0], b[0, 1]), (b[1, 0], b[1, 1])), nodes=nodes,
                         triangles=tris[kept], tri_kept=kept)


@dataclass(frozen=True)
class DarcyProblem:
    """-div(K grad p) = f with named-face boundary data (darcy.py:155-180)."""

    mesh: Triangulation | LineMesh
    coefficient: Callable[[np.ndarray], np.ndarray]
    dirichlet: Mapping[str, float | Callable]
    neumann: Mapping[str, float | Callable] = field(default_factory=dict)
    source: float | Callable = 0.0

    def __post_init__(self):
        faces = FACES_1D if self.mesh.dim == 1 else FACES_2D
        for name in (*self.dirichlet, *self.neumann):
            if name not in faces:
                raise ValueError(f"unknown face {name!r}; expected one of {faces}")
        both = set(self.dirichlet) & set(self.neumann)
        if both:
            raise ValueError(f"faces {sorted(both)} appear in both boundary sets")
        if not self.dirichlet:
            raise ValueError("at least one Dirichlet face is required")


@dataclass(frozen=True)
class PressureSolution:
    """Nodal pressure (NaN on nodes removed by holes), diagnostics, unconstrained (A, b)."""

    mesh: Triangulation | LineMesh
    values: np.ndarray
    diagnostics: dict
    system: tuple = field(repr=False, default=None)

    def interpolate(self, points) -> np.ndarray:
        if self.mesh.dim == 1:
            return np.interp(np.asarray(points, dtype=float).ravel(), self.mesh.nodes, self.values)
        return _interp_p1(self.mesh, self.values, points)

    def boundary_reaction(self, face: str) -> float:
        """Discrete flux through a face: sum over its nodes of A p - b (darcy.py:203-208)."""
        A, b = self.system
        vals = np.where(np.isfinite(self.values), self.values, 0.0)
        return float((A @ vals - b)[self.mesh.face_nodes(face)].sum())


def _interp_p1(tri: Triangulation, values, points) -> np.ndarray:
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    nx, ny = tri.counts
    (x0, x1), (y0, y1) = tri.bounds
    if np.any(pts[:, 0] < x0) or np.any(pts[:, 0] > x1) or np.any(pts[:, 1] < y0) or np.any(pts[:, 1] > y1):
        raise ValueError("interpolation point outside the mesh")
    dx, dy = (x1 - x0) / nx, (y1 - y0) / ny
    ix = np.minimum(((pts[:, 0] - x0) / dx).astype(int), nx - 1)
    iy = np.minimum(((pts[:, 1] - y0) / dy).astype(int), ny - 1)
    xi, yi = (pts[:, 0] - x0) / dx - ix, (pts[:, 1] - y0) / dy - iy
    base = iy * (nx + 1) + ix
    v00, v10 = values[base], values[base + 1]
    v01, v11 = values[base + nx + 1], values[base + nx + 2]
    lower = v00 + (v10 - v00) * xi + (v11 - v10) * yi
    upper = v00 + (v11 - v01) * xi + (v01 - v00) * yi
    return np.where(xi >= yi, lower, upper)


def _as_func(value):
    if callable(value):
        return value
    return lambda pts, v=float(value): np.full(np.atleast_2d(pts).shape[0], v)


def _elements(mesh):
    """(element nodes, centroids as evaluation points, kind) of a P1 mesh."""
    if mesh.dim == 1:
        e = np.column_stack([np.arange(mesh.count), np.arange(1, mesh.count + 1)]).astype(np.int64)
        mids = 0.5 * (mesh.nodes[:-1] + mesh.nodes[1:])
        return e, mids[:, None], "element"
    return np.ascontiguousarray(mesh.triangles, dtype=np.int64), mesh.centroids(), "triangle"


def _csr_pattern(elem, n_nodes):
    """CSR pattern of the COO (rows = repeat(elem), cols = tile(elem)) and, per nonzero,
    its contributions in COO order."""
    k = elem.shape[1]
    rows = np.repeat(elem, k, axis=1).ravel()
    cols = np.tile(elem, (1, k)).ravel()
    key = rows * n_nodes + cols
    order = np.argsort(key, kind="stable")
    skey = key[order]
    first = np.concatenate([[True], skey[1:] != skey[:-1]])
    slot_ptr = np.concatenate([np.flatnonzero(first), [skey.size]]).astype(np.int64)
    uk = skey[first]
    r, c = uk // n_nodes, uk % n_nodes
    row_ptr = np.zeros(n_nodes + 1, dtype=np.int64)
    np.add.at(row_ptr, r + 1, 1)
    return np.cumsum(row_ptr), c.astype(np.int64), slot_ptr, order.astype(np.int64)


def _rhs(problem, mesh, elem, pts):
    """Source and Neumann load vector (darcy.py:334-346, 365-375)."""
    b = np.zeros(mesh.n_nodes)
    f = np.asarray(_as_func(problem.source)(pts), dtype=float)
    if mesh.dim == 1:
        h = np.diff(mesh.nodes)
        np.add.at(b, np.arange(mesh.count), 0.5 * f * h)
        np.add.at(b, np.arange(1, mesh.count + 1), 0.5 * f * h)
        for face, data in problem.neumann.items():
            node = mesh.face_nodes(face)[0]
            b[node] += float(np.asarray(_as_func(data)(mesh.nodes[node:node + 1][:, None]))[0])
        return b
    np.add.at(b, elem.ravel(), np.repeat(f * mesh.areas() / 3.0, 3))
    if problem.neumann:
        bedges = mesh.boundary_edges()
        for face, data in problem.neumann.items():
            sel = np.isin(bedges, mesh.face_nodes(face)).all(axis=1)
            edges = bedges[sel]
            if edges.size == 0:
                continue
            a, c = mesh.nodes[edges[:, 0]], mesh.nodes[edges[:, 1]]
            q = np.asarray(_as_func(data)(0.5 * (a + c)), dtype=float)
            np.add.at(b, edges.ravel(), np.repeat(0.5 * q * np.linalg.norm(c - a, axis=1), 2))
    return b


def solve_darcy(problem: DarcyProblem) -> PressureSolution:
    """Assemble and solve the P1 pressure system on the device (reference darcy.py:238-305)."""
    import scipy.sparse as sp
    import torch

    mesh = problem.mesh
    dev = nat.device()
    lib = nat.lib()
    P = nat.ptr
    st = nat.stream_ptr()
    elem, pts, kind = _elements(mesh)
    k = np.asarray(problem.coefficient(pts), dtype=float).ravel()
    bad = ~(k > 0) | ~np.isfinite(k)
    if bad.any():
        j = int(np.argmax(bad))
        raise NumericalError(f"coefficient sample at {kind} {j} is not positive: {k[j]}")

    n = mesh.n_nodes
    row_ptr, col, slot_ptr, contrib = _csr_pattern(elem, n)
    nnz = col.size
    keep = [nat.to_dev(a) for a in (row_ptr, col, slot_ptr, contrib, elem,
                                    np.ascontiguousarray(mesh.nodes, dtype=np.float64).reshape(n, -1), k)]
    d_rp, d_col, d_sp, d_ctr, d_elem, d_nodes, d_k = keep
    d_val = torch.empty(nnz, dtype=torch.float64, device=dev)
    nat.check(lib.pam_p1_values_f64(mesh.dim, nnz, P(d_sp), P(d_ctr), P(d_elem), P(d_nodes), P(d_k),
                                    P(d_val), st), "pam_p1_values_f64")
    b = _rhs(problem, mesh, elem, pts)

    active = np.ones(n, dtype=bool)
    if mesh.dim == 2:
        active[:] = False
        active[np.unique(mesh.triangles)] = True
    x = np.zeros(n)
    dmask = np.zeros(n, dtype=bool)
    for face, data in problem.dirichlet.items():
        nodes = mesh.face_nodes(face)
        nodes = nodes[active[nodes]]
        coords = mesh.nodes[nodes] if mesh.dim == 2 else mesh.nodes[nodes][:, None]
        x[nodes] = np.asarray(_as_func(data)(coords), dtype=float)
        dmask[nodes] = True
    if not dmask.any():
        raise NumericalError("no Dirichlet nodes: the system is singular")
    free = active & ~dmask

    # rhs = b - A x_D on the device, restricted to the free nodes
    d_x = nat.to_dev(x)
    d_ax = torch.empty(n, dtype=torch.float64, device=dev)
    nat.check(lib.pam_csr_spmv_f64(n, P(d_rp), P(d_col), P(d_val), P(d_x), P(d_ax), st), "pam_csr_spmv_f64")
    fidx = np.flatnonzero(free)
    n_free = fidx.size
    d_fidx = nat.to_dev(fidx.astype(np.int64))
    d_bf = (nat.to_dev(b) - d_ax).index_select(0, d_fidx).contiguous()

    method, iterations, rel_res = "none", 0, 0.0
    if n_free > 0:
        # free-free block: host integer filtering of the pattern, device gather of the values
        newid = np.full(n, -1, dtype=np.int64)
        newid[fidx] = np.arange(n_free)
        rows_all = np.repeat(np.arange(n), np.diff(row_ptr))
        keepnz = free[rows_all] & free[col]
        src = np.flatnonzero(keepnz)
        frp = np.zeros(n_free + 1, dtype=np.int64)
        np.add.at(frp, newid[rows_all[src]] + 1, 1)
        frp = np.cumsum(frp)
        d_frp, d_fcol = nat.to_dev(frp), nat.to_dev(newid[col[src]])
        d_fval = d_val.index_select(0, nat.to_dev(src.astype(np.int64))).contiguous()
        rtol = DIRECT_EQUIVALENT_RTOL if n_free <= DIRECT_SOLVE_LIMIT else CG_RTOL
        work = torch.empty(int(lib.pam_pcg_workspace_bytes(n_free)), dtype=torch.uint8, device=dev)
        d_xf = torch.empty(n_free, dtype=torch.float64, device=dev)
        it = np.zeros(1, dtype=np.int64)
        conv = np.zeros(1, dtype=np.int32)
        rr = np.zeros(1, dtype=np.float64)
        nat.check(lib.pam_pcg_f64(n_free, P(d_frp), P(d_fcol), P(d_fval), P(d_bf), P(d_xf), rtol,
                                  20 * n_free, P(work), it.ctypes.data, conv.ctypes.data, rr.ctypes.data, st),
                  "pam_pcg_f64")
        if not conv[0]:
            raise NumericalError(f"conjugate gradient failed to converge (info={20 * n_free})")
        method, iterations = "cg", int(it[0])
        d_res = torch.empty(n_free, dtype=torch.float64, device=dev)
        nat.check(lib.pam_csr_spmv_f64(n_free, P(d_frp), P(d_fcol), P(d_fval), P(d_xf), P(d_res), st),
                  "pam_csr_spmv_f64")
        res = float(torch.linalg.vector_norm(d_res - d_bf))
        ref = float(torch.linalg.vector_norm(d_bf))
        rel_res = res / ref if ref > 0 else res
        x[fidx] = d_xf.cpu().numpy()
    del keep
    A = sp.csr_matrix((d_val.cpu().numpy(), col, row_ptr), shape=(n, n))
    return PressureSolution(mesh=mesh, values=np.where(active, x, np.nan),
                            diagnostics={"method": method, "iterations": iterations, "residual": rel_res},
                            system=(A, b))


def pressure_rel_error(p_ref: PressureSolution, p_test: PressureSolution) -> float:
    """Relative L2 distance of two pressures on the reference mesh (darcy.py:378-411)."""
    if p_ref.mesh.dim == 1:
        nodes = p_ref.mesh.nodes
        g = 0.5 / np.sqrt(3.0)
        mids, h = 0.5 * (nodes[:-1] + nodes[1:]), np.diff(nodes)
        pts = np.concatenate([mids - g * h, mids + g * h])
        w = np.concatenate([0.5 * h, 0.5 * h])
        a, t = p_ref.interpolate(pts), p_test.interpolate(pts)
        num, den = float(np.sum(w * (a - t) ** 2)), float(np.sum(w * a ** 2))
    else:
        tri = p_ref.mesh
        corners, vals, w = tri.nodes[tri.triangles], p_ref.values[tri.triangles], tri.areas() / 3.0
        num = den = 0.0
        for i, j in ((0, 1), (1, 2), (2, 0)):
            a = 0.5 * (vals[:, i] + vals[:, j])
            t = p_test.interpolate(0.5 * (corners[:, i] + corners[:, j]))
            num += float(np.sum(w * (a - t) ** 2))
            den += float(np.sum(w * a ** 2))
    if den == 0.0:
        raise ValueError("reference pressure has zero norm")
    return float(np.sqrt(num / den))


def field_rel_error(data: FieldData, surrogate, order: int = 1) -> float:
    """Relative L2 error of a continuous reconstruction against cell data (darcy.py:414-417)."""
    evaluate = surrogate.evaluate if hasattr(surrogate, "evaluate") else surrogate
    return relative_l2_error(data.whole(), evaluate, order=order)


def write_pressure_text(solution: PressureSolution, sink) -> None:
    """Nodal pressure in the field-file grammar (darcy.py:420-440)."""
    mesh = solution.mesh
    if mesh.dim == 1:
        header = [f"1 {mesh.n_nodes}", f"{mesh.bounds[0]:.17g} {mesh.bounds[1]:.17g}"]
    else:
        (nx, ny), ((x0, x1), (y0, y1)) = mesh.counts, mesh.bounds
        header = [f"2 {nx + 1} {ny + 1}", f"{x0:.17g} {x1:.17g} {y0:.17g} {y1:.17g}"]
    text = "\n".join(header + [f"{v:.17g}" for v in solution.values]) + "\n"
    if hasattr(sink, "write"):
        sink.write(text)
    else:
        with open(sink, "w") as fh:
            fh.write(text)
