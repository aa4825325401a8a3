"""ORACLE — TEST INFRASTRUCTURE ONLY.  Never imported by the product package.

CPU restatement of the reference's hot path (package ``fieldfit``, files
under /root/reference/pkg/src/fieldfit/, cited below as file:line) in numpy
plus a C restatement of the numba CD core (``cd_core.c``).  It is the checker
for the GPU path: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg and ``--impl reference`` arm) may import it.

Parity is PINNED: ``tests/test_oracle_pins.py`` checks this module against
golden vectors produced by running the reference itself in the build
container (``tests/golden/make_golden.py``), bit for bit where the reference
is deterministic numpy/numba arithmetic, plus the reference test suite's own
known answers (frozen 8x8 objective, mark tie order, centre-count sequences).

Everything operates on plain arrays so the oracle has no dependency on the
product's dataclasses.  Dimension-generic (1D-3D); the 3D mesh/partition/
lattice restatements follow the reference's 1D/2D formulas axis by axis
(geometry.py:122-132, partition.py:56-92, rbf.py:201-214), x fastest.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_CHUNK_BYTES = 64 * 2**20  # rbf.py:18
GAUSS2 = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))  # geometry.py:17
DUPLICATE_TOL = 1e-12  # adaptive.py:27
OFFSETS_1D = ((-0.25,), (0.25,), (0.0,))  # adaptive.py:23
OFFSETS_2D = ((-0.5, 0.0), (0.5, 0.0), (0.0, 0.5))  # adaptive.py:24


# ---------------------------------------------------------------------------
# C core (elastic_net.py:113-161)

_cd_lib = None


def build_cd_core(force: bool = False) -> Path:
    """Compile oracle/liboracle_cd.so with the committed Makefile."""
    so = HERE / "liboracle_cd.so"
    if force or not so.exists() or so.stat().st_mtime < (HERE / "cd_core.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle_cd.so"], check=True)
    return so


def _cd():
    global _cd_lib
    if _cd_lib is None:
        so = build_cd_core()
        lib = ctypes.CDLL(str(so))
        P = ctypes.c_void_p
        lib.oracle_cd_sweeps.restype = ctypes.c_int64
        lib.oracle_cd_sweeps.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, P, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_int64, P, P, P, P]
        _cd_lib = lib
    return _cd_lib


def cd_sweeps(Wf, col_sq, denom, lam1, lam2, tol, max_iters, beta, r, history):
    """Same signature and in-place semantics as _cd_sweeps_jit (elastic_net.py:113)."""
    assert Wf.flags.f_contiguous and Wf.dtype == np.float64
    conv = ctypes.c_int32(0)
    n, m = Wf.shape
    sweeps = _cd().oracle_cd_sweeps(
        Wf.ctypes.data, n, m, col_sq.ctypes.data, denom.ctypes.data, float(lam1), float(lam2),
        float(tol), int(max_iters), beta.ctypes.data, r.ctypes.data, history.ctypes.data,
        ctypes.byref(conv))
    return int(sweeps), bool(conv.value)


# ---------------------------------------------------------------------------
# features (rbf.py:79-91, 123-167)

def log_features(points, centers, widths):
    """L[n, m] = -(sum_k (x-c)^2) * 1/(2 w^2), numpy einsum order (rbf.py:79-91)."""
    pts = np.asarray(points, dtype=float)
    centers = np.asarray(centers, dtype=float)
    n, m, dim = pts.shape[0], centers.shape[0], centers.shape[1]
    inv = 1.0 / (2.0 * np.asarray(widths, dtype=float) ** 2)
    out = np.empty((n, m))
    step = max(1, _CHUNK_BYTES // (8 * m * dim))
    for a in range(0, n, step):
        d = pts[a:a + step, None, :] - centers[None, :, :]
        out[a:a + step] = -np.einsum("nmd,nmd->nm", d, d) * inv[None, :]
    return out


def shepard_features(points, centers, widths):
    """exp(L - rowmax) / rowsum (rbf.py:131-149)."""
    L = log_features(points, centers, widths)
    w = np.exp(L - L.max(axis=1, keepdims=True))
    w /= w.sum(axis=1, keepdims=True)
    return w


def shepard_eval(points, centers, widths, beta):
    """(sum e beta) / (sum e), e = exp(L - rowmax) (rbf.py:152-167)."""
    L = log_features(points, centers, widths)
    w = np.exp(L - L.max(axis=1, keepdims=True))
    den = w.sum(axis=1)
    if not np.all(np.isfinite(den)) or np.any(den <= 0):
        raise FloatingPointError("Shepard denominator degenerate")
    return (w @ np.asarray(beta, dtype=float)) / den


def surrogate_eval(points, centers, widths, beta, log_transform=True):
    v = shepard_eval(points, centers, widths, beta)
    return np.exp(v) if log_transform else v  # rbf.py:190-192


# ---------------------------------------------------------------------------
# Elastic Net fit (elastic_net.py:66-110, 197-205)

def fit(W, y, lam1, lam2, tol, max_iters, beta0=None):
    W = np.asarray(W, dtype=float)
    y = np.asarray(y, dtype=float).ravel()
    n, m = W.shape
    Wf = np.asfortranarray(W)
    col_sq = np.einsum("nm,nm->m", Wf, Wf)
    denom = col_sq + lam2
    beta = np.zeros(m) if beta0 is None else np.asarray(beta0, dtype=float).copy()
    r = y - Wf @ beta
    hist = np.empty(max_iters)
    sweeps, conv = cd_sweeps(Wf, col_sq, denom, lam1, lam2, tol, max_iters, beta, r, hist)
    return {"beta": beta, "objective": float(hist[sweeps - 1]), "iterations": sweeps,
            "converged": conv, "history": hist[:sweeps].copy(), "residual": r}


def fit_log(values, W, lam1, lam2, tol, max_iters, beta0=None):
    v = np.asarray(values, dtype=float).ravel()
    bad = ~(v > 0)
    if np.any(bad):
        j = int(np.argmax(bad))
        raise ValueError(f"field value at cell {j} is not positive: {v[j]}")
    return fit(W, np.log(v), lam1, lam2, tol, max_iters, beta0)


# ---------------------------------------------------------------------------
# mesh / partition / quadrature (geometry.py:105-132, 204-224; partition.py:45-93)

def tensor_points(axes):
    """Row-major tensor product, axis 0 fastest."""
    if len(axes) == 1:
        return np.asarray(axes[0])[:, None]
    grids = np.meshgrid(*axes[::-1], indexing="ij")
    return np.column_stack([g.ravel() for g in grids[::-1]])


def mesh_centroids(counts, bounds):
    sizes = [(b[1] - b[0]) / n for n, b in zip(counts, bounds)]
    axes = [b[0] + (np.arange(n) + 0.5) * d for n, b, d in zip(counts, bounds, sizes)]
    return tensor_points(axes), tuple(sizes)


def partition_boxes(counts, bounds, shape):
    """Boxes (lo, hi, open_hi) x fastest, and the integer cell -> subdomain map."""
    dim = len(counts)
    edges = [b[0] + (b[1] - b[0]) * np.arange(p + 1) / p for b, p in zip(bounds, shape)]
    boxes = []
    for multi in np.ndindex(*tuple(shape)[::-1]):
        m = multi[::-1]
        boxes.append((tuple(float(edges[k][m[k]]) for k in range(dim)),
                      tuple(float(edges[k][m[k] + 1]) for k in range(dim)),
                      tuple(m[k] < shape[k] - 1 for k in range(dim))))
    per = [n // p for n, p in zip(counts, shape)]
    idx = np.arange(int(np.prod(counts)))
    owner = (idx % counts[0]) // per[0]
    if dim >= 2:
        owner = owner + shape[0] * (((idx // counts[0]) % counts[1]) // per[1])
    if dim == 3:
        owner = owner + shape[0] * shape[1] * ((idx // (counts[0] * counts[1])) // per[2])
    return boxes, owner, edges


def box_contains(box, pts):
    lo, hi, open_hi = box
    mask = np.ones(pts.shape[0], dtype=bool)
    for k in range(len(lo)):
        mask &= pts[:, k] >= lo[k]
        mask &= (pts[:, k] < hi[k]) if open_hi[k] else (pts[:, k] <= hi[k])
    return mask


def locate_many(pts, boxes):
    """Per-box half-open masks (geometry.py:242-258)."""
    pts = np.asarray(pts, dtype=float)
    owner = np.full(pts.shape[0], -1, dtype=np.int64)
    claimed = np.zeros(pts.shape[0], dtype=bool)
    for i, b in enumerate(boxes):
        mask = box_contains(b, pts)
        if np.any(mask & claimed):
            j = int(np.argmax(mask & claimed))
            raise ValueError(f"point index {j} claimed by boxes {owner[j]} and {i}")
        owner[mask] = i
        claimed |= mask
    if not np.all(claimed):
        j = int(np.argmax(~claimed))
        raise ValueError(f"point index {j} lies outside all boxes")
    return owner


def subdomain_rows(centroids, box):
    """Cells whose centroid lies in the half-open box, ascending (fields.py:61-73)."""
    return np.flatnonzero(box_contains(box, centroids))


def quad_offsets(cell_size, order):
    size = np.atleast_1d(np.asarray(cell_size, dtype=float))
    dim = size.shape[0]
    measure = float(np.prod(size))
    if order == 1:
        offs = np.zeros((1, dim))
    elif order == 2:
        g = np.array(GAUSS2) - 0.5
        grids = np.meshgrid(*[g * size[k] for k in range(dim)], indexing="ij")
        offs = np.stack([gr.ravel() for gr in grids], axis=1)
    else:
        raise ValueError(f"unsupported quadrature order {order} (use 1 or 2)")
    return offs, np.full(offs.shape[0], measure / offs.shape[0])


def lattice_centers(lo, hi, g):
    """g^dim lattice at lo + (k + 1/2)(hi - lo)/g, x fastest (rbf.py:201-214)."""
    axes = [lo[k] + (np.arange(g) + 0.5) * (hi[k] - lo[k]) / g for k in range(len(lo))]
    return tensor_points(axes)


# ---------------------------------------------------------------------------
# adaptive loop (adaptive.py:122-271; fields.py:113-121)

def residuals(centroids, values, cell_size, centers, widths, beta, order=1, log_transform=True):
    """(R per cell, num, den) — residual_indicators + l2_misfit_parts."""
    offs, wts = quad_offsets(cell_size, order)
    c = np.asarray(centroids, dtype=float)
    pts = c[:, None, :] + offs[None, :, :]
    n, nq, dim = pts.shape
    vals = surrogate_eval(pts.reshape(-1, dim), centers, widths, beta, log_transform).reshape(n, nq)
    diff2 = (vals - np.asarray(values)[:, None]) ** 2
    R = diff2 @ wts
    num = float(np.sum(diff2 @ wts))
    den = float(np.sum(wts) * np.sum(np.asarray(values) ** 2))
    return R, num, den


def mark(R, k_top):
    r = np.asarray(R, dtype=float)
    if k_top > r.shape[0]:
        raise ValueError(f"k_top={k_top} exceeds cell count {r.shape[0]}")
    order = np.lexsort((np.arange(r.shape[0]), -r))
    order = order[r[order] > 0.0]
    return order[:k_top]


def nearest_entry(centers, widths, point):
    d2 = np.sum((centers - point[None, :]) ** 2, axis=1)
    return int(np.lexsort((np.arange(centers.shape[0]), widths, d2))[0])


def enrich(centers, widths, marked, centroids, cell_size, box_lo, box_hi, eta, m_q, offsets):
    marked = np.asarray(marked, dtype=int)
    if marked.size == 0:
        raise ValueError("marked cell set must not be empty")
    dim = centroids.shape[1]
    offs = np.asarray(offsets, dtype=float)[:m_q]
    scale = np.asarray(cell_size, dtype=float)
    out_c, out_w = [], []
    for cell in marked:
        x_t = centroids[cell]
        width = eta * float(widths[nearest_entry(centers, widths, x_t)])
        for off in offs:
            cand = np.clip(x_t + off * scale, box_lo, box_hi)
            same_c = np.all(np.abs(centers - cand[None, :]) <= DUPLICATE_TOL, axis=1)
            same_w = np.abs(widths - width) <= DUPLICATE_TOL
            if np.any(same_c & same_w):
                continue
            out_c.append(cand)
            out_w.append(width)
    if not out_c:
        return np.empty((0, dim)), np.empty(0)
    return np.asarray(out_c), np.asarray(out_w)


def fit_adaptive(centroids, values, cell_size, box_lo, box_hi, centers, widths, cfg, gens=None):
    """Round loop of adaptive.py:213-271 on plain arrays.

    cfg keys: lam1 lam2 tol max_iters k_top m_max eps_tol eta m_q max_rounds
    offsets (or None -> 1D/2D defaults) quad_order.
    Returns dict(centers, widths, generations, beta, reports=[dict...], marked=[...]).
    """
    centroids = np.asarray(centroids, dtype=float)
    values = np.asarray(values, dtype=float)
    dim = centroids.shape[1]
    centers = np.asarray(centers, dtype=float).copy()
    widths = np.asarray(widths, dtype=float).copy()
    gens = np.zeros(centers.shape[0], dtype=int) if gens is None else np.asarray(gens).copy()
    offsets = cfg.get("offsets") or (OFFSETS_1D if dim == 1 else OFFSETS_2D)
    beta = np.zeros(centers.shape[0])
    added = 0
    reports, marks = [], []
    order = cfg.get("quad_order", 1)
    for rnd in range(cfg["max_rounds"]):
        W = shepard_features(centroids, centers, widths)
        res = fit_log(values, W, cfg["lam1"], cfg["lam2"], cfg["tol"], cfg["max_iters"], beta)
        beta = res["beta"]
        R, num, den = residuals(centroids, values, cell_size, centers, widths, beta, order)
        reports.append({"round": rnd, "centers": centers.shape[0], "added": added,
                        "max_residual": float(R.max()), "rel_l2": float(np.sqrt(num / den)),
                        "abs_l2": float(np.sqrt(num)), "objective": res["objective"],
                        "iterations": res["iterations"], "converged": res["converged"]})
        if float(R.max()) < cfg.get("eps_tol", 0.0):
            break
        if added >= cfg["m_max"]:
            break
        if rnd == cfg["max_rounds"] - 1:
            break
        mk = mark(R, min(cfg["k_top"], centroids.shape[0]))
        marks.append(mk)
        if mk.size == 0:
            break
        nc, nw = enrich(centers, widths, mk, centroids, cell_size, box_lo, box_hi, cfg["eta"],
                        cfg["m_q"], offsets)
        if nc.shape[0] == 0:
            break
        centers = np.vstack([centers, nc])
        widths = np.concatenate([widths, nw])
        gens = np.concatenate([gens, np.full(nc.shape[0], rnd + 1, dtype=int)])
        beta = np.concatenate([beta, np.zeros(nc.shape[0])])
        added += nc.shape[0]
    return {"centers": centers, "widths": widths, "generations": gens, "beta": beta,
            "reports": reports, "marked": marks}


def global_evaluate(points, boxes, locals_, log_transform=True):
    """locate_many + per-owner evaluation, order preserved (partition.py:132-143).

    locals_: list of (centers, widths, beta)."""
    pts = np.asarray(points, dtype=float)
    owner = locate_many(pts, boxes)
    out = np.empty(pts.shape[0])
    for i, (c, w, b) in enumerate(locals_):
        sel = owner == i
        if np.any(sel):
            out[sel] = surrogate_eval(pts[sel], c, w, b, log_transform)
    return out, owner


def n_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
