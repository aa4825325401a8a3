"""Residual-driven fit/mark/enrich loop (mirror of reference adaptive.py:1-271).

``fit_adaptive`` runs the whole round loop on the GPU through the batched
engine (a batch of one); ``mark`` and ``enrich`` call the same device kernels
(K3c/K3d) the batched path uses, so the single-subdomain API and
``fit_parallel`` share one implementation.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .elastic_net import ElasticNetConfig
from .fields import SubdomainField
from .geometry import QuadratureRule
from .rbf import LocalSurrogate, RbfDictionary

# new-centre offsets per marked cell, in units of the cell size (adaptive.py:22-24)
DEFAULT_OFFSETS_1D = ((-0.25,), (0.25,), (0.0,))
DEFAULT_OFFSETS_2D = ((-0.5, 0.0), (0.5, 0.0), (0.0, 0.5))

# two entries are duplicates when centres and widths agree to this tolerance
DUPLICATE_TOL = 1e-12


@dataclass(frozen=True)
class AdaptiveConfig:
    """Controls for the enrichment loop (adaptive.py:30-75)."""

    k_top: int = 1
    m_max: int = 0
    eps_tol: float = 0.0
    eta: float = 0.5
    m_q: int = 3
    max_rounds: int = 50
    elastic: ElasticNetConfig = field(default_factory=ElasticNetConfig)
    offsets: tuple[tuple[float, ...], ...] | None = None
    quad_order: int = 1

    def __post_init__(self):
        if self.k_top < 1:
            raise ValueError(f"k_top must be >= 1, got {self.k_top}")
        if not 0.0 < self.eta < 1.0:
            raise ValueError(f"eta must lie in (0, 1), got {self.eta}")
        if self.m_q < 1:
            raise ValueError(f"m_q must be >= 1, got {self.m_q}")
        if self.m_max < 0:
            raise ValueError(f"m_max must be >= 0, got {self.m_max}")
        if self.eps_tol < 0:
            raise ValueError(f"eps_tol must be >= 0, got {self.eps_tol}")
        if self.max_rounds < 1:
            raise ValueError(f"max_rounds must be >= 1, got {self.max_rounds}")
        if self.offsets is not None and len(self.offsets) != self.m_q:
            raise ValueError(f"offsets has {len(self.offsets)} entries but m_q={self.m_q}")

    def offsets_for_dim(self, dim: int) -> tuple[tuple[float, ...], ...]:
        if self.offsets is not None:
            return self.offsets
        if self.m_q != 3:
            raise ValueError("default offsets exist only for m_q=3; pass offsets explicitly")
        return DEFAULT_OFFSETS_1D if dim == 1 else DEFAULT_OFFSETS_2D


@dataclass(frozen=True)
class RoundReport:
    """Per-round fitting record (adaptive.py:78-97); ``seconds`` is the batch round wall time."""

    round: int
    centers: int
    added: int
    max_residual: float
    rel_l2: float
    abs_l2: float
    objective: float
    seconds: float


REPORT_CSV_COLUMNS = ("round", "centers", "max_RT", "rel_L2", "objective", "seconds")


def reports_to_csv(reports, sink, provenance: str | None = None) -> None:
    """Write round reports as CSV; timing stays isolated in its own column."""
    lines = []
    if provenance:
        lines.append(f"# {provenance}")
    lines.append(",".join(REPORT_CSV_COLUMNS))
    for r in reports:
        lines.append(
            f"{r.round},{r.centers},{r.max_residual:.17g},{r.rel_l2:.17g},"
            f"{r.objective:.17g},{r.seconds:.6f}"
        )
    text = "\n".join(lines) + "\n"
    if hasattr(sink, "write"):
        sink.write(text)
    else:
        with open(sink, "w") as fh:
            fh.write(text)


def residual_indicator(surrogate, cell_value: float, quad: QuadratureRule) -> float:
    """Quadrature residual sum_l w_l (K*(x_l) - K_T)^2 on one cell (adaptive.py:122-130)."""
    vals = np.asarray(surrogate.evaluate(quad.points), dtype=float)
    return float(np.sum(quad.weights * (vals - cell_value) ** 2))


def residual_indicators(surrogate, sub: SubdomainField, order: int = 1) -> np.ndarray:
    """Residual indicator for every cell of a subdomain (adaptive.py:133-138)."""
    pts, wts = sub.quadrature(order)
    n, n_q, dim = pts.shape
    vals = np.asarray(surrogate.evaluate(pts.reshape(-1, dim)), dtype=float).reshape(n, n_q)
    return ((vals - sub.values[:, None]) ** 2) @ wts


def mark(indicators, k_top: int) -> np.ndarray:
    """Indices of the k_top worst cells by residual then index (adaptive.py:141-152), on the GPU."""
    from . import _native as nat

    r = np.ascontiguousarray(np.asarray(indicators, dtype=float).ravel())
    if k_top > r.shape[0]:
        raise ValueError(f"k_top={k_top} exceeds cell count {r.shape[0]}")
    if r.shape[0] == 0:
        return np.empty(0, dtype=np.int64)
    torch = nat.torch_mod()
    dev = nat.device()
    d_r = nat.to_dev(r)
    d_off = nat.to_dev(np.array([0, r.shape[0]], dtype=np.int64))
    d_k = nat.to_dev(np.array([k_top], dtype=np.int32))
    marked = torch.zeros(max(k_top, 1), dtype=torch.int32, device=dev)
    n_marked = torch.zeros(1, dtype=torch.int32, device=dev)
    nat.check(nat.lib().pam_mark_f64(1, nat.ptr(d_off), nat.ptr(d_r), nat.ptr(d_k), None,
                                     max(k_top, 1), nat.ptr(marked), nat.ptr(n_marked),
                                     nat.stream_ptr()), "pam_mark_f64")
    n = int(n_marked.item())
    return marked[:n].cpu().numpy().astype(np.int64)


def enrich(dictionary: RbfDictionary, marked, sub: SubdomainField, eta: float, m_q: int,
           offsets=None):
    """New (centre, width) entries for the marked cells (adaptive.py:167-210), on the GPU.

    Parent = nearest entry (ties: narrowest, then oldest); width = eta *
    parent width; candidates clamp(x_T + off * cell_size) into the box;
    candidates duplicating an EXISTING entry (<= 1e-12) are dropped.
    """
    from . import _native as nat

    marked = np.asarray(marked, dtype=int).ravel()
    if marked.size == 0:
        raise ValueError("marked cell set must not be empty")
    dim = sub.centroids.shape[1]
    if offsets is None:
        offsets = DEFAULT_OFFSETS_1D if dim == 1 else DEFAULT_OFFSETS_2D
    off = np.asarray(offsets, dtype=float)[:m_q]
    off = np.array(np.broadcast_to(off, (off.shape[0], dim)))  # numpy broadcast semantics
    mq = off.shape[0]
    torch = nat.torch_mod()
    dev = nat.device()
    M = len(dictionary)
    K = marked.size
    cap = M + K * mq
    cen = np.zeros((cap, dim))
    cen[:M] = dictionary.centers
    wid = np.ones(cap)
    wid[:M] = dictionary.widths
    d_c = nat.to_dev(cen)
    d_w = nat.to_dev(wid)
    d_g = torch.zeros(cap, dtype=torch.int32, device=dev)
    d_b = torch.zeros(cap, dtype=torch.float64, device=dev)
    d_pts = nat.to_dev(np.asarray(sub.centroids, dtype=float))
    n = sub.centroids.shape[0]
    if np.any(marked < 0) or np.any(marked >= n):
        raise IndexError("marked cell index out of range")
    i64 = nat.to_dev(np.array([0, n, 0], dtype=np.int64))  # row_off[2], dict_off
    i32 = nat.to_dev(np.array([cap, M, K, mq], dtype=np.int32))  # dict_cap, m_cur, n_marked, m_q
    d_marked = nat.to_dev(marked.astype(np.int32))
    d_eta = nat.to_dev(np.array([eta], dtype=np.float64))
    d_off = nat.to_dev(off.reshape(-1))
    d_size = nat.to_dev(np.asarray(sub.cell_size, dtype=float))
    d_lo = nat.to_dev(np.asarray(sub.box.lo, dtype=float))
    d_hi = nat.to_dev(np.asarray(sub.box.hi, dtype=float))
    n_added = torch.zeros(1, dtype=torch.int32, device=dev)
    err = nat.ErrorWord()
    nat.check(nat.lib().pam_enrich_f64(
        dim, 1, nat.ptr(i64), nat.ptr(d_pts), nat.ptr(d_marked), nat.ptr(i32[2:]), K, nat.ptr(d_eta),
        nat.ptr(i32[3:]), mq, nat.ptr(d_off), nat.ptr(d_size), nat.ptr(d_lo), nat.ptr(d_hi),
        nat.ptr(i64[2:]), nat.ptr(i32), nat.ptr(i32[1:]), nat.ptr(d_c), nat.ptr(d_w), nat.ptr(d_g),
        nat.ptr(d_b), 1, None, nat.ptr(n_added), nat.ptr(err.t), nat.stream_ptr()), "pam_enrich_f64")
    added = int(n_added.item())
    if added == 0:
        return np.empty((0, dim)), np.empty(0)
    return (d_c.view(cap, dim)[M:M + added].cpu().numpy(), d_w[M:M + added].cpu().numpy())


def fit_adaptive(sub: SubdomainField, initial: RbfDictionary,
                 config: AdaptiveConfig) -> tuple[LocalSurrogate, list[RoundReport]]:
    """Run the enrichment loop on the GPU; returns the surrogate and its history.

    Same contract as adaptive.py:213-271: every report corresponds to a
    completed fit and the dictionary only grows after a fit.
    """
    from . import _native as nat
    from .engine import EngineError, FitEngine, rcb_permutation, reports_for

    dim = sub.centroids.shape[1]
    if initial.dim != dim:
        raise ValueError(f"points have dim {dim}, dictionary has dim {initial.dim}")
    n = sub.centroids.shape[0]
    try:
        eng = FitEngine(
            dim, sub.cell_size, np.array([0, n], dtype=np.int64),
            nat.to_dev(np.asarray(sub.centroids, dtype=float).reshape(-1)),
            nat.to_dev(np.asarray(sub.values, dtype=float)),
            np.asarray(sub.box.lo, dtype=float)[None, :], np.asarray(sub.box.hi, dtype=float)[None, :],
            [config], init_centres=initial.centers, init_widths=initial.widths,
            init_gens=initial.generations, init_m=np.array([len(initial)]),
            row_perm=rcb_permutation(np.asarray(sub.centroids, dtype=float)),
        )
        res = eng.run()
    except EngineError as exc:
        raise exc.exc from None
    d = RbfDictionary(centers=res.centres[0], widths=res.widths[0], generations=res.generations[0])
    surrogate = LocalSurrogate(dictionary=d, beta=res.beta[0], log_transform=True)
    return surrogate, reports_for(res, 0, RoundReport)


def fit_subdomains(packed, budget_bytes=None):
    """Batched ``fit_adaptive`` over many independent subdomains on the GPU.

    ``packed`` carries dim, row_off, points, values, box_lo, box_hi, dict_m,
    centres, widths, cell_size and config (one AdaptiveConfig or a list), e.g.
    ``workloads.PackedSubdomains``.  Returns an ``engine.EngineResult``
    (per-subdomain dictionaries, beta, and per-round records).
    """
    from .engine import fit_packed

    return fit_packed(packed.dim, packed.row_off, packed.points, packed.values, packed.box_lo,
                      packed.box_hi, packed.config, packed.dict_m, packed.centres, packed.widths,
                      packed.cell_size, gens=getattr(packed, "generations", None), budget=budget_bytes)
