"""Device-resident batched adaptive fit engine (the B200 replacement of
``fit_parallel``'s per-subdomain task loop, reference partition.py:185-198,
and of ``fit_adaptive``'s round loop, adaptive.py:213-271).

One ``FitEngine`` holds a ragged batch of subdomain fit problems in HBM and
runs every adaptive round for all of them at once:

    K1  pam_assemble_f64   Shepard design matrices, column-major, capacity-strided
    K2b pam_cd_f64         batched cyclic CD (warm-started), one warp per fit
    K3  pam_residual_f64   residual indicators + L2 misfit parts + max R
    K3c pam_mark_f64       stable top-K marking
    K3d pam_enrich_f64     parent search, candidates, duplicate test, append

The host only reads a few per-subdomain scalars per round (max R, misfit
parts, objective, marked/added counts) to apply the reference's stop rules
in the reference's order (adaptive.py:252-266) and to build the
RoundReports.  Results are independent of batch composition and order.

HBM layout (per chunk of subdomains):
  pts (sum N_s, dim), values/y (sum N_s): rows of subdomain s contiguous,
      ascending global cell index;
  centres (sum cap_s, dim), widths, gens, beta (sum cap_s): dictionary slots
      reserved up to cap_s = M0_s + max additions (append-only growth);
  W: per subdomain an (ld_s x cap_s) column-major block, ld_s = N_s rounded
      up to 16 doubles (128-B aligned columns for the TMA bulk copies).
"""

from __future__ import annotations

import contextlib
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as nat


def _round16(n):
    return (np.asarray(n, dtype=np.int64) + 15) // 16 * 16


@dataclass
class RoundRecord:
    round: int
    centers: np.ndarray  # (S,) int
    added: np.ndarray  # (S,) int
    max_residual: np.ndarray  # (S,) float
    rel_l2: np.ndarray
    abs_l2: np.ndarray
    objective: np.ndarray
    sweeps: np.ndarray
    converged: np.ndarray
    seconds: float
    ran: np.ndarray  # (S,) bool: subdomain produced a report this round
    stream_doubles: np.ndarray = None  # (S,) design-matrix doubles the CD streams per sweep
    cd_seconds: float = 0.0  # device time of this round's CD launch (CUDA events)


@dataclass
class EngineResult:
    m_final: np.ndarray  # (S,)
    centres: list  # per subdomain (M_s, dim)
    widths: list
    generations: list
    beta: list
    rounds: list  # list[RoundRecord]
    seconds: float
    kernel_seconds: dict = field(default_factory=dict)


class EngineError(Exception):
    """A data error attributed to one subdomain of the batch."""

    def __init__(self, subdomain: int, exc: Exception):
        super().__init__(str(exc))
        self.subdomain = subdomain
        self.exc = exc


def _config_arrays(configs, n_rows, dim):
    """Per-subdomain parameter arrays from AdaptiveConfig objects."""
    S = len(configs)
    lam1 = np.array([c.elastic.lam1 for c in configs], dtype=np.float64)
    lam2 = np.array([c.elastic.lam2 for c in configs], dtype=np.float64)
    tol = np.array([c.elastic.tol for c in configs], dtype=np.float64)
    max_iters = np.array([c.elastic.max_iters for c in configs], dtype=np.int64)
    if np.any(max_iters > np.iinfo(np.int32).max):
        raise NotImplementedError("max_iters above 2^31-1 is outside the kernel envelope")
    k_top = np.minimum(np.array([c.k_top for c in configs], dtype=np.int64), n_rows)
    m_max = np.array([c.m_max for c in configs], dtype=np.int64)
    eps_tol = np.array([c.eps_tol for c in configs], dtype=np.float64)
    eta = np.array([c.eta for c in configs], dtype=np.float64)
    m_q = np.array([c.m_q for c in configs], dtype=np.int64)
    max_rounds = np.array([c.max_rounds for c in configs], dtype=np.int64)
    quad = np.array([c.quad_order for c in configs], dtype=np.int64)
    if np.any((quad != 1) & (quad != 2)):
        bad = int(np.argmax((quad != 1) & (quad != 2)))
        raise EngineError(bad, ValueError(f"unsupported quadrature order {quad[bad]} (use 1 or 2)"))
    mq_cap = int(m_q.max()) if S else 1
    offsets = np.zeros((S, mq_cap, dim))
    off_err = [None] * S
    cache = {}
    for s, c in enumerate(configs):
        key = (c.offsets, c.m_q)
        if key not in cache:
            try:
                off = np.asarray(c.offsets_for_dim(dim), dtype=float)[: c.m_q]
                # the reference broadcasts x_t + off * scale (adaptive.py:199)
                off = np.broadcast_to(off, (off.shape[0], dim)) if off.ndim == 2 else None
                if off is None:
                    raise ValueError("offsets must be a sequence of per-axis tuples")
                cache[key] = (np.array(off), None)
            except ValueError as exc:
                cache[key] = (None, exc)
        off, exc = cache[key]
        if exc is not None:
            off_err[s] = exc
        else:
            offsets[s, : off.shape[0]] = off
    return dict(lam1=lam1, lam2=lam2, tol=tol, max_iters=max_iters, k_top=k_top, m_max=m_max,
                eps_tol=eps_tol, eta=eta, m_q=m_q, max_rounds=max_rounds, quad=quad,
                offsets=offsets, mq_cap=mq_cap, off_err=off_err)


def dictionary_capacity(m0, k_top, m_q, m_max, max_rounds):
    """Largest dictionary the reference loop can reach (adaptive.py:254-269).

    Enrichment only runs while added < m_max and adds <= k_top*m_q per round,
    for at most max_rounds-1 rounds.
    """
    m0 = np.asarray(m0, dtype=np.int64)
    per = np.asarray(k_top, dtype=np.int64) * np.asarray(m_q, dtype=np.int64)
    m_max = np.asarray(m_max, dtype=np.int64)
    extra = np.minimum((np.asarray(max_rounds, dtype=np.int64) - 1) * per, np.maximum(m_max - 1, 0) + per)
    extra = np.where(m_max > 0, extra, 0)
    return m0 + extra


# Tiles (32 rows) whose Shepard weights are all below tau are not streamed by
# the CD.  Every row of W sums to 1, so 1e-16 is below the FP64 unit roundoff
# (1.1e-16) of each row's mass; zeroing every entry below it moves the
# reference's adaptive fits by ~1e-13 relative (tests/test_oracle_pins.py,
# DESIGN.md §3).  Dropping is used only when every fit of the batch has
# lam1 > 0: a column whose kept part is empty then gets beta = 0 exactly as in
# the reference (|z| <= tau * sum|r| < lam1), while an unregularised fit
# (lam1 = 0) of such a column divides by a vanishing col_sq + lam2 and must
# see every entry.  tile_tau = 2^-100 keeps the exactly-invisible
# threshold, 0 the dense stream.
DEFAULT_TILE_TAU = 1e-16

CD_KERNELS = {"auto": 0, "lean": 1, "dual": 2, "pair": 3, "block": 4}


@dataclass(frozen=True)
class EngineOptions:
    """Implementation choices of the device fit (results agree to ~1e-12).

    cd_form: "auto" | "residual" | "gram" (engine.cd_form); tile_tau: tile-drop
    threshold of the packed CD stream (0 = dense); cd_kernel: "auto" | "lean"
    | "dual" | "pair" | "block" (pam_cd_tiles_f64 kernel selection); w_budget_gb: HBM
    budget of one device batch (None = 60 % of free memory).
    """

    cd_form: str = "auto"
    tile_tau: float = DEFAULT_TILE_TAU
    cd_kernel: str = "auto"
    w_budget_gb: float | None = None


OPTIONS = EngineOptions()


@contextlib.contextmanager
def options(**kw):
    """Temporarily override engine options: ``with options(cd_form="residual"): ...``"""
    global OPTIONS
    old = OPTIONS
    if "cd_kernel" in kw and kw["cd_kernel"] not in CD_KERNELS:
        raise ValueError(f"unknown cd_kernel {kw['cd_kernel']!r}")
    if "cd_form" in kw and kw["cd_form"] not in ("auto", "residual", "gram"):
        raise ValueError(f"unknown cd_form {kw['cd_form']!r}")
    OPTIONS = replace(old, **kw)
    try:
        yield OPTIONS
    finally:
        OPTIONS = old


def set_options(**kw):
    """Set engine options for the rest of the process (bench.py flags)."""
    global OPTIONS
    OPTIONS = replace(OPTIONS, **kw)


def tile_tau() -> float:
    """Tile-drop threshold for the packed CD stream (0 = dense)."""
    return float(OPTIONS.tile_tau)


def rcb_permutation(points: np.ndarray, leaf: int = 32) -> np.ndarray:
    """Recursive coordinate bisection order of one subdomain's sample points.

    Splits along the longest physical extent at a multiple of `leaf` near the
    median, so every 32-row tile of the CD stream is a compact blob of cells
    and a narrow Gaussian column touches few tiles.  Deterministic (stable
    sorts).  Only the CD's row order changes; results are order-independent
    up to FP64 rounding of the dot products.
    """
    pts = np.asarray(points, dtype=np.float64)
    n = pts.shape[0]
    out = np.empty(n, dtype=np.int64)
    pos = 0
    stack = [np.arange(n)]
    while stack:
        ids = stack.pop()
        if ids.size <= leaf:
            out[pos:pos + ids.size] = ids
            pos += ids.size
            continue
        p = pts[ids]
        ax = int(np.argmax(p.max(axis=0) - p.min(axis=0)))
        o = ids[np.argsort(p[:, ax], kind="stable")]
        half = min(max(((ids.size // 2 + leaf - 1) // leaf) * leaf, leaf), ids.size - 1)
        stack.append(o[half:])  # LIFO: the lower half is emitted first
        stack.append(o[:half])
    return out


GRAM_MAX_M = 512
GRAM_WIDE_MAX_M = 3072  # covariance form for few-fit batches (gram.cu wide configurations)


def _sm_count() -> int:
    try:
        torch = nat.torch_mod()
        if torch.cuda.is_available():
            return int(torch.cuda.get_device_properties(0).multi_processor_count)
    except Exception:  # noqa: BLE001 - host-only use (tests): B200's count
        pass
    return 148


def cd_form(n_rows, cap, tiles_ok: bool = True) -> str:
    """Which CD formulation is faster for this batch.

    Residual form streams N*M doubles per sweep, the covariance (Gram) form
    M*M (hard part 1).  Many fits: the form that streams fewer
    bytes (Gram needs M <= 512 and cap <= 0.75 N).  Few fits (at most one per
    SM, e.g. BASELINE config 2, the Table-2 run): with the tile-packed stream
    (``tiles_ok``: <= 1024 rows, lam1 > 0, tau > 0) the exact blocked CD
    (cd_block.cu) wins (C2 6.7 s vs 8.3 s, Table-2 9.8 s vs 19.8 s measured);
    otherwise the per-column chain of the dense residual kernels (~0.55 us)
    loses to the covariance form's (~0.12 us per coordinate) whenever its M*M
    stream still fits the HBM time (M <= 3072).  OPTIONS.cd_form forces one form.
    """
    forced = OPTIONS.cd_form
    cap = np.asarray(cap, dtype=np.int64)
    cmax = int(cap.max())
    if forced == "gram" and cmax <= GRAM_WIDE_MAX_M:
        return "gram"
    if forced == "residual":
        return "residual"
    if cmax <= GRAM_MAX_M and np.all(cap * 4 <= np.asarray(n_rows) * 3):
        return "gram"
    if cap.size <= _sm_count() and tiles_ok and int(np.max(n_rows)) <= 1024:
        return "residual"
    if cap.size <= _sm_count() and cmax <= GRAM_WIDE_MAX_M:
        t_res = cmax * 0.55e-6                                   # per sweep, chain-bound
        t_gram = max(cmax * 0.12e-6, float(np.sum(cap.astype(np.float64) ** 2)) * 8 / 6.5e12)
        if t_gram < 0.7 * t_res:
            return "gram"
    return "residual"


def device_bytes(n_rows, cap) -> np.ndarray:
    """Per-subdomain HBM for design matrices (+ Gram matrices) in one device batch."""
    n_rows = np.asarray(n_rows, dtype=np.int64)
    cap = np.asarray(cap, dtype=np.int64)
    w = (n_rows + 31) // 32 * 32 * cap * 8
    return w + np.where(cap <= GRAM_MAX_M, _round16(cap) * cap * 8, 0)


def estimate_w_bytes(n_rows, cap):
    return int(np.sum(_round16(n_rows) * np.asarray(cap, dtype=np.int64)) * 8)


class FitEngine:
    """Ragged batch of adaptive subdomain fits resident on one GPU."""

    def __init__(self, dim, cell_size, row_off, pts, values, box_lo, box_hi, configs,
                 init_centres=None, init_widths=None, init_gens=None, init_m=None,
                 centroid_sigma=None, row_perm=None, tau=None):
        """
        row_off: host int64 (S+1,); pts/values: device tensors (rows packed);
        box_lo/box_hi: host (S, dim).  The initial dictionary is either the
        per-cell centroid dictionary (``centroid_sigma``: (S,) widths,
        DictionarySpec(lattice=None), partition.py:109-111) or explicit packed
        host arrays (init_centres (sum M0, dim), init_widths, init_gens,
        init_m (S,)).  ``row_perm`` (host, packed like the rows: local row
        index per CD position) orders the CD stream; default identity.
        ``tau`` > 0 enables the tile-packed CD stream (tiles.cu) for batches
        of <= 1024 rows per subdomain; 0 streams the dense design matrix.
        """
        torch = nat.torch_mod()
        self.torch = torch
        self.dev = nat.device()
        self.dim = int(dim)
        self.S = S = len(configs)
        self.row_off = np.asarray(row_off, dtype=np.int64)
        self.n_rows = np.diff(self.row_off)
        if np.any(self.n_rows < 1):
            bad = int(np.argmax(self.n_rows < 1))
            raise EngineError(bad, ValueError("subdomain box contains no cell centroids"))
        self.max_rows = int(self.n_rows.max())
        if self.max_rows > nat.lib().pam_cd_max_rows():
            raise NotImplementedError(
                f"a subdomain has {self.max_rows} cells; the CD kernels take at most "
                f"{nat.lib().pam_cd_max_rows()} rows per subdomain"
            )
        self.cell_size = np.asarray(cell_size, dtype=np.float64)
        self.p = _config_arrays(configs, self.n_rows, self.dim)
        p = self.p

        # ---- initial dictionary sizes and capacities
        if centroid_sigma is not None:
            m0 = self.n_rows.copy()
        else:
            m0 = np.asarray(init_m, dtype=np.int64)
        self.cap = dictionary_capacity(m0, p["k_top"], p["m_q"], p["m_max"], p["max_rounds"])
        self.dict_off = np.concatenate([[0], np.cumsum(self.cap)[:-1]]).astype(np.int64)
        cap_tot = int(self.cap.sum())
        tau0 = tile_tau() if tau is None else float(tau)
        self.form = cd_form(self.n_rows, self.cap, tiles_ok=tau0 > 0 and bool(np.all(p["lam1"] > 0)))
        # the device column stream (prologue + sweeps) is counted in 32 bits
        if np.any(self.cap * (1 + p["max_iters"]) >= 2**31):
            raise NotImplementedError("dictionary capacity x (max_iters + 1) >= 2^31 is outside the "
                                      "CD kernel envelope")
        self.tau = tile_tau() if tau is None else float(tau)
        if S and not np.all(p["lam1"] > 0):
            self.tau = 0.0  # unregularised fits see every entry (see DEFAULT_TILE_TAU)
        self.tiles = self.form == "residual" and self.tau > 0.0 and self.max_rows <= 1024
        self.cd_kernel = CD_KERNELS[OPTIONS.cd_kernel]
        self.ld = _round16(self.n_rows) if not self.tiles else (self.n_rows + 31) // 32 * 32
        wsz = self.ld * self.cap
        self.w_off = np.concatenate([[0], np.cumsum(wsz)[:-1]]).astype(np.int64)
        self.w_total = int(wsz.sum())

        t = torch
        dev = self.dev
        f64, i64, i32 = t.float64, t.int64, t.int32
        self.d_row_off = nat.to_dev(self.row_off)
        self.d_pts = pts
        self.d_values = values
        self.d_dict_off = nat.to_dev(self.dict_off)
        self.d_dict_cap = nat.to_dev(self.cap.astype(np.int32))
        self.d_w_off = nat.to_dev(self.w_off)
        self.d_ld = nat.to_dev(self.ld.astype(np.int32))
        self.d_centres = t.empty(cap_tot * self.dim, dtype=f64, device=dev)
        self.d_widths = t.empty(cap_tot, dtype=f64, device=dev)
        self.d_gens = t.empty(cap_tot, dtype=i32, device=dev)
        self.d_beta = t.zeros(cap_tot, dtype=f64, device=dev)
        self.d_col_sq = t.empty(cap_tot, dtype=f64, device=dev)
        self.d_W = t.empty(self.w_total, dtype=f64, device=dev)
        ntot = int(self.row_off[-1])
        self.d_y = t.empty(ntot, dtype=f64, device=dev)
        self.d_R = t.empty(ntot, dtype=f64, device=dev)
        self.d_parts = t.empty(2 * S, dtype=f64, device=dev)
        self.d_rmax = t.empty(S, dtype=f64, device=dev)
        self.d_sweeps = t.zeros(S, dtype=i32, device=dev)
        self.d_conv = t.zeros(S, dtype=i32, device=dev)
        self.d_obj = t.zeros(S, dtype=f64, device=dev)
        self.kcap = max(1, int(p["k_top"].max()))
        self.d_marked = t.zeros(S * self.kcap, dtype=i32, device=dev)
        self.d_nmarked = t.zeros(S, dtype=i32, device=dev)
        self.d_nadded = t.zeros(S, dtype=i32, device=dev)
        self.d_active = t.ones(S, dtype=i32, device=dev)
        self.d_lam1 = nat.to_dev(p["lam1"])
        self.d_lam2 = nat.to_dev(p["lam2"])
        self.d_tol = nat.to_dev(p["tol"])
        self.d_max_iters = nat.to_dev(p["max_iters"].astype(np.int32))
        self.d_ktop = nat.to_dev(p["k_top"].astype(np.int32))
        self.d_eta = nat.to_dev(p["eta"])
        self.d_mq = nat.to_dev(p["m_q"].astype(np.int32))
        self.d_quad = nat.to_dev(p["quad"].astype(np.int32))
        self.d_offsets = nat.to_dev(p["offsets"].reshape(-1))
        self.d_cell_size = nat.to_dev(self.cell_size)
        self.d_box_lo = nat.to_dev(np.asarray(box_lo, dtype=np.float64).reshape(-1))
        self.d_box_hi = nat.to_dev(np.asarray(box_hi, dtype=np.float64).reshape(-1))
        from .geometry import quadrature_offsets

        q1o, q1w = quadrature_offsets(self.cell_size, 1)
        q2o, q2w = quadrature_offsets(self.cell_size, 2)
        self.d_qoff = nat.to_dev(np.concatenate([q1o, q2o]).reshape(-1))
        self.d_qw = nat.to_dev(np.concatenate([q1w, q2w]))
        self.err = nat.ErrorWord()
        self.d_work = t.zeros(int(nat.lib().pam_cd_workspace_bytes(
            S, ntot, cap_tot, self.max_rows, self.cd_kernel if self.tiles else 0)), dtype=t.uint8, device=dev)
        if self.form == "gram":
            self.ldg = _round16(self.cap)
            gsz = self.ldg * self.cap
            self.g_off = np.concatenate([[0], np.cumsum(gsz)[:-1]]).astype(np.int64)
            self.d_G = t.empty(int(gsz.sum()), dtype=f64, device=dev)
            self.d_g_off = nat.to_dev(self.g_off)
            self.d_ldg = nat.to_dev(self.ldg.astype(np.int32))
            self.d_q = t.empty(cap_tot, dtype=f64, device=dev)
            self.d_zero_iters = t.zeros(S, dtype=i32, device=dev)
            self.d_obj_sweeps = t.zeros(S, dtype=i32, device=dev)
            self.d_obj_conv = t.zeros(S, dtype=i32, device=dev)
            self.d_obj_colsq = t.empty(cap_tot, dtype=f64, device=dev)
        if self.tiles:
            self.d_perm = None if row_perm is None else nat.to_dev(np.asarray(row_perm, dtype=np.int32))
            self.d_rowmax = t.empty(ntot, dtype=f64, device=dev)
            self.d_rowsum = t.empty(ntot, dtype=f64, device=dev)
            self.d_tile_mask = t.zeros(cap_tot, dtype=i64, device=dev)
            self.d_col_off = t.zeros(cap_tot, dtype=i64, device=dev)
            self.d_packed = t.zeros(S, dtype=i64, device=dev)

        # ---- initial dictionary into the capacity slots (one device scatter)
        self.m_cur = m0.copy()
        if centroid_sigma is not None:
            # per-cell dictionary: the gathered sample points themselves
            d_sigma = nat.to_dev(np.asarray(centroid_sigma, dtype=np.float64))
            nat.check(nat.lib().pam_dict_scatter_f64(
                self.dim, S, nat.ptr(self.d_row_off), nat.ptr(pts), None, nat.ptr(d_sigma), None,
                nat.ptr(self.d_dict_off), nat.ptr(self.d_centres), nat.ptr(self.d_widths), nat.ptr(self.d_gens),
                nat.stream_ptr()), "pam_dict_scatter_f64")
        else:
            src_off = nat.to_dev(np.concatenate([[0], np.cumsum(m0)]).astype(np.int64))
            d_c = nat.to_dev(np.asarray(init_centres, dtype=np.float64).reshape(-1))
            d_w = nat.to_dev(np.asarray(init_widths, dtype=np.float64))
            d_g = None if init_gens is None else nat.to_dev(np.asarray(init_gens, dtype=np.int32))
            nat.check(nat.lib().pam_dict_scatter_f64(
                self.dim, S, nat.ptr(src_off), nat.ptr(d_c), nat.ptr(d_w), None, nat.ptr(d_g),
                nat.ptr(self.d_dict_off), nat.ptr(self.d_centres), nat.ptr(self.d_widths), nat.ptr(self.d_gens),
                nat.stream_ptr()), "pam_dict_scatter_f64")
        self.d_m_cur = nat.to_dev(self.m_cur.astype(np.int32))

    # ------------------------------------------------------------------
    def _sync_err(self, what):
        code, idx = self.err.read()
        if code:
            s = int(np.searchsorted(self.row_off, idx, side="right") - 1) if code in (
                nat.PAM_ERR_NONPOSITIVE, nat.PAM_ERR_DEGENERATE) else int(idx)
            local = idx - int(self.row_off[s]) if code == nat.PAM_ERR_NONPOSITIVE else idx
            try:
                nat.raise_data_error(code, local)
            except Exception as exc:  # noqa: BLE001 - attribute to the subdomain
                raise EngineError(s, exc) from exc

    def run(self, timers=None) -> EngineResult:
        torch = self.torch
        lib = nat.lib()
        p = self.p
        S, dim = self.S, self.dim
        st = nat.stream_ptr()
        P = nat.ptr
        t_start = time.perf_counter()

        # y = log(values) with the positivity check (elastic_net.py:197-205)
        nat.check(lib.pam_log_values_f64(P(self.d_values), int(self.row_off[-1]), P(self.d_y),
                                         P(self.err.t), st), "pam_log_values_f64")
        self._sync_err("log")

        active = np.ones(S, dtype=bool)
        added_total = np.zeros(S, dtype=np.int64)
        rounds = []
        kt = {"assemble": 0.0, "cd": 0.0, "residual": 0.0, "mark_enrich": 0.0}
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        max_rounds = int(p["max_rounds"].max())
        for rnd in range(max_rounds):
            t0 = time.perf_counter()
            idx = np.flatnonzero(active)
            self.d_active.copy_(torch.from_numpy(active.astype(np.int32)))
            # longest fits first: balances the ragged batch across warps
            work = self.n_rows * self.m_cur
            order = idx[np.argsort(-work[idx], kind="stable")]
            d_order = nat.to_dev(order.astype(np.int64))
            e0, e1, e2, e3 = ev(), ev(), ev(), ev()
            e0.record()
            if self.tiles:
                nat.check(lib.pam_assemble_tiles_f64(
                    dim, S, P(self.d_row_off), P(self.d_pts), P(self.d_perm), P(self.d_dict_off),
                    P(self.d_m_cur), P(self.d_centres), P(self.d_widths), P(self.d_w_off),
                    P(self.d_active), self.max_rows, self.tau, P(self.d_rowmax), P(self.d_rowsum),
                    P(self.d_tile_mask), P(self.d_col_off), P(self.d_packed), int(self.cap.sum()),
                    P(self.d_W), st), "pam_assemble_tiles_f64")
            else:
                nat.check(lib.pam_assemble_f64(
                    dim, S, P(self.d_row_off), P(self.d_pts), P(self.d_dict_off), P(self.d_m_cur),
                    P(self.d_centres), P(self.d_widths), P(self.d_w_off), P(self.d_ld), P(self.d_active),
                    self.max_rows, 0, P(self.d_W), st), "pam_assemble_f64")
            e1.record()
            if self.form == "gram":
                max_m = int(self.m_cur.max())
                nat.check(lib.pam_gram_f64(
                    S, P(self.d_row_off), P(self.d_m_cur), P(self.d_dict_off), P(self.d_w_off),
                    P(self.d_ld), P(self.d_g_off), P(self.d_ldg), P(self.d_active), max_m, P(self.d_W),
                    P(self.d_y), P(self.d_G), P(self.d_q), P(self.d_col_sq), st), "pam_gram_f64")
                nat.check(lib.pam_cd_gram_f64(
                    len(order), P(d_order), P(self.d_dict_off), P(self.d_m_cur), P(self.d_g_off),
                    P(self.d_ldg), P(self.d_G), P(self.d_q), P(self.d_col_sq), P(self.d_lam1),
                    P(self.d_lam2), P(self.d_tol), P(self.d_max_iters), P(self.d_active), max_m,
                    P(self.d_beta), P(self.d_sweeps), P(self.d_conv), P(self.d_work), st), "pam_cd_gram_f64")
                # exact objective at the final beta: residual form with zero sweeps
                nat.check(lib.pam_cd_f64(
                    len(order), P(d_order), P(self.d_row_off), P(self.d_y), P(self.d_dict_off),
                    P(self.d_m_cur), P(self.d_w_off), P(self.d_ld), P(self.d_W), P(self.d_lam1),
                    P(self.d_lam2), P(self.d_tol), P(self.d_zero_iters), P(self.d_active),
                    self.max_rows, P(self.d_beta), P(self.d_obj_colsq), P(self.d_obj_sweeps),
                    P(self.d_obj_conv), P(self.d_obj), None, None, P(self.d_work), st), "pam_cd_f64")
            elif self.tiles:
                nat.check(lib.pam_cd_tiles_f64(
                    len(order), P(d_order), P(self.d_row_off), P(self.d_y), P(self.d_perm),
                    P(self.d_dict_off), P(self.d_m_cur), P(self.d_w_off), P(self.d_tile_mask),
                    P(self.d_col_off), P(self.d_W), P(self.d_lam1), P(self.d_lam2), P(self.d_tol),
                    P(self.d_max_iters), P(self.d_active), self.max_rows, int(self.m_cur.max()),
                    P(self.d_beta), P(self.d_col_sq), P(self.d_sweeps), P(self.d_conv), P(self.d_obj), None,
                    None, self.cd_kernel, P(self.d_work), st), "pam_cd_tiles_f64")
            else:
                nat.check(lib.pam_cd_f64(
                    len(order), P(d_order), P(self.d_row_off), P(self.d_y), P(self.d_dict_off),
                    P(self.d_m_cur), P(self.d_w_off), P(self.d_ld), P(self.d_W), P(self.d_lam1),
                    P(self.d_lam2), P(self.d_tol), P(self.d_max_iters), P(self.d_active), self.max_rows,
                    P(self.d_beta), P(self.d_col_sq), P(self.d_sweeps), P(self.d_conv), P(self.d_obj),
                    None, None, P(self.d_work), st), "pam_cd_f64")
            e2.record()
            nat.check(lib.pam_residual_f64(
                dim, S, P(self.d_row_off), P(self.d_pts), P(self.d_values), P(self.d_dict_off),
                P(self.d_m_cur), P(self.d_centres), P(self.d_widths), P(self.d_beta),
                P(self.d_quad), P(self.d_qoff), P(self.d_qw), 1, P(self.d_active), self.max_rows,
                P(self.d_R), P(self.d_parts), P(self.d_rmax), P(self.err.t), st), "pam_residual_f64")
            e3.record()
            # small per-subdomain scalars back to the host (one sync per round)
            rmax = self.d_rmax.cpu().numpy()
            parts = self.d_parts.cpu().numpy().reshape(S, 2)
            obj = self.d_obj.cpu().numpy()
            sweeps = self.d_sweeps.cpu().numpy()
            conv = self.d_conv.cpu().numpy()
            if self.form == "gram":
                stream_doubles = self.m_cur * self.m_cur  # one G column per coordinate
            elif self.tiles:
                stream_doubles = self.d_packed.cpu().numpy()
            else:
                stream_doubles = self.n_rows * self.m_cur
            self._sync_err("residual")
            kt["assemble"] += e0.elapsed_time(e1) / 1e3
            kt["cd"] += e1.elapsed_time(e2) / 1e3
            kt["residual"] += e2.elapsed_time(e3) / 1e3
            num, den = parts[:, 0], parts[:, 1]
            with np.errstate(divide="ignore", invalid="ignore"):
                rel = np.sqrt(num / den)
            rec = RoundRecord(
                round=rnd, centers=self.m_cur.copy(), added=added_total.copy(), max_residual=rmax,
                rel_l2=rel, abs_l2=np.sqrt(num), objective=obj, sweeps=sweeps,
                converged=conv.astype(bool), seconds=0.0, ran=active.copy(),
                stream_doubles=np.asarray(stream_doubles, dtype=np.int64).copy(),
                cd_seconds=e1.elapsed_time(e2) / 1e3,
            )
            # stop rules in the reference's order (adaptive.py:252-260)
            stop = (rmax < p["eps_tol"]) | (added_total >= p["m_max"]) | (rnd == p["max_rounds"] - 1)
            cont = active & ~stop
            if cont.any():
                bad = [s for s in np.flatnonzero(cont) if p["off_err"][s] is not None]
                if bad:
                    raise EngineError(int(bad[0]), p["off_err"][bad[0]])
                e4, e5 = ev(), ev()
                e4.record()
                self.d_active.copy_(torch.from_numpy(cont.astype(np.int32)))
                nat.check(lib.pam_mark_f64(
                    S, P(self.d_row_off), P(self.d_R), P(self.d_ktop), P(self.d_active), self.kcap,
                    P(self.d_marked), P(self.d_nmarked), st), "pam_mark_f64")
                n_marked = self.d_nmarked.cpu().numpy()
                cont &= n_marked > 0
                if cont.any():
                    self.d_active.copy_(torch.from_numpy(cont.astype(np.int32)))
                    nat.check(lib.pam_enrich_f64(
                        dim, S, P(self.d_row_off), P(self.d_pts), P(self.d_marked), P(self.d_nmarked),
                        self.kcap, P(self.d_eta), P(self.d_mq), p["mq_cap"], P(self.d_offsets),
                        P(self.d_cell_size), P(self.d_box_lo), P(self.d_box_hi), P(self.d_dict_off),
                        P(self.d_dict_cap), P(self.d_m_cur), P(self.d_centres), P(self.d_widths),
                        P(self.d_gens), P(self.d_beta), rnd + 1, P(self.d_active), P(self.d_nadded),
                        P(self.err.t), st), "pam_enrich_f64")
                    n_added = self.d_nadded.cpu().numpy().astype(np.int64)
                    self._sync_err("enrich")
                    n_added = np.where(cont, n_added, 0)
                    cont &= n_added > 0
                    added_total += n_added
                    self.m_cur = self.m_cur + n_added
                e5.record()
                torch.cuda.current_stream().synchronize()
                kt["mark_enrich"] += e4.elapsed_time(e5) / 1e3
            rec.seconds = time.perf_counter() - t0
            rounds.append(rec)
            active = cont
            if not active.any():
                break
        # ---- results back to the host
        m_final = self.d_m_cur.cpu().numpy().astype(np.int64)
        cen = self.d_centres.view(-1, dim).cpu().numpy()
        wid = self.d_widths.cpu().numpy()
        gen = self.d_gens.cpu().numpy()
        bet = self.d_beta.cpu().numpy()
        out_c, out_w, out_g, out_b = [], [], [], []
        for s in range(S):
            a, b = int(self.dict_off[s]), int(self.dict_off[s] + m_final[s])
            out_c.append(cen[a:b])
            out_w.append(wid[a:b])
            out_g.append(gen[a:b])
            out_b.append(bet[a:b])
        return EngineResult(m_final=m_final, centres=out_c, widths=out_w, generations=out_g,
                            beta=out_b, rounds=rounds, seconds=time.perf_counter() - t_start,
                            kernel_seconds=kt)

    def release(self):
        for k in list(vars(self)):
            if k.startswith("d_"):
                setattr(self, k, None)


def reports_for(result: EngineResult, s: int, report_cls):
    """RoundReports of subdomain s in the reference's field order (adaptive.py:239-250)."""
    out = []
    for rec in result.rounds:
        if not rec.ran[s]:
            continue
        out.append(report_cls(
            round=rec.round,
            centers=int(rec.centers[s]),
            added=int(rec.added[s]),
            max_residual=float(rec.max_residual[s]),
            rel_l2=float(rec.rel_l2[s]),
            abs_l2=float(rec.abs_l2[s]),
            objective=float(rec.objective[s]),
            seconds=float(rec.seconds),
        ))
    return out


def w_budget_bytes() -> int:
    """HBM budget for one chunk's design matrices (OPTIONS.w_budget_gb overrides)."""
    if OPTIONS.w_budget_gb is not None:
        return int(float(OPTIONS.w_budget_gb) * 2**30)
    torch = nat.torch_mod()
    free, _total = torch.cuda.mem_get_info()
    return int(free * 0.6)


def chunk_ranges(wbytes_per_sub: np.ndarray, budget: int):
    """Consecutive subdomain ranges whose W fits the budget."""
    out, start, acc = [], 0, 0
    for s, b in enumerate(wbytes_per_sub):
        if acc and acc + b > budget:
            out.append((start, s))
            start, acc = s, 0
        acc += int(b)
    out.append((start, len(wbytes_per_sub)))
    return out



def _merge_results(parts, offsets):
    """Concatenate per-chunk EngineResults (subdomain order preserved)."""
    if len(parts) == 1:
        return parts[0]
    S = sum(len(p.m_final) for p in parts)
    n_rounds = max(len(p.rounds) for p in parts)
    rounds = []
    for k in range(n_rounds):
        def cat(attr, fill):
            out = []
            for p in parts:
                n = len(p.m_final)
                out.append(getattr(p.rounds[k], attr) if k < len(p.rounds) else np.full(n, fill))
            return np.concatenate(out)
        rounds.append(RoundRecord(
            round=k, centers=cat("centers", 0), added=cat("added", 0),
            max_residual=cat("max_residual", np.nan), rel_l2=cat("rel_l2", np.nan),
            abs_l2=cat("abs_l2", np.nan), objective=cat("objective", np.nan), sweeps=cat("sweeps", 0),
            converged=cat("converged", False), stream_doubles=cat("stream_doubles", 0),
            seconds=float(sum(p.rounds[k].seconds for p in parts if k < len(p.rounds))),
            ran=cat("ran", False),
            cd_seconds=float(sum(p.rounds[k].cd_seconds for p in parts if k < len(p.rounds)))))
    kt = {}
    for p in parts:
        for key, v in p.kernel_seconds.items():
            kt[key] = kt.get(key, 0.0) + v
    res = EngineResult(
        m_final=np.concatenate([p.m_final for p in parts]),
        centres=sum((p.centres for p in parts), []), widths=sum((p.widths for p in parts), []),
        generations=sum((p.generations for p in parts), []), beta=sum((p.beta for p in parts), []),
        rounds=rounds, seconds=float(sum(p.seconds for p in parts)), kernel_seconds=kt)
    assert len(res.m_final) == S
    return res


def fit_packed(dim, row_off, points, values, box_lo, box_hi, configs, dict_m, centres, widths,
               cell_size, gens=None, budget=None) -> EngineResult:
    """Batched adaptive fits of independent subdomains given as packed host arrays.

    The subdomain-level equivalent of calling fit_adaptive(SubdomainField,
    RbfDictionary, AdaptiveConfig) once per subdomain (adaptive.py:213-271),
    used for workloads whose samples are not mesh cells (BASELINE config 5).
    Chunked automatically so each device batch's design matrices fit in HBM.
    """
    row_off = np.asarray(row_off, dtype=np.int64)
    S = row_off.shape[0] - 1
    if not isinstance(configs, (list, tuple)):
        configs = [configs] * S
    dict_m = np.asarray(dict_m, dtype=np.int64)
    m_off = np.concatenate([[0], np.cumsum(dict_m)]).astype(np.int64)
    n_rows = np.diff(row_off)
    k_top = np.minimum([c.k_top for c in configs], n_rows)
    cap = dictionary_capacity(dict_m, k_top, [c.m_q for c in configs], [c.m_max for c in configs],
                              [c.max_rounds for c in configs])
    chunks = chunk_ranges(device_bytes(n_rows, cap), budget or w_budget_bytes())
    points = np.asarray(points, dtype=np.float64).reshape(-1, dim)
    values = np.asarray(values, dtype=np.float64).reshape(-1)
    centres = np.asarray(centres, dtype=np.float64).reshape(-1, dim)
    widths = np.asarray(widths, dtype=np.float64).reshape(-1)
    parts = []
    for a, b in chunks:
        r0, r1 = int(row_off[a]), int(row_off[b])
        m0, m1 = int(m_off[a]), int(m_off[b])
        # the CD row order only matters for the tile-packed stream
        lam1_pos = all(c.elastic.lam1 > 0 for c in configs[a:b])
        use_tiles = (cd_form(n_rows[a:b], cap[a:b], tile_tau() > 0 and lam1_pos) == "residual"
                     and tile_tau() > 0 and lam1_pos
                     and int(n_rows[a:b].max()) <= 1024)
        perm = np.concatenate([rcb_permutation(points[row_off[i]:row_off[i + 1]])
                               for i in range(a, b)]) if use_tiles and b - a <= 16384 else None
        try:
            eng = FitEngine(dim, cell_size, row_off[a:b + 1] - r0, nat.to_dev(points[r0:r1].reshape(-1)),
                            nat.to_dev(values[r0:r1]), np.asarray(box_lo)[a:b], np.asarray(box_hi)[a:b],
                            list(configs[a:b]), init_centres=centres[m0:m1], init_widths=widths[m0:m1],
                            init_gens=None if gens is None else np.asarray(gens)[m0:m1],
                            init_m=dict_m[a:b], row_perm=perm)
            parts.append(eng.run())
        except EngineError as exc:
            raise EngineError(a + exc.subdomain, exc.exc) from exc.exc
        eng.release()
    return _merge_results(parts, chunks)
