"""Multi-GPU sharding of the batched fit.

Subdomains are independent (PAPER §2; reference partition.py:167-208 fans
them out to a process pool), so across GPUs the fit shards with NO
collective on the data path: each rank fits a contiguous range of
subdomains balanced by estimated CD work (N_s · M_s), then the ragged
results (dictionaries + β + reports) are gathered once so every rank holds
the full GlobalSurrogate, identical to the single-process result.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on the GPU
box; the host-side logic is tested with gloo, world_size 2, on CPU).
"""

from __future__ import annotations

import numpy as np


def balanced_ranges(work, world: int):
    """Split [0, S) into `world` contiguous ranges of ~equal total work."""
    w = np.asarray(work, dtype=np.float64)
    S = w.shape[0]
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        bounds.append(min(max(b, bounds[-1]), S))
    bounds.append(S)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def gather_by_index(local: dict, n: int, group=None) -> list:
    """All-gather {subdomain index: item} dicts into one list ordered by index."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        parts = [local]
    else:
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, local, group=group)
    out = [None] * n
    for part in parts:
        for i, item in part.items():
            if out[i] is not None:
                raise RuntimeError(f"subdomain {i} fitted by more than one rank")
            out[i] = item
    missing = [i for i, v in enumerate(out) if v is None]
    if missing:
        raise RuntimeError(f"subdomains {missing[:5]} were not fitted by any rank")
    return out


def estimate_work(n_rows, m0, cap):
    """Per-subdomain CD work proxy: rows x (initial + final) columns."""
    return np.asarray(n_rows, dtype=np.float64) * (np.asarray(m0) + np.asarray(cap)) / 2.0


def fit_parallel_sharded(data, partition, configs, spec, group=None, fit_range=None,
                         metadata=None):
    """Sharded ``fit_parallel``: rank r fits its balanced range, results all-gathered.

    ``fit_range(a, b) -> list[(LocalSurrogate, tuple[RoundReport, ...])]`` does
    the local work; the default runs the device engine on this rank's GPU.
    Returns (GlobalSurrogate, per-subdomain reports) identical on all ranks.
    """
    import torch.distributed as dist

    from .engine import dictionary_capacity
    from .partition import GlobalSurrogate, _broadcast
    from .adaptive import AdaptiveConfig
    from .partition import DictionarySpec

    n = partition.n_subdomains
    cfgs = _broadcast(configs, n, AdaptiveConfig, "configs")
    specs = _broadcast(spec, n, DictionarySpec, "spec")
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n_rows = np.bincount(partition.cell_to_subdomain, minlength=n)
    m0 = np.array([n_rows[i] if sp.lattice is None else sp.lattice ** partition.mesh.dim
                   for i, sp in enumerate(specs)])
    cap = dictionary_capacity(m0, np.minimum([c.k_top for c in cfgs], n_rows), [c.m_q for c in cfgs],
                              [c.m_max for c in cfgs], [c.max_rounds for c in cfgs])
    a, b = balanced_ranges(estimate_work(n_rows, m0, cap), world)[rank]
    if fit_range is None:
        fit_range = _device_fit_range(data, partition, cfgs, specs)
    local = dict(zip(range(a, b), fit_range(a, b))) if b > a else {}
    items = gather_by_index(local, n, group)
    locals_ = tuple(it[0] for it in items)
    reports = tuple(it[1] for it in items)
    meta = dict(metadata or {})
    meta.setdefault("field_checksum", data.checksum())
    return GlobalSurrogate(partition=partition, locals=locals_, metadata=meta), reports


def _device_fit_range(data, partition, cfgs, specs):
    """fit_range backed by the GPU engine: fit_parallel on the sub-box set [a, b)."""

    def run(a, b):
        from .partition import fit_subset

        return fit_subset(data, partition, cfgs, specs, a, b)

    return run
