"""Multi-GPU sharding of the batched fit.

Subdomains are independent (PAPER §2; reference partition.py:167-208 fans
them out to a process pool), so across GPUs the fit shards with NO
collective on the data path: each rank fits a contiguous range of
subdomains balanced by estimated CD work (N_s · M_s), then the ragged
results (dictionaries + β + reports) are gathered once -- a packed
allgatherv: one flat float64 payload per rank, padded, exchanged with
``all_gather_into_tensor`` (NCCL over NVLink/NVSwitch on the GPU box) -- so
every rank holds the full GlobalSurrogate, identical to the single-process
result (reference partition.py:188-198 gathers by index after its pool).

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


REPORT_FIELDS = ("round", "centers", "added", "max_residual", "rel_l2", "abs_l2", "objective", "seconds")


def pack_results(items, dim: int) -> np.ndarray:
    """[(LocalSurrogate, reports)] -> one flat float64 buffer (allgatherv payload).

    Layout: [count, then per item (M, n_rounds, log_transform)] + centres (sum M x dim)
    + widths + beta + generations + reports (8 values per round, REPORT_FIELDS).
    Integers are carried exactly (|v| < 2^53).
    """
    head = [float(len(items))]
    cen, wid, bet, gen, rep = [], [], [], [], []
    for loc, reps in items:
        d = loc.dictionary
        head += [float(len(d)), float(len(reps)), float(bool(loc.log_transform))]
        cen.append(np.asarray(d.centers, dtype=np.float64).reshape(-1))
        wid.append(np.asarray(d.widths, dtype=np.float64))
        bet.append(np.asarray(loc.beta, dtype=np.float64))
        gen.append(np.asarray(d.generations, dtype=np.float64))
        rep.append(np.array([[float(getattr(r, f)) for f in REPORT_FIELDS] for r in reps],
                            dtype=np.float64).reshape(-1))
    parts = [np.asarray(head)] + cen + wid + bet + gen + rep
    return np.concatenate(parts) if parts else np.zeros(1)


def unpack_results(buf: np.ndarray, dim: int):
    """Inverse of pack_results -> [(LocalSurrogate, tuple[RoundReport])]."""
    from .adaptive import RoundReport
    from .rbf import LocalSurrogate, RbfDictionary

    n = int(buf[0])
    meta = buf[1:1 + 3 * n].reshape(n, 3).astype(np.int64)
    m = meta[:, 0]
    pos = 1 + 3 * n
    tot = int(m.sum())
    cen = buf[pos:pos + tot * dim].reshape(tot, dim)
    pos += tot * dim
    wid = buf[pos:pos + tot]
    pos += tot
    bet = buf[pos:pos + tot]
    pos += tot
    gen = buf[pos:pos + tot].astype(np.int64)
    pos += tot
    out, o = [], 0
    for k in range(n):
        mk, rk, lf = int(m[k]), int(meta[k, 1]), bool(meta[k, 2])
        d = RbfDictionary(centers=cen[o:o + mk], widths=wid[o:o + mk], generations=gen[o:o + mk])
        loc = LocalSurrogate(dictionary=d, beta=bet[o:o + mk].copy(), log_transform=lf)
        rows = buf[pos:pos + 8 * rk].reshape(rk, 8)
        pos += 8 * rk
        reps = tuple(RoundReport(int(r[0]), int(r[1]), int(r[2]), float(r[3]), float(r[4]), float(r[5]),
                                 float(r[6]), float(r[7])) for r in rows)
        out.append((loc, reps))
        o += mk
    return out


def gather_packed(items, a: int, b: int, n: int, dim: int, group=None, device=None) -> list:
    """Allgatherv of every rank's [a, b) results, ordered by subdomain index.

    Two collectives: an all_gather of the (range, payload length) headers, then
    one all_gather_into_tensor of the payloads padded to the longest (NCCL over
    NVLink on the GPU box, gloo on CPU).  No Python object pickling.
    """
    import torch
    import torch.distributed as dist

    buf = pack_results(items, dim)
    if not dist.is_available() or not dist.is_initialized():
        parts = [(a, b, buf)]
    else:
        world = dist.get_world_size(group)
        dev = device if device is not None else torch.device("cpu")
        hdr = torch.tensor([a, b, buf.size], dtype=torch.int64, device=dev)
        hdrs = torch.empty(world * 3, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(hdrs, hdr, group=group)
        hdrs = hdrs.cpu().numpy().reshape(world, 3)
        width = int(hdrs[:, 2].max())
        mine = torch.zeros(width, dtype=torch.float64, device=dev)
        mine[:buf.size] = torch.from_numpy(buf).to(dev)
        allb = torch.empty(world * width, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(allb, mine, group=group)
        allb = allb.cpu().numpy().reshape(world, width)
        parts = [(int(h[0]), int(h[1]), allb[r, :int(h[2])]) for r, h in enumerate(hdrs)]
    out = [None] * n
    for lo, hi, pb in parts:
        got = unpack_results(pb, dim)
        if len(got) != hi - lo:
            raise RuntimeError(f"rank payload for [{lo}, {hi}) holds {len(got)} subdomains")
        for i, it in zip(range(lo, hi), got):
            if out[i] is not None:
                raise RuntimeError(f"subdomain {i} fitted by more than one rank")
            out[i] = it
    missing = [i for i, v in enumerate(out) if v is None]
    if missing:
        raise RuntimeError(f"subdomains {missing[:5]} were not fitted by any rank")
    return out


def gather_device_dictionaries(dict_off, m_cur, centres, widths, beta, dim: int, group=None):
    """Allgatherv of device-resident dictionaries (the engine's capacity-slot arrays).

    Every rank holds its contiguous subdomain range: dict_off (S_r,) int64 slot
    offsets, m_cur (S_r,) int32 sizes, centres (L_r * dim,), widths / beta (L_r,)
    float64.  Returns the same five arrays for the whole job, rank-major (=
    subdomain order), slot offsets rebased.  Padded all_gather_into_tensor per
    array (NCCL device buffers on the GPU box, gloo CPU tensors in the tests).
    """
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return dict_off, m_cur, centres, widths, beta
    world = dist.get_world_size(group)
    dev = widths.device
    hdr = torch.tensor([m_cur.numel(), widths.numel()], dtype=torch.int64, device=dev)
    hdrs = torch.empty(2 * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(hdrs, hdr, group=group)
    hdrs = hdrs.cpu().numpy().reshape(world, 2)
    s_max, l_max = int(hdrs[:, 0].max()), int(hdrs[:, 1].max())

    def ag(t, width):
        pad = torch.zeros(width, dtype=t.dtype, device=dev)
        pad[:t.numel()] = t.reshape(-1)
        out = torch.empty(world * width, dtype=t.dtype, device=dev)
        dist.all_gather_into_tensor(out, pad, group=group)
        return out.view(world, width)

    g_off = ag(dict_off.to(torch.int64), s_max)
    g_m = ag(m_cur.to(torch.int64), s_max)
    g_c = ag(centres, l_max * dim)
    g_w = ag(widths, l_max)
    g_b = ag(beta, l_max)
    base = np.concatenate([[0], np.cumsum(hdrs[:, 1])[:-1]])
    offs, ms, cs, ws, bs = [], [], [], [], []
    for r in range(world):
        n_s, n_l = int(hdrs[r, 0]), int(hdrs[r, 1])
        offs.append(g_off[r, :n_s] + int(base[r]))
        ms.append(g_m[r, :n_s])
        cs.append(g_c[r, :n_l * dim])
        ws.append(g_w[r, :n_l])
        bs.append(g_b[r, :n_l])
    return (torch.cat(offs), torch.cat(ms).to(torch.int32), torch.cat(cs), torch.cat(ws), torch.cat(bs))


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
    local = list(fit_range(a, b)) if b > a else []
    dev = None
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        import torch

        dev = torch.device("cuda", torch.cuda.current_device())
    items = gather_packed(local, a, b, n, partition.mesh.dim, group, dev)
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
