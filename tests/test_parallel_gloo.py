"""Multi-process sharding of the fit (parallel.py), world_size 2 over gloo on CPU.

The device engine is replaced by the CPU oracle as the per-rank ``fit_range``
so the host-side sharding + gather logic is exercised without a GPU; the
gathered surrogate must equal the single-process one bit for bit.
"""

import os
import socket

import numpy as np
import pytest

from paper_2605_16564_b200 import parallel


def test_balanced_ranges():
    r = parallel.balanced_ranges(np.ones(10), 3)
    assert r[0][0] == 0 and r[-1][1] == 10
    assert all(a <= b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(2))
    w = np.array([100.0, 1, 1, 1, 1, 1])
    r = parallel.balanced_ranges(w, 2)
    assert r[0] == (0, 1) and r[1] == (1, 6)
    assert parallel.balanced_ranges(np.ones(3), 5)[-1][1] == 3


def _oracle_fit_range(field, part, cfg, sigma):
    from oracle import pam_oracle as O
    import paper_2605_16564_b200 as pam

    c = dict(lam1=cfg.elastic.lam1, lam2=cfg.elastic.lam2, tol=cfg.elastic.tol,
             max_iters=cfg.elastic.max_iters, k_top=cfg.k_top, m_max=cfg.m_max, eta=cfg.eta,
             m_q=cfg.m_q, max_rounds=cfg.max_rounds, offsets=cfg.offsets)

    def run(a, b):
        out = []
        for i in range(a, b):
            bx = part.boxes[i]
            rows = O.subdomain_rows(field.mesh.centroids, (bx.lo, bx.hi, bx.open_hi))
            cen = field.mesh.centroids[rows]
            od = O.fit_adaptive(cen, field.values[rows], field.mesh.cell_size, bx.lo, bx.hi, cen,
                                np.full(rows.size, sigma), c)
            d = pam.RbfDictionary(centers=od["centers"], widths=od["widths"], generations=od["generations"])
            reps = tuple(pam.RoundReport(r["round"], r["centers"], r["added"], r["max_residual"],
                                         r["rel_l2"], r["abs_l2"], r["objective"], 0.0)
                         for r in od["reports"])
            out.append((pam.LocalSurrogate(dictionary=d, beta=od["beta"]), reps))
        return out

    return run


def _problem():
    import paper_2605_16564_b200 as pam

    field = pam.box_field_2d(12, 12)
    part = pam.make_partition(field.mesh, 3, 2)
    cfg = pam.AdaptiveConfig(k_top=5, m_max=30, m_q=3, max_rounds=3,
                             elastic=pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=200),
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    return field, part, cfg, 1.0 / 12


def _worker(rank, world, port, outq):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_16564_b200 as pam

        field, part, cfg, sigma = _problem()
        sur, reps = parallel.fit_parallel_sharded(
            field, part, cfg, pam.DictionarySpec(sigma=sigma),
            fit_range=_oracle_fit_range(field, part, cfg, sigma))
        outq.put((rank, pam.dumps(sur), [[r.centers for r in rr] for rr in reps]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_fit_gloo_world2_matches_single_process():
    import multiprocessing as mp

    import paper_2605_16564_b200 as pam

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1]  # identical surrogate on every rank
    field, part, cfg, sigma = _problem()
    single = _oracle_fit_range(field, part, cfg, sigma)(0, part.n_subdomains)
    ref = pam.GlobalSurrogate(partition=part, locals=tuple(s[0] for s in single),
                              metadata={"field_checksum": field.checksum()})
    assert res[0][1] == pam.dumps(ref)
    assert res[0][2] == [[r.centers for r in s[1]] for s in single]
