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


def test_pack_unpack_round_trip():
    """The allgatherv payload carries dictionaries, beta, generations and reports exactly."""
    import paper_2605_16564_b200 as pam

    rng = np.random.default_rng(3)
    items = []
    for k in range(4):
        m = 3 + k
        d = pam.RbfDictionary(centers=rng.random((m, 2)), widths=rng.uniform(0.1, 1, m),
                              generations=rng.integers(0, 4, m))
        reps = tuple(pam.RoundReport(r, m, r, *rng.random(4), 0.25) for r in range(k + 1))
        beta = rng.standard_normal(m) * 10.0 ** rng.integers(-300, 300, m)
        items.append((pam.LocalSurrogate(dictionary=d, beta=beta, log_transform=bool(k % 2)), reps))
    back = parallel.unpack_results(parallel.pack_results(items, 2), 2)
    for (l0, r0), (l1, r1) in zip(items, back):
        np.testing.assert_array_equal(l0.dictionary.centers, l1.dictionary.centers)
        np.testing.assert_array_equal(l0.dictionary.widths, l1.dictionary.widths)
        np.testing.assert_array_equal(l0.dictionary.generations, l1.dictionary.generations)
        np.testing.assert_array_equal(l0.beta, l1.beta)
        assert l0.log_transform == l1.log_transform
        assert r0 == r1
    out = parallel.gather_packed(items, 0, 4, 4, 2)  # single process: no collective
    assert [len(l.dictionary) for l, _ in out] == [3, 4, 5, 6]


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


def _dict_worker(rank, world, port, outq):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r owns subdomains with sizes m_r (ragged, different counts per rank)
        m = [np.array([3, 1, 4]), np.array([2, 5])][rank]
        cap = m + 1  # capacity slots beyond the size stay unused
        off = np.concatenate([[0], np.cumsum(cap)[:-1]])
        L = int(cap.sum())
        cen = np.arange(L * 2, dtype=np.float64) + 1000 * rank
        wid = np.arange(L, dtype=np.float64) + 100 * rank
        bet = -np.arange(L, dtype=np.float64) - 100 * rank
        out = parallel.gather_device_dictionaries(torch.from_numpy(off), torch.from_numpy(m.astype(np.int32)),
                                                  torch.from_numpy(cen), torch.from_numpy(wid),
                                                  torch.from_numpy(bet), 2)
        outq.put((rank, [t.numpy().tolist() for t in out]))
    finally:
        dist.destroy_process_group()


def test_device_dictionary_allgatherv_gloo_world2():
    """The packed device allgatherv (parallel.gather_device_dictionaries): ragged
    ranges, rebased slot offsets, identical on both ranks."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dict_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]
    off, m, cen, wid, bet = res[0][1]
    assert m == [3, 1, 4, 2, 5]
    assert off == [0, 4, 6, 11, 14]  # rank 1's offsets rebased by rank 0's 11 slots
    assert wid[:11] == list(range(11)) and wid[11:] == [100.0 + k for k in range(9)]
    assert cen[22:24] == [1000.0, 1001.0] and bet[11] == -100.0


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
