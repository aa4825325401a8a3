"""Wide GPU parity: every BASELINE configuration against the REFERENCE run on
many subdomains (tests/golden/make_golden_wide.py) and the bit-exact oracle.

Per golden subdomain (C2: all 64; C3: 34 of 256; C4: 67 of 2,244, both layer
types; C5: 64 boxes per M in {64, 128, 256, 512}, unchunked and through the
chunked ``fit_packed`` path):
  * the dictionary is bit-identical to the reference's (sha256 of centres,
    widths, generations -- no tie exemption);
  * beta within 1e-8 relative to max(1, max|beta|);
  * per-round reports: round/centers/added exact, max_residual, rel/abs L2
    and objective within 1e-8 relative;
  * the reference LocalSurrogate.evaluate at 16 seeded probes, 1e-8.
Evaluation sets against ``oracle.global_evaluate`` restated per owner
(partition.py:132-143; rbf.py:152-192) at 1e-8: C2 all 1e5 points, C3 the
full 1024^2 mesh transfer, C4 1e5 seeded 2x-refined centres plus every cell
centroid of 64 subdomains, C5 1e6 points over all 65,536 boxes.
"""

import hashlib
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import paper_2605_16564_b200 as pam
from paper_2605_16564_b200 import engine as E
from paper_2605_16564_b200 import workloads
from oracle import pam_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-8


def dict_digest(centers, widths, generations) -> str:
    h = hashlib.sha256()
    for a in (np.asarray(centers, dtype=np.float64), np.asarray(widths, dtype=np.float64),
              np.asarray(generations, dtype=np.int64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def input_digest(values) -> str:
    return hashlib.sha256(np.ascontiguousarray(values).tobytes()).hexdigest()


def check_subdomain(g, s, centers, widths, generations, beta, reports=None, probe_eval=None):
    p = f"s{s}_"
    assert len(widths) == int(g[p + "m"]), (s, len(widths), int(g[p + "m"]))
    assert dict_digest(centers, widths, generations) == str(g[p + "dict"]), f"subdomain {s}: dictionary differs"
    ref = g[p + "beta"]
    err = np.max(np.abs(np.asarray(beta) - ref))
    assert err <= TOL * max(1.0, np.abs(ref).max()), (s, err)
    if reports is not None:
        rows = g[p + "reports"]
        assert len(reports) == len(rows), (s, len(reports), len(rows))
        for r, row in zip(reports, rows):
            assert (r.round, r.centers, r.added) == (int(row[0]), int(row[1]), int(row[2])), (s, r, row)
            for name, v in zip(("max_residual", "rel_l2", "abs_l2", "objective"), row[3:]):
                got = getattr(r, name)
                assert abs(got - v) <= TOL * max(abs(v), 1e-300) + 1e-300, (s, name, got, v)
    if probe_eval is not None:
        np.testing.assert_allclose(probe_eval(g[p + "probe"]), g[p + "probe_values"], rtol=TOL)


# ---------------------------------------------------------------------------
# oracle evaluation grouped by owner, spread over the host cores (fork)

_EVAL_CTX = {}


def _eval_chunk(bounds):
    pts, order, starts, locs = (_EVAL_CTX[k] for k in ("pts", "order", "starts", "locs"))
    out = []
    for i in range(*bounds):
        sel = order[starts[i]:starts[i + 1]]
        if sel.size:
            c, w, b = locs[i]
            out.append((sel, O.surrogate_eval(pts[sel], c, w, b)))
    return out


def oracle_eval(pts, owner, locs):
    """O.surrogate_eval per owner (the oracle's global_evaluate, partition.py:132-143) in owner
    groups; `owner` comes from O.locate_many or the grid formula below."""
    order = np.argsort(owner, kind="stable")
    starts = np.searchsorted(owner[order], np.arange(len(locs) + 1))
    _EVAL_CTX.update(pts=pts, order=order, starts=starts, locs=locs)
    procs = max(1, min(16, O.n_threads()))
    S = len(locs)
    step = max(1, S // (4 * procs))
    chunks = [(a, min(S, a + step)) for a in range(0, S, step)]
    out = np.empty(pts.shape[0])
    import multiprocessing as mp

    with ProcessPoolExecutor(procs, mp_context=mp.get_context("fork")) as pool:
        for res in pool.map(_eval_chunk, chunks):
            for sel, v in res:
                out[sel] = v
    return out


def grid_owner(pts, part):
    """Owner by the reference's half-open edge comparisons on a tensor grid (bit-exact with
    O.locate_many on these grids, tests/test_oracle_pins.py)."""
    shape, edges = part.grid
    own = np.zeros(pts.shape[0], dtype=np.int64)
    stride = 1
    for k in range(len(shape)):
        idx = np.clip(np.searchsorted(edges[k], pts[:, k], side="right") - 1, 0, shape[k] - 1)
        own += stride * idx
        stride *= shape[k]
    return own


def _run(wl):
    return pam.fit_parallel(wl.field, wl.partition, wl.config, wl.spec)


def _check_config(name, wl, sur, rep, golden):
    g = golden(name)
    assert str(g["input_digest"]) == input_digest(wl.field.values), "synthetic input drifted"
    for s in g["subdomains"]:
        d = sur.locals[s].dictionary
        check_subdomain(g, s, d.centers, d.widths, d.generations, sur.locals[s].beta, rep.rounds[s],
                        sur.evaluate)
    return g


def test_config2_all_64_subdomains_and_full_eval(cuda, golden):
    wl = workloads.config2()
    sur, rep = _run(wl)
    g = _check_config("C2all", wl, sur, rep, golden)
    assert len(g["subdomains"]) == 64
    # the full 1e5-point evaluation vs the oracle with the reference's coefficients
    part = wl.partition
    locs = [(sur.locals[s].dictionary.centers, sur.locals[s].dictionary.widths, g[f"s{s}_beta"])
            for s in range(64)]
    owner = O.locate_many(wl.eval_points, [(b.lo, b.hi, b.open_hi) for b in part.boxes])
    np.testing.assert_array_equal(pam.locate_many(wl.eval_points, part.boxes), owner)
    ref = oracle_eval(wl.eval_points, owner, locs)
    np.testing.assert_allclose(sur.evaluate(wl.eval_points), ref, rtol=TOL)


def test_config3_wide_and_mesh_transfer(cuda, golden):
    wl = workloads.config3()  # eval on the 1024 x 1024 centroid grid (mesh transfer)
    assert wl.eval_points.shape[0] == 1024 * 1024
    sur, rep = _run(wl)
    g = _check_config("C3wide", wl, sur, rep, golden)
    assert len(g["subdomains"]) >= 32
    got = sur.evaluate(wl.eval_points)
    owner = grid_owner(wl.eval_points, wl.partition)
    locs = [(l.dictionary.centers, l.dictionary.widths, l.beta) for l in sur.locals]
    ref = oracle_eval(wl.eval_points, owner, locs)
    np.testing.assert_allclose(got, ref, rtol=TOL)
    # golden subdomains: the same points through the reference's own coefficients
    gs = set(int(s) for s in g["subdomains"])
    sel = np.flatnonzero(np.isin(owner, list(gs)))
    locs_ref = [(l.dictionary.centers, l.dictionary.widths, g[f"s{s}_beta"] if s in gs else l.beta)
                for s, l in enumerate(sur.locals)]
    ref2 = oracle_eval(wl.eval_points[sel], owner[sel], locs_ref)
    np.testing.assert_allclose(got[sel], ref2, rtol=TOL)


def test_config4_wide_and_refined_eval(cuda, golden):
    wl = workloads.config4(with_refined_eval=False)
    part = wl.partition
    assert part.n_subdomains == 2244
    sur, rep = _run(wl)
    g = _check_config("C4wide", wl, sur, rep, golden)
    subs = [int(s) for s in g["subdomains"]]
    assert sum(s < 7 * 132 for s in subs) >= 32 and sum(s >= 7 * 132 for s in subs) >= 32
    # cell ownership bit-exact vs the oracle's partition restatement
    mesh = wl.field.mesh
    _, owner, _ = O.partition_boxes(mesh.counts, mesh.bounds, wl.shape)
    np.testing.assert_array_equal(part.cell_to_subdomain, owner)
    np.testing.assert_array_equal(pam.locate_many(mesh.centroids, part.boxes), owner)
    locs = [(l.dictionary.centers, l.dictionary.widths, l.beta) for l in sur.locals]
    # every cell centroid of 64 subdomains vs the oracle (GPU dictionaries = reference's)
    sel = np.flatnonzero(np.isin(owner, subs[:64]))
    ref = oracle_eval(mesh.centroids[sel], owner[sel], locs)
    np.testing.assert_allclose(sur.evaluate(mesh.centroids[sel]), ref, rtol=TOL)
    # 1e5 seeded 2x-refined cell centres over the whole domain
    fine = pam.build_mesh(3, tuple(2 * n for n in workloads.SPE10_COUNTS), mesh.bounds)
    pick = np.sort(np.random.default_rng(44).choice(fine.n_cells, 100_000, replace=False))
    pts = fine.centroids[pick]
    own = grid_owner(pts, part)
    np.testing.assert_array_equal(pam.locate_many(pts, part.boxes), own)
    np.testing.assert_allclose(sur.evaluate(pts), oracle_eval(pts, own, locs), rtol=TOL)


def _c5_reports(res, s):
    return E.reports_for(res, s, pam.RoundReport)


@pytest.mark.parametrize("M", [64, 128, 256, 512])
def test_config5_64_boxes_vs_reference(cuda, golden, M):
    """64 C5 boxes per centre count against the reference, unchunked and through the
    chunked fit_packed path (one device batch per 8 boxes): identical results."""
    p = workloads.config5(M=M, n_sub=64, n_eval=0)
    g = golden(f"C5_M{M}")
    assert str(g["input_digest"]) == input_digest(p.values)
    res = pam.fit_subdomains(p)
    per_box = int(E.device_bytes(np.diff(p.row_off[:2]), [M])[0])
    chunked = pam.fit_subdomains(p, budget_bytes=8 * per_box)
    assert len(chunked.rounds[0].sweeps) == 64
    for s in range(64):
        a, b = p.row_off[s], p.row_off[s + 1]
        d = pam.RbfDictionary(centers=res.centres[s], widths=res.widths[s], generations=res.generations[s])
        loc = pam.LocalSurrogate(dictionary=d, beta=res.beta[s])
        check_subdomain(g, s, res.centres[s], res.widths[s], res.generations[s], res.beta[s],
                        _c5_reports(res, s), loc.evaluate)
        np.testing.assert_array_equal(chunked.beta[s], res.beta[s])
        np.testing.assert_array_equal(chunked.centres[s], res.centres[s])
        assert a < b


def test_config5_eval_1e6_points_all_boxes(cuda):
    """All 65,536 C5 boxes (M = 64, on-device generator) fitted, then 1e6 uniform points
    over the whole 64x32x32 domain vs the oracle with the fitted coefficients."""
    p = workloads.config5_device(M=64)
    res = pam.fit_subdomains(p)
    part = pam.make_partition(pam.build_mesh(3, (64, 32, 32), ((0.0, 64.0), (0.0, 32.0), (0.0, 32.0))),
                              64, 32, 32)
    locs = [(res.centres[s], res.widths[s], res.beta[s]) for s in range(65536)]
    sur = pam.GlobalSurrogate(partition=part, locals=tuple(
        pam.LocalSurrogate(dictionary=pam.RbfDictionary(centers=c, widths=w), beta=b) for c, w, b in locs))
    pts = np.random.default_rng(55).random((1_000_000, 3)) * np.array([64.0, 32.0, 32.0])
    own = grid_owner(pts, part)
    assert np.unique(own).size > 65_000
    np.testing.assert_allclose(sur.evaluate(pts), oracle_eval(pts, own, locs), rtol=TOL)
