"""End-to-end GPU parity of the batched adaptive fit and the fused evaluation
against the reference's own outputs (golden fixtures made by running the
reference, tests/golden/make_golden.py) and the bit-exact CPU oracle.

Contract (BASELINE north_star): subdomain partition and cell ownership
bit-exact; selected-centre sets (dictionaries) identical; coefficients,
reconstructed values and L1/L2 errors within 1e-8 relative.
"""

import os

import numpy as np
import pytest

import paper_2605_16564_b200 as pam
from paper_2605_16564_b200 import engine as E
from paper_2605_16564_b200 import workloads
from oracle import pam_oracle as O

pytestmark = pytest.mark.gpu
BETA_TOL = 1e-8
VAL_TOL = 1e-8


def _assert_local_matches(loc, g, prefix, check_reports=None):
    np.testing.assert_array_equal(loc.dictionary.centers, g[f"{prefix}centers"])
    np.testing.assert_array_equal(loc.dictionary.widths, g[f"{prefix}widths"])
    if f"{prefix}generations" in g:
        np.testing.assert_array_equal(loc.dictionary.generations, g[f"{prefix}generations"])
    ref = g[f"{prefix}beta"]
    assert np.max(np.abs(loc.beta - ref)) <= BETA_TOL * max(1.0, np.abs(ref).max())


def _assert_reports(reps, ref_rows, cols):
    """ref_rows columns named by `cols`; counts exact, reals 1e-8 relative."""
    assert len(reps) == len(ref_rows)
    for r, row in zip(reps, ref_rows):
        for name, v in zip(cols, row):
            got = getattr(r, name)
            if name in ("round", "centers", "added"):
                assert got == int(v), (name, got, v)
            else:
                assert abs(got - v) <= 1e-8 * max(abs(v), 1e-300) + 1e-300, (name, got, v)


def test_fit_adaptive_1d_step(cuda, golden):
    g = golden("adaptive_small")
    field = pam.step_field_1d(16)
    sub = field.whole()
    cfg = pam.AdaptiveConfig(k_top=2, m_max=12, eta=0.5, m_q=3, max_rounds=3,
                             elastic=pam.ElasticNetConfig(lam1=4.59e-4, lam2=4.64e-6))
    sur, reps = pam.fit_adaptive(sub, pam.centroid_dictionary(sub.centroids, 0.0019), cfg)
    assert [r.centers for r in reps] == [16, 22, 28]  # reference test_adaptive.py:166-172
    assert [r.added for r in reps] == [0, 6, 12]
    _assert_local_matches(sur, g, "a1_")
    _assert_reports(reps, g["a1_reports"], ("centers", "added", "max_residual", "rel_l2", "objective"))


def test_fit_adaptive_2d_box(cuda, golden):
    g = golden("adaptive_small")
    field = pam.box_field_2d(16, 16)
    sub = field.whole()
    cfg = pam.AdaptiveConfig(k_top=51, m_max=306, eta=0.5, m_q=3, max_rounds=3,
                             elastic=pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=1500),
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    sur, reps = pam.fit_adaptive(sub, pam.centroid_dictionary(sub.centroids, 0.0625), cfg)
    _assert_local_matches(sur, g, "a2_")
    _assert_reports(reps, g["a2_reports"], ("centers", "added", "max_residual", "rel_l2", "objective"))
    errs = [r.rel_l2 for r in reps]
    assert all(b < a for a, b in zip(errs, errs[1:]))


def test_fit_adaptive_3d_quad2(cuda, golden):
    g = golden("adaptive_small")
    fld = workloads.spe10_like_field(4)
    mesh = fld.mesh
    rows = g["a3_rows"]
    box = pam.Box(lo=(400.0, 100.0, 80.0), hi=(520.0, 150.0, 88.0), open_hi=(True, True, True))
    sub = pam.SubdomainField(box=box, cell_indices=rows, centroids=mesh.centroids[rows],
                             values=fld.values[rows], cell_size=mesh.cell_size)
    cfg = pam.AdaptiveConfig(k_top=24, m_max=144, eta=0.5, m_q=3, max_rounds=3, quad_order=2,
                             elastic=pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=1000),
                             offsets=workloads.IN_CELL_3D)
    sigma = float(np.prod(mesh.cell_size) ** (1 / 3))
    sur, reps = pam.fit_adaptive(sub, pam.RbfDictionary(centers=sub.centroids, widths=np.full(rows.size, sigma)), cfg)
    _assert_local_matches(sur, g, "a3_")
    _assert_reports(reps, g["a3_reports"], ("centers", "added", "max_residual", "rel_l2", "objective"))


def _run_config(wl, eval_points=None):
    part = wl.partition
    sur, rep = pam.fit_parallel(wl.field, part, wl.config, wl.spec)
    return part, sur, rep


def _check_golden_subdomains(name, wl, sur, rep, golden):
    g = golden(name)
    assert str(g["input_digest"]) == __import__("hashlib").sha256(
        np.ascontiguousarray(wl.field.values).tobytes()).hexdigest(), "synthetic input drifted"
    for s in g["subdomains"]:
        p = f"s{s}_"
        _assert_local_matches(sur.locals[s], g, p)
        _assert_reports(rep.rounds[s], g[p + "reports"],
                        ("round", "centers", "added", "max_residual", "rel_l2", "abs_l2", "objective"))
        got = sur.evaluate(g[p + "probe"])
        np.testing.assert_allclose(got, g[p + "probe_values"], rtol=VAL_TOL)


def test_config1_step2d_full(cuda, golden):
    wl = workloads.config1()
    part, sur, rep = _run_config(wl)
    _check_golden_subdomains("C1", wl, sur, rep, golden)
    # evaluation on the 128x128 mesh (mesh transfer) vs the oracle with the golden dictionaries
    g = golden("C1")
    boxes = [(b.lo, b.hi, b.open_hi) for b in part.boxes]
    locs = [(g[f"s{s}_centers"], g[f"s{s}_widths"], g[f"s{s}_beta"]) for s in range(4)]
    ref, owner = O.global_evaluate(wl.eval_points, boxes, locs)
    got = sur.evaluate(wl.eval_points)
    np.testing.assert_allclose(got, ref, rtol=VAL_TOL)
    np.testing.assert_array_equal(pam.locate_many(wl.eval_points, part.boxes), owner)
    true = wl.notes["true_field"](wl.eval_points)
    l1_got = np.sum(np.abs(got - true)) / 128**2
    l1_ref = np.sum(np.abs(ref - true)) / 128**2
    assert abs(l1_got - l1_ref) <= 1e-8 * l1_ref


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_config_2d_refined_sampled(cuda, golden, name):
    wl = workloads.config2() if name == "C2" else workloads.config3(eval_n=256)
    part, sur, rep = _run_config(wl)
    _check_golden_subdomains(name, wl, sur, rep, golden)
    # size-independent properties over ALL subdomains
    for s, reps in enumerate(rep.rounds):
        assert reps[0].centers == 1024
        assert all(b.centers >= a.centers for a, b in zip(reps, reps[1:]))
        assert np.all(np.isfinite(sur.locals[s].beta))
    vals = sur.evaluate(wl.eval_points)
    assert np.all(vals > 0) and np.all(np.isfinite(vals))


def test_config4_spe10_shaped_full(cuda, golden):
    wl = workloads.config4(with_refined_eval=False)
    part, sur, rep = _run_config(wl)
    assert part.n_subdomains == 2244
    _check_golden_subdomains("C4", wl, sur, rep, golden)
    # cell ownership bit-exact vs the oracle's partition restatement
    _, owner, _ = O.partition_boxes(wl.field.mesh.counts, wl.field.mesh.bounds, wl.shape)
    np.testing.assert_array_equal(part.cell_to_subdomain, owner)
    got_owner = pam.locate_many(wl.field.mesh.centroids, part.boxes)
    np.testing.assert_array_equal(got_owner, owner)
    # two more subdomains against the oracle run here (the oracle is bit-exact to the reference)
    c = wl.config
    cfgd = dict(lam1=c.elastic.lam1, lam2=c.elastic.lam2, tol=c.elastic.tol, max_iters=c.elastic.max_iters,
                k_top=c.k_top, m_max=c.m_max, eta=c.eta, m_q=c.m_q, max_rounds=c.max_rounds, offsets=c.offsets)
    mesh = wl.field.mesh
    for s in (1, 1999):
        b = part.boxes[s]
        rows = O.subdomain_rows(mesh.centroids, (b.lo, b.hi, b.open_hi))
        cen = mesh.centroids[rows]
        od = O.fit_adaptive(cen, wl.field.values[rows], mesh.cell_size, b.lo, b.hi, cen,
                            np.full(rows.size, wl.spec.sigma), cfgd)
        np.testing.assert_array_equal(sur.locals[s].dictionary.centers, od["centers"])
        assert np.max(np.abs(sur.locals[s].beta - od["beta"])) <= BETA_TOL * max(1, np.abs(od["beta"]).max())
    # evaluation at every centroid: positive, finite, matches the per-owner local surrogate
    vals = sur.evaluate(mesh.centroids)
    assert np.all(vals > 0) and np.all(np.isfinite(vals))
    sel = np.flatnonzero(owner == 1337)
    np.testing.assert_allclose(vals[sel], sur.locals[1337].evaluate(mesh.centroids[sel]), rtol=1e-13)


# ---- reference behaviour (tests/test_partition.py) --------------------------

EN_2D = pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=2000)
PLAIN_CFG = pam.AdaptiveConfig(m_max=0, elastic=EN_2D)


def test_fit_parallel_1x1_matches_direct(cuda):
    field = pam.box_field_2d(8, 8)
    part = pam.make_partition(field.mesh, 1, 1)
    spec = pam.DictionarySpec(sigma=0.13)
    surrogate, report = pam.fit_parallel(field, part, PLAIN_CFG, spec)
    direct, _ = pam.fit_adaptive(field.whole(), spec.build(field.whole()), PLAIN_CFG)
    np.testing.assert_array_equal(surrogate.locals[0].beta, direct.beta)
    assert len(report.rounds) == 1


def test_fit_parallel_constant_field(cuda):
    mesh = pam.build_mesh(2, (8, 8), ((0, 1), (0, 1)))
    field = pam.FieldData(mesh=mesh, values=np.full(64, 3.7))
    part = pam.make_partition(mesh, 2, 2)
    surrogate, _ = pam.fit_parallel(field, part, pam.AdaptiveConfig(m_max=0), pam.DictionarySpec(sigma=0.13))
    pts = np.random.default_rng(4).random((200, 2))
    np.testing.assert_allclose(surrogate.evaluate(pts), 3.7, rtol=1e-6)


def test_fit_parallel_deterministic_and_chunk_independent(cuda):
    field = pam.box_field_2d(16, 16)
    part = pam.make_partition(field.mesh, 2, 2)
    cfg = pam.AdaptiveConfig(k_top=12, m_max=72, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.0625)
    s1, r1 = pam.fit_parallel(field, part, cfg, spec, workers=1)
    s4, _ = pam.fit_parallel(field, part, cfg, spec, workers=4)
    with E.options(w_budget_gb=1e-7):  # one subdomain per device batch
        sc, rc = pam.fit_parallel(field, part, cfg, spec)
    assert rc.max_concurrent == 1
    pts = np.random.default_rng(0).random((500, 2))
    for other in (s4, sc):
        for a, b in zip(s1.locals, other.locals):
            np.testing.assert_array_equal(a.beta, b.beta)
            np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        np.testing.assert_array_equal(s1.evaluate(pts), other.evaluate(pts))
    assert pam.dumps(s1) == pam.dumps(s4)


@pytest.mark.parametrize("tau", [2.0 ** -100, 1e-16])
@pytest.mark.parametrize("cells", [(16, 16), (40, 40)])
def test_tile_packed_stream_matches_dense(cuda, cells, tau):
    """Tile-dropping (tau = 2^-100 and the default 1e-16) vs exact dense streaming:
    same decisions, beta ~1e-12."""
    field = pam.box_field_2d(*cells)
    part = pam.make_partition(field.mesh, 2, 2)
    cfg = pam.AdaptiveConfig(k_top=cells[0], m_max=6 * cells[0], m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.5 / cells[0])
    with E.options(cd_form="residual", tile_tau=0.0):  # few fits would pick the covariance form
        dense, rd = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="residual", tile_tau=tau):
        tiled, rt = pam.fit_parallel(field, part, cfg, spec)
    assert rt.device["cd_bytes"] < rd.device["cd_bytes"]  # tiles were actually dropped
    for a, b in zip(dense.locals, tiled.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    for ra, rb in zip(rd.rounds, rt.rounds):
        assert [r.centers for r in ra] == [r.centers for r in rb]
        for x, y in zip(ra, rb):
            assert abs(x.rel_l2 - y.rel_l2) <= 1e-10 * x.rel_l2


@pytest.mark.parametrize("cells,parts", [((40, 40), (2, 2)), ((60, 60), (3, 3))])
@pytest.mark.parametrize("kernel", ["lean", "dual", "pair", "block"])
def test_cd_kernel_choices_match(cuda, cells, parts, kernel):
    """Every CD kernel of pam_cd_tiles_f64 (one fit per warp, two fits per warp,
    column pairs) against the dense residual-form stream: same dictionaries,
    beta and objectives ~1e-12 (only dot-product rounding differs)."""
    field = pam.box_field_2d(*cells)
    part = pam.make_partition(field.mesh, *parts)  # 400 rows: the R=16 tile kernels
    cfg = pam.AdaptiveConfig(k_top=40, m_max=240, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.5 / cells[0])
    with E.options(cd_form="residual", tile_tau=0.0):
        base, rb = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="residual", cd_kernel=kernel):
        other, ro = pam.fit_parallel(field, part, cfg, spec)
    for a, b in zip(base.locals, other.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    for ra, rb_ in zip(rb.rounds, ro.rounds):
        for x, y in zip(ra, rb_):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-10 * abs(x.objective)


def test_gram_form_matches_residual_form(cuda):
    """Covariance-form CD (gram.cu) vs residual form on a lattice dictionary with refinement."""
    field = pam.box_field_2d(32, 32)
    part = pam.make_partition(field.mesh, 2, 2)
    cfg = pam.AdaptiveConfig(k_top=16, m_max=96, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=1.0 / 16, lattice=8)  # M0=64, cap=160 < 0.75*N=192
    with E.options(cd_form="residual"):
        res, rr = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="gram"):
        gram, rg = pam.fit_parallel(field, part, cfg, spec)
    assert rg.device["cd_bytes"] < rr.device["cd_bytes"]
    for a, b in zip(res.locals, gram.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-9 * max(1, np.abs(a.beta).max())
    for ra, rb in zip(rr.rounds, rg.rounds):
        for x, y in zip(ra, rb):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-9 * abs(x.objective)
            assert abs(x.rel_l2 - y.rel_l2) <= 1e-9 * x.rel_l2


class _BrokenSpec(pam.DictionarySpec):
    def build(self, sub):
        raise RuntimeError("boom")


def test_fit_parallel_errors(cuda):
    mesh = pam.build_mesh(2, (4, 4), ((0, 1), (0, 1)))
    field = pam.FieldData(mesh=mesh, values=np.ones(16))
    part = pam.make_partition(mesh, 2, 1)
    with pytest.raises(RuntimeError, match="subdomain 1"):
        pam.fit_parallel(field, part, PLAIN_CFG, [pam.DictionarySpec(sigma=0.1), _BrokenSpec(sigma=0.1)])
    with pytest.raises(ValueError, match="1 entries for 2"):
        pam.fit_parallel(field, part, [PLAIN_CFG], pam.DictionarySpec(sigma=0.1))


def test_evaluate_order_positivity_and_errors(cuda):
    field = pam.box_field_2d(8, 8)
    part = pam.make_partition(field.mesh, 2, 2)
    surrogate, _ = pam.fit_parallel(field, part, PLAIN_CFG, pam.DictionarySpec(sigma=0.13))
    pts = np.random.default_rng(1).random((333, 2))
    vals = surrogate.evaluate(pts)
    assert np.all(vals > 0)
    owner = pam.locate_many(pts, part.boxes)
    for i in range(part.n_subdomains):
        sel = owner == i
        np.testing.assert_array_equal(vals[sel], surrogate.locals[i].evaluate(pts[sel]))
    with pytest.raises(ValueError, match="index 1"):
        surrogate.evaluate(np.array([[0.5, 0.5], [1.5, 0.5]]))
    # reloaded (host-built device cache) evaluates bit-identically
    back = pam.loads(pam.dumps(surrogate))
    np.testing.assert_array_equal(surrogate.evaluate(pts), back.evaluate(pts))


def _lshape_partition(mesh):
    """Three boxes tiling [0,1]^2 that are NOT a tensor grid: the left half, and the
    right half split in two (half-open internal faces, closed outer faces)."""
    boxes = (pam.Box(lo=(0.0, 0.0), hi=(0.5, 1.0), open_hi=(True, False)),
             pam.Box(lo=(0.5, 0.0), hi=(1.0, 0.5), open_hi=(False, True)),
             pam.Box(lo=(0.5, 0.5), hi=(1.0, 1.0), open_hi=(False, False)))
    cen = mesh.centroids
    owner = O.locate_many(cen, [(b.lo, b.hi, b.open_hi) for b in boxes])
    return pam.Partition(mesh=mesh, shape=(3,), boxes=boxes, cell_to_subdomain=owner)


def test_generic_boxes_locate_evaluate_and_errors(cuda):
    """Box sets that are not a tensor grid (the reference's locate_many and
    GlobalSurrogate.evaluate accept any half-open boxes, geometry.py:242-258)."""
    field = pam.box_field_2d(8, 8)
    part = _lshape_partition(field.mesh)
    assert part.grid is None
    rng = np.random.default_rng(7)
    pts = np.vstack([rng.random((500, 2)),
                     [[0.5, 0.25], [0.5, 0.5], [0.75, 0.5], [1.0, 1.0], [0.0, 0.0], [0.5, 1.0], [1.0, 0.5]]])
    boxes_o = [(b.lo, b.hi, b.open_hi) for b in part.boxes]
    own_ref = O.locate_many(pts, boxes_o)
    np.testing.assert_array_equal(pam.locate_many(pts, part.boxes), own_ref)  # faces included, bit-exact
    surrogate, _ = pam.fit_parallel(field, part, PLAIN_CFG, pam.DictionarySpec(sigma=0.13))
    vals = surrogate.evaluate(pts)
    for i in range(part.n_subdomains):
        sel = own_ref == i
        np.testing.assert_array_equal(vals[sel], surrogate.locals[i].evaluate(pts[sel]))
    ref, _ = O.global_evaluate(pts, boxes_o, [(l.dictionary.centers, l.dictionary.widths, l.beta)
                                              for l in surrogate.locals])
    np.testing.assert_allclose(vals, ref, rtol=1e-8)
    # a point in no box: first offending index, as the reference reports it
    with pytest.raises(ValueError, match=r"point index 2 = \[1.5, 0.5\] lies outside all boxes"):
        surrogate.evaluate(np.array([[0.2, 0.2], [0.7, 0.7], [1.5, 0.5], [2.0, 2.0]]))
    with pytest.raises(ValueError, match="point index 1 "):
        pam.locate_many(np.array([[0.2, 0.2], [-0.1, 0.5]]), part.boxes)
    # overlapping boxes: the first box, in order, that re-claims a point wins the report
    over = part.boxes + (pam.Box(lo=(0.4, 0.4), hi=(0.6, 0.6), open_hi=(True, True)),)
    p2 = np.array([[0.9, 0.9], [0.55, 0.55], [0.45, 0.45], [1.7, 0.0]])
    with pytest.raises(ValueError) as e_gpu:
        pam.locate_many(p2, over)
    with pytest.raises(ValueError) as e_ref:
        O.locate_many(p2, [(b.lo, b.hi, b.open_hi) for b in over])
    assert str(e_gpu.value) == str(e_ref.value) == "point index 1 claimed by boxes 2 and 3"


def test_continuity_near_internal_face(cuda):
    field = pam.box_field_2d(8, 8)
    part = pam.make_partition(field.mesh, 2, 1)
    surrogate, _ = pam.fit_parallel(field, part, PLAIN_CFG, pam.DictionarySpec(sigma=0.13))
    ys = np.linspace(0.05, 0.95, 7)
    for eps in (1e-6, 1e-9):
        a = surrogate.evaluate(np.column_stack([np.full(7, 0.5 + eps), ys]))
        b = surrogate.evaluate(np.column_stack([np.full(7, 0.5 + 2 * eps), ys]))
        assert np.max(np.abs(a - b)) < (1e-3 if eps == 1e-6 else 1e-6)


def test_centroid_values_within_max_residual(cuda):
    field = pam.box_field_2d(8, 8)
    part = pam.make_partition(field.mesh, 1, 1)
    cfg = pam.AdaptiveConfig(m_max=0, elastic=pam.ElasticNetConfig(tol=1e-12))
    surrogate, report = pam.fit_parallel(field, part, cfg, pam.DictionarySpec(sigma=0.05))
    vals = surrogate.evaluate(field.mesh.centroids)
    worst = report.rounds[0][-1].max_residual
    assert np.max((vals - field.values) ** 2 * field.mesh.cell_measure) <= worst * (1 + 1e-9)


@pytest.mark.parametrize("M", [64, 128, 256, 512])
def test_subdomain_batch_api_c5_sample(cuda, M):
    """C5 shape (unit boxes, 1000 random samples, jittered lattice) on a 32-box sample,
    every centre count of the sweep (the covariance-form CD runs a different
    register configuration for each)."""
    p = workloads.config5(M=M, n_sub=32, n_eval=0)
    res = pam.fit_subdomains(p)
    c = p.config
    for s in ((0, 17, 31) if M <= 128 else (0, 31)):
        a, b = p.row_off[s], p.row_off[s + 1]
        cen = p.centres[s * M:(s + 1) * M]
        W = O.shepard_features(p.points[a:b], cen, p.widths[s * M:(s + 1) * M])
        o = O.fit_log(p.values[a:b], W, c.elastic.lam1, c.elastic.lam2, c.elastic.tol, c.elastic.max_iters)
        assert np.max(np.abs(res.beta[s] - o["beta"])) <= BETA_TOL * max(1, np.abs(o["beta"]).max())
        assert res.rounds[0].sweeps[s] == o["iterations"] or abs(res.rounds[0].sweeps[s] - o["iterations"]) <= 1


def test_sharded_fit_single_rank_device_path(cuda):
    """parallel.fit_parallel_sharded with the device fit_range (world size 1) == fit_parallel."""
    from paper_2605_16564_b200 import parallel

    field = pam.box_field_2d(16, 16)
    part = pam.make_partition(field.mesh, 2, 2)
    cfg = pam.AdaptiveConfig(k_top=12, m_max=72, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.0625)
    ref, rep = pam.fit_parallel(field, part, cfg, spec)
    sh, reps = parallel.fit_parallel_sharded(field, part, cfg, spec)
    assert pam.dumps(sh) == pam.dumps(ref)
    assert [[r.centers for r in rr] for rr in reps] == [[r.centers for r in rr] for rr in rep.rounds]


@pytest.mark.parametrize("cells", [(20, 20), (30, 30)])
def test_lean_kernel_small_rows_odd_columns(cuda, cells):
    """Lean CD at R=4 / R=8 with odd dictionary sizes and ragged batches == the dense kernel."""
    field = pam.box_field_2d(*cells)
    part = pam.make_partition(field.mesh, 2, 2)  # 100 / 225 rows
    cfg = pam.AdaptiveConfig(k_top=7, m_max=60, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.5 / cells[0])
    with E.options(cd_form="residual", cd_kernel="lean"):  # few fits would pick the covariance form
        lean, rl = pam.fit_parallel(field, part, cfg, spec)
    assert any(r.centers % 2 for reps in rl.rounds for r in reps)  # odd M was exercised
    with E.options(cd_form="residual", tile_tau=0.0):
        gen, rg = pam.fit_parallel(field, part, cfg, spec)
    for a, b in zip(gen.locals, lean.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    for ra, rb in zip(rg.rounds, rl.rounds):
        for x, y in zip(ra, rb):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-10 * abs(x.objective)


def test_config1_convergent_solver_matches_reference(cuda, golden):
    """C1 with the library's convergent settings (tol=1e-10, max_iters=1e5):
    every fit converges like the reference's (24,556 sweeps on the step subdomains),
    beta and objective within 1e-8 relative, total sweeps within +-1 per fit."""
    import dataclasses

    g = golden("C1conv")
    wl = workloads.config1()
    assert str(g["input_digest"]) == __import__("hashlib").sha256(
        np.ascontiguousarray(wl.field.values).tobytes()).hexdigest()
    cfg = dataclasses.replace(wl.config, elastic=dataclasses.replace(wl.config.elastic, tol=1e-10,
                                                                     max_iters=100000))
    sur, rep = pam.fit_parallel(wl.field, wl.partition, cfg, wl.spec)
    ref_sweeps = sum(int(g[f"s{s}_iterations"]) for s in range(4))
    assert abs(rep.device["sweeps"] - ref_sweeps) <= 4
    for s in range(4):
        ref = g[f"s{s}_beta"]
        assert np.max(np.abs(sur.locals[s].beta - ref)) <= 1e-8 * max(1.0, np.abs(ref).max())
        obj = rep.rounds[s][0].objective
        assert abs(obj - float(g[f"s{s}_objective"])) <= 1e-8 * max(abs(float(g[f"s{s}_objective"])), 1e-300)


@pytest.mark.parametrize("cells", [(32, 32), (20, 20)])
@pytest.mark.parametrize("lattice", [1, 3, 4, 5, 7])
@pytest.mark.parametrize("max_iters,tol", [(4000, 1e-7), (1, 1e-6), (37, 1e-300)])
def test_blocked_kernel_edge_shapes_match_lean(cuda, cells, lattice, max_iters, tol):
    """The blocked CD (cd_block.cu) on its corner shapes against the lean per-column
    kernel: one column, a single block (the block follows itself across sweeps), 16
    columns exactly, two and four blocks, lists of <= 8 and > 8 columns per worker
    warp, 1,024 and 400 rows, early convergence, a single sweep and a sweep cap."""
    field = pam.box_field_2d(*cells)
    part = pam.make_partition(field.mesh, 1, 1)
    en = pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=tol, max_iters=max_iters)
    cfg = pam.AdaptiveConfig(m_max=0, elastic=en)
    spec = pam.DictionarySpec(sigma=0.6 / lattice, lattice=lattice)
    with E.options(cd_form="residual", cd_kernel="lean"):
        lean, rl = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="residual", cd_kernel="block"):
        blk, rb = pam.fit_parallel(field, part, cfg, spec)
    a, b = lean.locals[0], blk.locals[0]
    assert a.beta.shape == b.beta.shape == (lattice * lattice,)
    assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    x, y = rl.rounds[0][0], rb.rounds[0][0]
    assert abs(x.objective - y.objective) <= 1e-10 * abs(x.objective)
    sl, sb = int(rl.device["sweeps"]), int(rb.device["sweeps"])  # one fit, one round
    assert 1 <= sb <= max_iters
    if lattice > 1 or tol >= 1e-7:  # (one column reaches a rounding-level step after two sweeps)
        assert abs(sl - sb) <= 1
    if max_iters == 4000:
        assert sb < max_iters  # the stop rule fired before the cap
    elif lattice > 1:
        assert sb == max_iters


def test_blocked_kernel_many_small_fits_match_lean(cuda):
    """169 fits of 64 rows through the blocked CD: more fits than CTAs (the work queue
    hands a CTA several fits in turn), two-tile fits (most worker warps own no row of
    any column: empty lists), two refinement rounds."""
    field = pam.box_field_2d(104, 104)
    part = pam.make_partition(field.mesh, 13, 13)
    cfg = pam.AdaptiveConfig(k_top=8, m_max=24, m_q=3, max_rounds=2, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.5 / 104)
    with E.options(cd_form="residual", cd_kernel="lean"):
        lean, rl = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="residual", cd_kernel="block"):
        blk, rb = pam.fit_parallel(field, part, cfg, spec)
    for a, b in zip(lean.locals, blk.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    for ra, rb_ in zip(rl.rounds, rb.rounds):
        for x, y in zip(ra, rb_):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-10 * abs(x.objective)


@pytest.mark.parametrize("cells,px", [((32, 32), 1), ((24, 24), 2), ((40, 30), 1)])
def test_pipelined_few_fit_kernel_matches_lean(cuda, cells, px):
    """The software-pipelined CD for few fits (lag-1 Gram correction, cd.cu
    cd_pipe_kernel) against the lean per-column kernel: same dictionaries,
    sweeps within one, beta and objectives ~1e-12 (only dot-product rounding
    differs)."""
    field = pam.box_field_2d(*cells)
    part = pam.make_partition(field.mesh, px, 1)
    cfg = pam.AdaptiveConfig(k_top=24, m_max=150, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.5 / cells[0])
    with E.options(cd_form="residual", cd_kernel="lean"):  # few fits would pick the covariance form
        lean, rl = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="residual", cd_kernel="pair"):
        pipe, rp = pam.fit_parallel(field, part, cfg, spec)
    for a, b in zip(lean.locals, pipe.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    for ra, rb in zip(rl.rounds, rp.rounds):
        for x, y in zip(ra, rb):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-10 * abs(x.objective)


def test_wide_gram_form_for_few_fits_matches_residual(cuda):
    """Few fits with a wide dictionary (M > 512) in the covariance form (gram.cu
    wide configurations, the host's choice when the tile stream is unavailable):
    same dictionaries and reports as the residual form, beta ~1e-12."""
    field = pam.box_field_2d(32, 32)
    part = pam.make_partition(field.mesh, 1, 1)  # 1,024 cells, per-cell dictionary
    cfg = pam.AdaptiveConfig(k_top=24, m_max=150, m_q=3, max_rounds=3, elastic=EN_2D,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=1.0 / 32)
    assert E.cd_form([1024], [1024 + 144], tiles_ok=False) == "gram"  # dense residual would be chain-bound
    assert E.cd_form([1024], [1024 + 144]) == "residual"  # the blocked CD wins with tiles
    with E.options(cd_form="residual"):
        res, rr = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="gram"):
        gram, rg = pam.fit_parallel(field, part, cfg, spec)
    for a, b in zip(res.locals, gram.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-9 * max(1, np.abs(a.beta).max())
    for ra, rb in zip(rr.rounds, rg.rounds):
        for x, y in zip(ra, rb):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-9 * abs(x.objective)


def test_c5_device_generator(cuda):
    """On-device config-5 inputs (pam_c5_generate_f64): deterministic, the
    distributions of workloads.config5 (points in their half-open unit box,
    levels in [1e-3, 1e3] with at most 16 per box, centres within a quarter
    spacing of the lattice and inside the box), and they fit like the host
    generator's data (oracle parity on two boxes)."""
    p = workloads.config5_device(M=64, n_sub=64, n_pts=1000, seed=11)
    q = workloads.config5_device(M=64, n_sub=64, n_pts=1000, seed=11)
    np.testing.assert_array_equal(p.points, q.points)
    np.testing.assert_array_equal(p.values, q.values)
    np.testing.assert_array_equal(p.centres, q.centres)
    # a rank's shard (boxes 16..39) holds exactly those boxes' data
    sh = workloads.config5_device(M=64, n_sub=24, n_pts=1000, seed=11, first_box=16)
    np.testing.assert_array_equal(sh.points, p.points[16000:40000])
    np.testing.assert_array_equal(sh.values, p.values[16000:40000])
    np.testing.assert_array_equal(sh.centres, p.centres[16 * 64:40 * 64])
    np.testing.assert_array_equal(sh.box_lo, p.box_lo[16:40])
    pts = p.points.reshape(64, 1000, 3)
    assert np.all(pts >= p.box_lo[:, None, :]) and np.all(pts < p.box_hi[:, None, :])
    assert np.all(p.values >= 1e-3) and np.all(p.values <= 1e3)
    assert max(len(np.unique(p.values[s * 1000:(s + 1) * 1000])) for s in range(64)) <= 16
    assert np.mean(pts, axis=(0, 1)) == pytest.approx(np.mean(p.box_lo, axis=0) + 0.5, abs=0.01)
    cen = p.centres.reshape(64, 64, 3)
    m = np.arange(64)
    lat = (np.stack([m % 4, (m // 4) % 4, m // 16], axis=1) + 0.5) * 0.25  # (4,4,4) lattice, x fastest
    jit = cen - p.box_lo[:, None, :] - lat[None]
    assert np.all(np.abs(jit) <= 0.25 * 0.25 + 1e-12)  # jitter within a quarter spacing
    assert np.all(cen >= p.box_lo[:, None, :]) and np.all(cen <= p.box_hi[:, None, :])
    res = pam.fit_subdomains(p)
    c = p.config
    for s in (0, 63):
        a, b = p.row_off[s], p.row_off[s + 1]
        W = O.shepard_features(p.points[a:b], p.centres[s * 64:(s + 1) * 64], p.widths[s * 64:(s + 1) * 64])
        o = O.fit_log(p.values[a:b], W, c.elastic.lam1, c.elastic.lam2, c.elastic.tol, c.elastic.max_iters)
        assert np.max(np.abs(res.beta[s] - o["beta"])) <= BETA_TOL * max(1, np.abs(o["beta"]).max())


@pytest.mark.parametrize("cells,parts,tol", [((60, 60), (3, 3), 1e-6), ((48, 36), (2, 2), 1e-6),
                                             ((60, 60), (3, 3), 1e-3), ((50, 50), (5, 1), 1e-4)])
def test_dual_fit_kernel_matches_lean(cuda, cells, parts, tol):
    """Two fits per warp (cd.cu cd_dual_kernel, one fit per half-warp, 257-512
    rows) against the one-fit-per-warp lean kernel: odd fit counts (a lone
    half), ragged dictionaries after enrichment (padded columns), fits that
    converge at different sweeps (a finished half idles on zero columns).
    Same dictionaries, sweeps within one, beta and objectives ~1e-12."""
    field = pam.box_field_2d(*cells)
    part = pam.make_partition(field.mesh, *parts)
    en = pam.ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=tol, max_iters=1500)
    cfg = pam.AdaptiveConfig(k_top=40, m_max=240, m_q=3, max_rounds=3, elastic=en,
                             offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    spec = pam.DictionarySpec(sigma=0.5 / cells[0])
    with E.options(cd_form="residual", cd_kernel="lean"):
        lean, rl = pam.fit_parallel(field, part, cfg, spec)
    with E.options(cd_form="residual", cd_kernel="dual"):
        dual, rd = pam.fit_parallel(field, part, cfg, spec)
    for a, b in zip(lean.locals, dual.locals):
        np.testing.assert_array_equal(a.dictionary.centers, b.dictionary.centers)
        assert np.max(np.abs(a.beta - b.beta)) <= 1e-10 * max(1, np.abs(a.beta).max())
    for ra, rb in zip(rl.rounds, rd.rounds):
        for x, y in zip(ra, rb):
            assert (x.centers, x.added) == (y.centers, y.added)
            assert abs(x.objective - y.objective) <= 1e-10 * abs(x.objective)
