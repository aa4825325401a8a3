"""Generate the committed golden fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture stores the reference's outputs for seeded inputs that the
GPU box regenerates deterministically from ``paper_2605_16564_b200.workloads``
(an input checksum is stored alongside so drift is detected).  3D cases use
the reference's dimension-generic subdomain-level functions
(SubdomainField / RbfDictionary / fit_adaptive with explicit 3D offsets,
SURVEY F4), fed by this repo's 3D mesh/partition restatement, which is
itself pinned against the reference formulas in tests/test_oracle_pins.py.
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent

import fieldfit as ff  # noqa: E402  (the reference)
from fieldfit.adaptive import AdaptiveConfig as RAdaptive  # noqa: E402
from fieldfit.adaptive import fit_adaptive as r_fit_adaptive  # noqa: E402
from fieldfit.adaptive import mark as r_mark, enrich as r_enrich  # noqa: E402
from fieldfit.elastic_net import ElasticNetConfig as REN, fit as r_fit  # noqa: E402
from fieldfit.fields import SubdomainField as RSub  # noqa: E402
from fieldfit.geometry import Box as RBox  # noqa: E402
from fieldfit.rbf import RbfDictionary as RDict, shepard_features as r_features, shepard_eval as r_eval  # noqa: E402

from paper_2605_16564_b200 import workloads  # noqa: E402  (host-only generators)
from oracle import pam_oracle as O  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def r_cfg(cfg):
    e = cfg.elastic
    return RAdaptive(k_top=cfg.k_top, m_max=cfg.m_max, eps_tol=cfg.eps_tol, eta=cfg.eta, m_q=cfg.m_q,
                     max_rounds=cfg.max_rounds, offsets=cfg.offsets, quad_order=cfg.quad_order,
                     elastic=REN(lam1=e.lam1, lam2=e.lam2, tol=e.tol, max_iters=e.max_iters))


def run_subdomain(field, shape, s, cfg, spec, n_probe=64, seed=0):
    """Reference fit of subdomain s of a workload (what _fit_one does, partition.py:157-164)."""
    mesh = field.mesh
    boxes, owner, _ = O.partition_boxes(mesh.counts, mesh.bounds, shape)
    lo, hi, op = boxes[s]
    box = RBox(lo=lo, hi=hi, open_hi=op)
    rows = O.subdomain_rows(mesh.centroids, boxes[s])
    sub = RSub(box=box, cell_indices=rows, centroids=mesh.centroids[rows], values=field.values[rows],
               cell_size=mesh.cell_size)
    if spec.lattice is None:
        d0 = RDict(centers=sub.centroids, widths=np.full(rows.size, spec.sigma))
    else:
        d0 = RDict(centers=O.lattice_centers(lo, hi, spec.lattice),
                   widths=np.full(spec.lattice ** mesh.dim, spec.sigma))
    t = time.time()
    sur, reps = r_fit_adaptive(sub, d0, r_cfg(cfg))
    dt = time.time() - t
    rng = np.random.default_rng(seed + s)
    probe = np.asarray(lo) + rng.random((n_probe, mesh.dim)) * (np.asarray(hi) - np.asarray(lo))
    vals = sur.evaluate(probe)
    rep = np.array([[r.round, r.centers, r.added, r.max_residual, r.rel_l2, r.abs_l2, r.objective]
                    for r in reps])
    return dict(rows=rows, centers=sur.dictionary.centers, widths=sur.dictionary.widths,
                generations=sur.dictionary.generations, beta=sur.beta, reports=rep, probe=probe,
                probe_values=vals, seconds=dt)


def save_case(name, field, shape, subs, cfg, spec, extra=None):
    out = {"input_digest": digest(field.values), "shape": np.array(shape),
           "subdomains": np.array(subs)}
    for s in subs:
        t = time.time()
        r = run_subdomain(field, shape, s, cfg, spec)
        for k, v in r.items():
            if k != "seconds":
                out[f"s{s}_{k}"] = v
        print(f"  {name} subdomain {s}: centres {r['reports'][:, 1].astype(int).tolist()} "
              f"({time.time() - t:.1f}s)", flush=True)
    if extra:
        out.update(extra)
    np.savez_compressed(OUT / f"{name}.npz", **out)


def kernels_case():
    """Feature/eval/CD/mark/enrich vectors from the reference's own functions."""
    rng = np.random.default_rng(1234)
    out = {}
    for dim in (1, 2, 3):
        M, N = 37, 53
        c = rng.random((M, dim))
        w = rng.uniform(0.05, 0.3, M)
        x = rng.random((N, dim))
        d = RDict(centers=c, widths=w)
        out[f"feat{dim}_c"], out[f"feat{dim}_w"], out[f"feat{dim}_x"] = c, w, x
        out[f"feat{dim}_L"] = d.log_features(x)
        out[f"feat{dim}_W"] = r_features(x, d)
        b = rng.standard_normal(M)
        out[f"feat{dim}_beta"] = b
        out[f"feat{dim}_eval"] = r_eval(x, d, b)
    # CD fits at several shapes / tolerances (elastic_net.py:66-110)
    for k, (n, m, l1, l2, tol, it) in enumerate([(40, 25, 0.05, 0.01, 1e-10, 100000),
                                                 (100, 150, 4.59e-4, 1e-4, 1e-6, 4000),
                                                 (257, 64, 0.01, 0.0, 1e-12, 20000),
                                                 (600, 300, 4.59e-4, 1e-4, 1e-6, 700)]):
        W = np.abs(rng.standard_normal((n, m)))
        W /= W.sum(axis=1, keepdims=True)
        y = rng.standard_normal(n)
        b0 = rng.standard_normal(m) * 0.1 if k == 1 else None
        res = r_fit(W, y, REN(lam1=l1, lam2=l2, tol=tol, max_iters=it), beta0=b0)
        out[f"cd{k}_W"], out[f"cd{k}_y"] = W, y
        out[f"cd{k}_params"] = np.array([l1, l2, tol, it])
        if b0 is not None:
            out[f"cd{k}_beta0"] = b0
        out[f"cd{k}_beta"], out[f"cd{k}_hist"] = res.beta, res.objective_history
        out[f"cd{k}_iters"] = np.array([res.iterations, int(res.converged)])
    # mark with ties (adaptive.py:141-152)
    R = np.round(rng.random(300) * 20) / 20
    R[::7] = 0.0
    out["mark_R"] = R
    out["mark_out"] = r_mark(R, 50)
    # enrich 2D with duplicates against the existing dictionary (adaptive.py:167-210)
    f = ff.box_field_2d(8, 8)
    sub = f.whole()
    d = RDict(centers=sub.centroids, widths=np.full(64, 0.1))
    mk = np.array([3, 9, 27, 63, 0])
    nc, nw = r_enrich(d, mk, sub, 0.5, 3, offsets=((0.0, 0.0), (-0.5, 0.0), (0.5, 0.5)))
    d2 = d.extended(nc, nw, 1)
    nc2, nw2 = r_enrich(d2, mk, sub, 0.5, 3, offsets=((0.0, 0.0), (-0.5, 0.0), (0.5, 0.5)))
    out["enr_centers2"], out["enr_widths2"] = d2.centers, d2.widths
    out["enr_new1_c"], out["enr_new1_w"], out["enr_new2_c"], out["enr_new2_w"] = nc, nw, nc2, nw2
    np.savez_compressed(OUT / "kernels.npz", **out)
    print("  kernels.npz written")


def adaptive_small_cases():
    """Reference fit_adaptive on the reference's own test fields (1D/2D) and a 3D field."""
    out = {}
    # 1D step (tests/test_adaptive.py:166-172): centers [16, 22, 28]
    f = ff.step_field_1d(16)
    sub = f.whole()
    cfg = RAdaptive(k_top=2, m_max=12, eta=0.5, m_q=3, max_rounds=3,
                    elastic=REN(lam1=4.59e-4, lam2=4.64e-6))
    sur, reps = r_fit_adaptive(sub, ff.centroid_dictionary(sub.centroids, 0.0019), cfg)
    out["a1_centers"], out["a1_widths"], out["a1_beta"] = sur.dictionary.centers, sur.dictionary.widths, sur.beta
    out["a1_reports"] = np.array([[r.centers, r.added, r.max_residual, r.rel_l2, r.objective] for r in reps])
    # 2D box field (tests/test_adaptive.py:212-223 at 16x16)
    f = ff.box_field_2d(16, 16)
    sub = f.whole()
    cfg = RAdaptive(k_top=51, m_max=306, eta=0.5, m_q=3, max_rounds=3,
                    elastic=REN(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=1500),
                    offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    sur, reps = r_fit_adaptive(sub, ff.centroid_dictionary(sub.centroids, 0.0625), cfg)
    out["a2_centers"], out["a2_widths"], out["a2_beta"] = sur.dictionary.centers, sur.dictionary.widths, sur.beta
    out["a2_gens"] = sur.dictionary.generations
    out["a2_reports"] = np.array([[r.centers, r.added, r.max_residual, r.rel_l2, r.objective] for r in reps])
    # 3D: 6x5x4 cells of the SPE10-shaped field, explicit 3D offsets, order-2 quadrature
    fld = workloads.spe10_like_field(4)
    mesh = fld.mesh
    rows = np.array([((iz * 220 + iy) * 60 + ix) for iz in range(40, 44) for iy in range(10, 15)
                     for ix in range(20, 26)])
    box = RBox(lo=(400.0, 100.0, 80.0), hi=(520.0, 150.0, 88.0), open_hi=(True, True, True))
    sub = RSub(box=box, cell_indices=rows, centroids=mesh.centroids[rows], values=fld.values[rows],
               cell_size=mesh.cell_size)
    cfg = RAdaptive(k_top=24, m_max=144, eta=0.5, m_q=3, max_rounds=3, quad_order=2,
                    elastic=REN(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=1000),
                    offsets=workloads.IN_CELL_3D)
    sigma = float(np.prod(mesh.cell_size) ** (1 / 3))
    sur, reps = r_fit_adaptive(sub, RDict(centers=sub.centroids, widths=np.full(rows.size, sigma)), cfg)
    out["a3_rows"] = rows
    out["a3_centers"], out["a3_widths"], out["a3_beta"] = sur.dictionary.centers, sur.dictionary.widths, sur.beta
    out["a3_gens"] = sur.dictionary.generations
    out["a3_reports"] = np.array([[r.centers, r.added, r.max_residual, r.rel_l2, r.objective] for r in reps])
    np.savez_compressed(OUT / "adaptive_small.npz", **out)
    print("  adaptive_small.npz written", [r.centers for r in reps])


def geometry_case():
    """Reference mesh / partition / quadrature / lattice outputs (1D and 2D)."""
    from fieldfit.geometry import build_mesh as r_mesh, cell_quadrature as r_cq
    from fieldfit.partition import make_partition as r_part
    from fieldfit.rbf import lattice_dictionary as r_lat

    out = {}
    cases = [(1, (12,), ((0.2, 1.7),), (3,)), (2, (17, 9), ((0.2, 1.7), (-1.0, 2.0)), (1, 3)),
             (2, (60, 220), ((0.0, 1200.0), (0.0, 2200.0)), (6, 22)),
             (2, (12, 10), ((0.1, 1.7), (-3.3, 2.9)), (4, 5))]
    for k, (dim, counts, bounds, shape) in enumerate(cases):
        mesh = r_mesh(dim, counts, bounds)
        part = r_part(mesh, *shape)
        out[f"g{k}_centroids"] = mesh.centroids
        out[f"g{k}_owner"] = part.cell_to_subdomain
        out[f"g{k}_lo"] = np.array([b.lo for b in part.boxes])
        out[f"g{k}_hi"] = np.array([b.hi for b in part.boxes])
        out[f"g{k}_open"] = np.array([b.open_hi for b in part.boxes])
        pts, w = r_cq(mesh.centroids[:5], mesh.cell_size, 2)
        out[f"g{k}_q2"], out[f"g{k}_q2w"] = pts, w
        out[f"g{k}_lattice"] = r_lat(part.boxes[-1], 3, 0.1).centers
    np.savez_compressed(OUT / "geometry.npz", **out)
    print("  geometry.npz written")


def persistence_case():
    """Reference `dumps` text of a surrogate with awkward values (-0.0, denormals, 1e+/-300)."""
    from fieldfit.partition import dumps as r_dumps, make_partition as r_part
    from fieldfit.geometry import build_mesh as r_mesh

    rng = np.random.default_rng(99)
    part = r_part(r_mesh(2, (8, 6), ((0.0, 1.0), (-2.0, 1.0))), 2, 3)
    out, locs = {}, []
    for i, b in enumerate(part.boxes):
        n = 5 + i
        c = np.asarray(b.lo) + rng.random((n, 2)) * (np.asarray(b.hi) - np.asarray(b.lo))
        w = rng.uniform(1e-5, 0.3, n)
        be = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
        be[0], be[1] = -0.0, 5e-324
        g = rng.integers(0, 5, n)
        out[f"c{i}"], out[f"w{i}"], out[f"b{i}"], out[f"g{i}"] = c, w, be, g
        locs.append(ff.LocalSurrogate(dictionary=RDict(centers=c, widths=w, generations=g), beta=be))
    text = r_dumps(ff.GlobalSurrogate(partition=part, locals=tuple(locs),
                                      metadata={"config": "golden persistence", "field_checksum": "abc"}))
    np.savez_compressed(OUT / "persistence.npz", **out)
    (OUT / "surrogate_ref.txt").write_text(text)
    print("  persistence fixtures written")


def c1_convergent_case():
    """C1 with the library's convergent solver settings (tol=1e-10, max_iters=1e5; SURVEY
    Appendix A): the reference's own fit() on each subdomain's lattice design matrix."""
    wl = workloads.config1()
    mesh = wl.field.mesh
    boxes, _, _ = O.partition_boxes(mesh.counts, mesh.bounds, wl.shape)
    e = wl.config.elastic
    cfg = REN(lam1=e.lam1, lam2=e.lam2, tol=1e-10, max_iters=100000)
    out = {"input_digest": digest(wl.field.values), "tol": 1e-10, "max_iters": 100000}
    for s in range(len(boxes)):
        lo, hi, _ = boxes[s]
        rows = O.subdomain_rows(mesh.centroids, boxes[s])
        d0 = RDict(centers=O.lattice_centers(lo, hi, wl.spec.lattice),
                   widths=np.full(wl.spec.lattice ** mesh.dim, wl.spec.sigma))
        W = r_features(mesh.centroids[rows], d0)
        t = time.time()
        res = r_fit(W, np.log(wl.field.values[rows]), cfg)
        out[f"s{s}_beta"] = res.beta
        out[f"s{s}_iterations"] = res.iterations
        out[f"s{s}_converged"] = res.converged
        out[f"s{s}_objective"] = res.objective
        print(f"  C1conv subdomain {s}: {res.iterations} sweeps, converged={res.converged} "
              f"({time.time() - t:.1f}s)", flush=True)
    np.savez_compressed(OUT / "C1conv.npz", **out)


def darcy_case():
    """The reference's P1 Darcy solver on four problems (direct and CG paths, holes, Neumann,
    source, 1D, and a fitted surrogate as the coefficient)."""
    from fieldfit import darcy as rd

    out = {}
    coef = lambda p: np.exp(np.sin(3 * p[:, 0]) * np.cos(2 * p[:, 1]))  # noqa: E731
    cases = {
        "d1": rd.DarcyProblem(mesh=rd.triangulate(40, 30, ((0.0, 2.0), (0.0, 1.0))), coefficient=coef,
                              dirichlet={"left": 1.0, "right": 0.0}),
        "d2": rd.DarcyProblem(mesh=rd.triangulate(160, 140, ((0.0, 1.0), (0.0, 1.0)), holes=[(0.5, 0.5, 0.12)]),
                              coefficient=lambda p: 10.0 ** (np.where(p[:, 0] > 0.3, 1.0, -0.5)
                                                            + 0.3 * np.sin(7 * p[:, 1])),
                              dirichlet={"left": lambda p: 1.0 + p[:, 1], "right": 0.0},
                              neumann={"top": 0.3}, source=1.0),
        "d3": rd.DarcyProblem(mesh=rd.line_mesh(50, (0.0, 2.0)), coefficient=lambda p: np.exp(p[:, 0]),
                              dirichlet={"left": 1.0}, neumann={"right": 0.5}, source=2.0),
    }
    field = ff.box_field_2d(16, 16)
    part = ff.make_partition(field.mesh, 2, 2)
    sur, _ = ff.fit_parallel(field, part, ff.AdaptiveConfig(
        k_top=12, m_max=72, m_q=3, max_rounds=2, offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)),
        elastic=REN(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=400)), ff.DictionarySpec(sigma=0.0625))
    import io as _io
    buf = _io.StringIO()
    ff.save(sur, buf)
    out["d4_surrogate"] = np.array(buf.getvalue())
    cases["d4"] = rd.DarcyProblem(mesh=rd.triangulate(30, 30, ((0.0, 1.0), (0.0, 1.0))),
                                  coefficient=sur.evaluate, dirichlet={"bottom": 0.0, "top": 1.0})
    for name, prob in cases.items():
        sol = rd.solve_darcy(prob)
        A, b = sol.system
        A = A.tocsr()
        A.sort_indices()
        out[f"{name}_values"] = sol.values
        out[f"{name}_iterations"] = sol.diagnostics["iterations"]
        out[f"{name}_method"] = np.array(sol.diagnostics["method"])
        out[f"{name}_A_data"], out[f"{name}_A_indices"], out[f"{name}_A_indptr"] = A.data, A.indices, A.indptr
        out[f"{name}_b"] = b
        if prob.mesh.dim == 2:
            out[f"{name}_reaction_left"] = sol.boundary_reaction(list(prob.dirichlet)[0])
        print(f"  darcy {name}: {sol.diagnostics}", flush=True)
    np.savez_compressed(OUT / "darcy.npz", **out)


def main(which):
    if "persistence" in which:
        persistence_case()
    if "geometry" in which:
        geometry_case()
    if "kernels" in which:
        kernels_case()
    if "adaptive" in which:
        adaptive_small_cases()
    if "C1" in which:
        wl = workloads.config1()
        save_case("C1", wl.field, wl.shape, [0, 1, 2, 3], wl.config, wl.spec)
    if "darcy" in which:
        darcy_case()
    if "C1conv" in which:
        c1_convergent_case()
    if "C2" in which:
        wl = workloads.config2()
        save_case("C2", wl.field, wl.shape, [19, 42], wl.config, wl.spec)
    if "C3" in which:
        wl = workloads.config3()
        save_case("C3", wl.field, wl.shape, [77], wl.config, wl.spec)
    if "C4" in which:
        wl = workloads.config4(with_refined_eval=False)
        save_case("C4", wl.field, wl.shape, [0, 500, 1337, 2243], wl.config, wl.spec)


if __name__ == "__main__":
    main(sys.argv[1:] or ["kernels", "adaptive", "C1", "C2", "C3", "C4"])
