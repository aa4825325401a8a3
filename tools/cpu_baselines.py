"""CPU baselines of BASELINE configs 1-3 (full) and 5 (sampled) with the
REFERENCE itself (baseline/_ref, unmodified, numba CD) on all host cores.

    python tools/cpu_baselines.py C1 C2 C3 C5 > profiles/r02_cpu_baselines.jsonl

C1-C3: ``fieldfit.fit_parallel(workers=cores)`` over the whole configuration
(the reference's own process-pool fan-out, partition.py:188-195) and
``GlobalSurrogate.evaluate`` at the config's evaluation points (single
process, as the reference does it).  C5: a ProcessPoolExecutor(cores) over
the subdomain-level ``fit_adaptive`` (the 65,536-box sweep is
sampled, >= 256 boxes per M) + LocalSurrogate.evaluate of 2,000 points per
fitted box; throughput extrapolates as boxes / wall.  Inputs are the same
seeded generators the GPU path uses (paper_2605_16564_b200.workloads).
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    for ln in open("/proc/cpuinfo"):
        if ln.startswith("model name"):
            return ln.split(":", 1)[1].strip()
    return "unknown"


def r_cfg(cfg):
    from fieldfit.adaptive import AdaptiveConfig as RA
    from fieldfit.elastic_net import ElasticNetConfig as REN

    e = cfg.elastic
    return RA(k_top=cfg.k_top, m_max=cfg.m_max, eps_tol=cfg.eps_tol, eta=cfg.eta, m_q=cfg.m_q,
              max_rounds=cfg.max_rounds, offsets=cfg.offsets, quad_order=cfg.quad_order,
              elastic=REN(lam1=e.lam1, lam2=e.lam2, tol=e.tol, max_iters=e.max_iters))


def run_2d(name):
    import fieldfit as ff
    from fieldfit.elastic_net import _HAVE_NUMBA

    from paper_2605_16564_b200 import workloads

    assert _HAVE_NUMBA
    wl = {"C1": workloads.config1, "C2": workloads.config2, "C3": workloads.config3}[name]()
    m = wl.field.mesh
    mesh = ff.build_mesh(2, tuple(m.counts), tuple(tuple(b) for b in m.bounds))
    field = ff.FieldData(mesh=mesh, values=np.asarray(wl.field.values))
    part = ff.make_partition(mesh, *wl.shape)
    spec = ff.DictionarySpec(sigma=wl.spec.sigma, lattice=wl.spec.lattice)
    n = cores()
    t0 = time.perf_counter()
    sur, rep = ff.fit_parallel(field, part, r_cfg(wl.config), spec, workers=n)
    t_fit = time.perf_counter() - t0
    t0 = time.perf_counter()
    sur.evaluate(wl.eval_points)
    t_eval = time.perf_counter() - t0
    return {"config": name, "impl": "reference (baseline/_ref, numba)", "cores": n, "cpu_model": cpu_model(),
            "subdomains": part.n_subdomains, "fit_s": t_fit, "fits_per_s": part.n_subdomains / t_fit,
            "eval_points": int(len(wl.eval_points)), "eval_s": t_eval,
            "evals_per_s": len(wl.eval_points) / t_eval, "sample": "full configuration",
            "rounds_subdomain0": [r.centers for r in rep.rounds[0]]}


_P = {}


def _c5_init(M, n_sub):
    os.environ["OMP_NUM_THREADS"] = "1"
    from paper_2605_16564_b200 import workloads

    _P["p"] = workloads.config5(M=M, n_sub=n_sub, n_eval=0)


def _c5_one(s):
    from fieldfit.adaptive import fit_adaptive
    from fieldfit.fields import SubdomainField
    from fieldfit.geometry import Box
    from fieldfit.rbf import RbfDictionary

    p = _P["p"]
    M = int(p.dict_m[s])
    a, b = int(p.row_off[s]), int(p.row_off[s + 1])
    lo, hi = tuple(p.box_lo[s]), tuple(p.box_hi[s])
    sub = SubdomainField(box=Box(lo=lo, hi=hi, open_hi=(True, True, True)), cell_indices=np.arange(b - a),
                         centroids=p.points[a:b], values=p.values[a:b], cell_size=p.cell_size)
    d0 = RbfDictionary(centers=p.centres[s * M:(s + 1) * M], widths=p.widths[s * M:(s + 1) * M])
    t0 = time.perf_counter()
    sur, _ = fit_adaptive(sub, d0, r_cfg(p.config))
    t_fit = time.perf_counter() - t0
    pts = np.asarray(lo) + np.random.default_rng(s).random((2000, 3))
    t0 = time.perf_counter()
    sur.evaluate(pts)
    return t_fit, time.perf_counter() - t0


def run_c5(M, n_boxes=256):
    import multiprocessing as mp

    n = cores()
    with ProcessPoolExecutor(n, mp_context=mp.get_context("spawn"), initializer=_c5_init,
                             initargs=(M, n_boxes)) as pool:
        list(pool.map(_c5_one, range(n)))  # JIT + init every worker
        t0 = time.perf_counter()
        res = list(pool.map(_c5_one, range(n_boxes)))
        wall = time.perf_counter() - t0
    fit_core = sum(r[0] for r in res)
    ev_core = sum(r[1] for r in res)
    return {"config": f"C5 M={M}", "impl": "reference (baseline/_ref, numba)", "cores": n, "cpu_model": cpu_model(),
            "sample": f"{n_boxes} of 65,536 boxes (first {n_boxes} of workloads.config5(M, n_sub={n_boxes}))",
            "boxes": n_boxes, "wall_s": wall, "fits_per_s": n_boxes / wall,
            "fit_core_s_per_box": fit_core / n_boxes, "evals_per_s": n_boxes * 2000 / ev_core * n,
            "extrapolated_full_sweep_s": 65536 / (n_boxes / wall)}


def main():
    which = sys.argv[1:] or ["C1", "C2", "C3", "C5"]
    for w in which:
        if w == "C5":
            for M in (64, 128, 256, 512):
                print(json.dumps(run_c5(M)), flush=True)
        else:
            print(json.dumps(run_2d(w)), flush=True)


if __name__ == "__main__":
    main()
