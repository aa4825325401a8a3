"""Wide golden fixtures: the REFERENCE run on many subdomains of every config.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_wide.py [C2all C3wide C4wide C5]

Per subdomain the fixture keeps what the GPU parity tests compare:
  * ``s{i}_dict``   sha256 of the reference dictionary bytes (centres, widths,
    generations) -- a bit-exact comparison of the selected-centre set;
  * ``s{i}_m``      its size;
  * ``s{i}_beta``   the reference coefficients (1e-8 relative check);
  * ``s{i}_reports`` (round, centers, added, max_residual, rel_l2, abs_l2,
    objective) per round;
  * ``s{i}_probe`` / ``s{i}_probe_values``: 16 seeded points in the box and
    the reference ``LocalSurrogate.evaluate`` there.
The inputs are regenerated on the GPU box by ``paper_2605_16564_b200.workloads``
(input digest stored).  C5 uses the reference's dimension-generic
subdomain-level API (SubdomainField + RbfDictionary + fit_adaptive, SURVEY
F4) on the first 64 boxes of ``workloads.config5(M, n_sub=64)``.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
from multiprocessing import Pool
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent

N_PROBE = 16


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def dict_digest(centers, widths, generations) -> str:
    return digest(np.asarray(centers, dtype=np.float64), np.asarray(widths, dtype=np.float64),
                  np.asarray(generations, dtype=np.int64))


_WL = {}


def _workload(name):
    from paper_2605_16564_b200 import workloads

    if name not in _WL:
        if name == "C2":
            _WL[name] = workloads.config2(n_eval=0)
        elif name == "C3":
            _WL[name] = workloads.config3(eval_n=1)
        elif name == "C4":
            _WL[name] = workloads.config4(with_refined_eval=False)
        elif name.startswith("C5_"):
            _WL[name] = workloads.config5(M=int(name[3:]), n_sub=64, n_eval=0)
    return _WL[name]


def _r_cfg(cfg):
    from fieldfit.adaptive import AdaptiveConfig as RAdaptive
    from fieldfit.elastic_net import ElasticNetConfig as REN

    e = cfg.elastic
    return RAdaptive(k_top=cfg.k_top, m_max=cfg.m_max, eps_tol=cfg.eps_tol, eta=cfg.eta, m_q=cfg.m_q,
                     max_rounds=cfg.max_rounds, offsets=cfg.offsets, quad_order=cfg.quad_order,
                     elastic=REN(lam1=e.lam1, lam2=e.lam2, tol=e.tol, max_iters=e.max_iters))


def _task(args):
    """Reference fit of one subdomain (what _fit_one does, partition.py:157-164)."""
    name, s = args
    from fieldfit.adaptive import fit_adaptive as r_fit_adaptive
    from fieldfit.fields import SubdomainField as RSub
    from fieldfit.geometry import Box as RBox
    from fieldfit.rbf import RbfDictionary as RDict
    from oracle import pam_oracle as O

    wl = _workload(name)
    t = time.time()
    if name.startswith("C5_"):
        p = wl
        M = int(p.dict_m[s])
        a, b = int(p.row_off[s]), int(p.row_off[s + 1])
        lo, hi = tuple(p.box_lo[s]), tuple(p.box_hi[s])
        box = RBox(lo=lo, hi=hi, open_hi=(True, True, True))
        sub = RSub(box=box, cell_indices=np.arange(b - a), centroids=p.points[a:b], values=p.values[a:b],
                   cell_size=p.cell_size)
        d0 = RDict(centers=p.centres[s * M:(s + 1) * M], widths=p.widths[s * M:(s + 1) * M])
        cfg = p.config
    else:
        mesh = wl.field.mesh
        boxes, _, _ = O.partition_boxes(mesh.counts, mesh.bounds, wl.shape)
        lo, hi, op = boxes[s]
        box = RBox(lo=lo, hi=hi, open_hi=op)
        rows = O.subdomain_rows(mesh.centroids, boxes[s])
        sub = RSub(box=box, cell_indices=rows, centroids=mesh.centroids[rows], values=wl.field.values[rows],
                   cell_size=mesh.cell_size)
        spec = wl.spec
        if spec.lattice is None:
            d0 = RDict(centers=sub.centroids, widths=np.full(rows.size, spec.sigma))
        else:
            d0 = RDict(centers=O.lattice_centers(lo, hi, spec.lattice),
                       widths=np.full(spec.lattice ** mesh.dim, spec.sigma))
        cfg = wl.config
    sur, reps = r_fit_adaptive(sub, d0, _r_cfg(cfg))
    rng = np.random.default_rng(1000 + s)
    probe = np.asarray(lo) + rng.random((N_PROBE, len(lo))) * (np.asarray(hi) - np.asarray(lo))
    d = sur.dictionary
    rep = np.array([[r.round, r.centers, r.added, r.max_residual, r.rel_l2, r.abs_l2, r.objective]
                    for r in reps])
    return name, s, dict(dict=dict_digest(d.centers, d.widths, d.generations), m=len(d.widths),
                         beta=np.asarray(sur.beta), reports=rep, probe=probe,
                         probe_values=sur.evaluate(probe)), time.time() - t


def c4_stratified():
    """>= 64 C4 subdomains: 32 in the log-normal layers (z-box < 7), 32 in the channel layers."""
    rng = np.random.default_rng(404)
    per_layer = 6 * 22
    logn = rng.choice(7 * per_layer, 32, replace=False)
    chan = 7 * per_layer + rng.choice(10 * per_layer, 32, replace=False)
    return sorted(set(logn.tolist()) | set(chan.tolist()) | {0, 500, 1337, 2243})


CASES = {
    "C2all": ("C2", list(range(64))),
    "C3wide": ("C3", sorted(set(range(0, 256, 8)) | {77, 255})),
    "C4wide": ("C4", c4_stratified()),
}


def acceptance5_case():
    """The paper's Table-2 experiment (reference tests/test_acceptance.py:77-89, 202-210):
    32x32 box field, 1x1 partition, sigma 0.031, k_top=204, m_max=1836, 4 rounds ->
    centre counts [1024, 1636, 2248, 2860]; the only path to the widest Gram-form CD."""
    import fieldfit as ff
    from fieldfit.adaptive import AdaptiveConfig as RAdaptive
    from fieldfit.elastic_net import ElasticNetConfig as REN

    field = ff.box_field_2d()
    part = ff.make_partition(field.mesh, 1, 1)
    cfg = RAdaptive(k_top=204, m_max=1836, eta=0.5, m_q=3, max_rounds=4,
                    elastic=REN(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=4000),
                    offsets=((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0)))
    t = time.time()
    sur, rep = ff.fit_parallel(field, part, cfg, ff.DictionarySpec(sigma=0.031))
    loc = sur.locals[0]
    reps = rep.rounds[0]
    rng = np.random.default_rng(5)
    probe = rng.random((256, 2))
    d = loc.dictionary
    out = {"input_digest": digest(field.values), "subdomains": np.array([0]),
           "s0_dict": dict_digest(d.centers, d.widths, d.generations), "s0_m": len(d.widths),
           "s0_beta": np.asarray(loc.beta),
           "s0_reports": np.array([[r.round, r.centers, r.added, r.max_residual, r.rel_l2, r.abs_l2, r.objective]
                                   for r in reps]),
           "s0_probe": probe, "s0_probe_values": sur.evaluate(probe)}
    np.savez_compressed(OUT / "ACC5.npz", **out)
    print(f"wrote ACC5.npz: counts {[r.centers for r in reps]} ({time.time() - t:.0f}s)", flush=True)


def main(which):
    if "ACC5" in which:
        acceptance5_case()
        which = [w for w in which if w != "ACC5"]
        if not which:
            return
    tasks, files = [], {}
    for key in which:
        if key == "C5":
            for M in (64, 128, 256, 512):
                files[f"C5_M{M}"] = (f"C5_{M}", list(range(64)))
        else:
            files[key] = CASES[key]
    for fname, (wname, subs) in files.items():
        tasks += [(wname, s) for s in subs]
    # longest first: C3 > C2 > C4 > C5
    weight = {"C3": 0, "C2": 1, "C4": 2}
    tasks.sort(key=lambda t: (weight.get(t[0], 3), t[1]))
    results = {}
    t0 = time.time()
    with Pool(int(os.environ.get("GOLDEN_PROCS", os.cpu_count()))) as pool:
        for k, (wname, s, res, dt) in enumerate(pool.imap_unordered(_task, tasks)):
            results[(wname, s)] = res
            print(f"[{k + 1}/{len(tasks)}] {wname} s{s}: m={res['m']} "
                  f"rounds={res['reports'][:, 1].astype(int).tolist()} {dt:.1f}s "
                  f"(elapsed {time.time() - t0:.0f}s)", flush=True)
    for fname, (wname, subs) in files.items():
        wl = _workload(wname)
        vals = wl.values if wname.startswith("C5_") else wl.field.values
        out = {"input_digest": digest(vals), "subdomains": np.array(subs)}
        for s in subs:
            for k, v in results[(wname, s)].items():
                out[f"s{s}_{k}"] = v
        np.savez_compressed(OUT / f"{fname}.npz", **out)
        print(f"wrote {fname}.npz ({len(subs)} subdomains)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C5", "C4wide", "C2all", "C3wide"])
