"""CD per-column time vs concurrent fits per SM (C4 subdomain shape).

Fits the SPE10-shaped field restricted to k z-slabs of 5 layers (6 x 22 x k
subdomains of 500 cells, the C4 fit per subdomain) with the default kernels
and reports, per adaptive round, the CD launch time divided by the columns
each fit visits ((sweeps + 1) * M): the time a warp needs per column at a
given number of concurrent fits per SM (the kernel puts one fit per warp,
16 warps per SM).  k = 1 leaves ~1 warp per SM (the dependency chain of one
fit in isolation), k = 17 is the full C4 batch.

    python tools/cd_occupancy.py 1 4 8 17
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2605_16564_b200 as pam
    from paper_2605_16564_b200 import workloads

    ks = [int(a) for a in sys.argv[1:]] or [1, 4, 8, 17]
    wl = workloads.config4(with_refined_eval=False)
    full = wl.field
    nx, ny, nz = full.mesh.counts
    for k in ks:
        nzk = 5 * k
        mesh = pam.build_mesh(3, (nx, ny, nzk), tuple((0.0, n * d) for n, d in
                                                      zip((nx, ny, nzk), workloads.SPE10_CELL)))
        # bottom k slabs of the C4 field (cell order x fastest, then y, then z)
        vals = full.values.reshape(nz, ny, nx)[:nzk].reshape(-1)
        field = pam.FieldData(mesh=mesh, values=vals)
        part = pam.make_partition(mesh, 6, 22, k)
        pam.fit_parallel(field, part, wl.config, wl.spec)  # warm-up (module load, allocator)
        _, rep = pam.fit_parallel(field, part, wl.config, wl.spec)
        rows = []
        for r in rep.device["cd_rounds"]:
            m = 500 + 300 * r["round"]
            cols = (wl.config.elastic.max_iters + 1) * m
            rows.append({"round": r["round"], "fits": r["fits"], "cd_s": r["seconds"],
                         "us_per_column": r["seconds"] / cols * 1e6,
                         "fits_per_sm": r["fits"] / 148})
        print(json.dumps({"slabs": k, "subdomains": part.n_subdomains, "rounds": rows}), flush=True)


if __name__ == "__main__":
    main()
