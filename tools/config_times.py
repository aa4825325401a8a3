"""Wall time of the full BASELINE configs 1-4 through the public API on one GPU.

For each config: fit_parallel (all subdomains, all adaptive rounds) and
GlobalSurrogate.evaluate at the config's evaluation points, host arrays in and
out (the call a user makes), after one warm-up run.  The CPU reference times
for the same configs are in SURVEY.md §8d / Appendix B (C2 ~3 min, C3 ~20 min
on 8 cores) and the bench's CPU arm (C4).

    python tools/config_times.py C1 C2 C3
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np

    import paper_2605_16564_b200 as pam
    from paper_2605_16564_b200 import workloads

    names = sys.argv[1:] or ["C1", "C2", "C3"]
    makers = {"C1": workloads.config1, "C2": workloads.config2, "C3": workloads.config3,
              "C4": workloads.config4}
    for name in names:
        wl = makers[name]()
        part = wl.partition
        pam.fit_parallel(wl.field, part, wl.config, wl.spec)  # warm-up
        t0 = time.perf_counter()
        sur, rep = pam.fit_parallel(wl.field, part, wl.config, wl.spec)
        t1 = time.perf_counter()
        vals = sur.evaluate(wl.eval_points)
        t2 = time.perf_counter()
        rounds = [r.centers for r in rep.rounds[0]]
        print(json.dumps({"config": name, "subdomains": part.n_subdomains, "cells": int(wl.field.mesh.n_cells),
                          "fit_s": t1 - t0, "eval_points": int(len(wl.eval_points)), "eval_s": t2 - t1,
                          "fits_per_s": part.n_subdomains / (t1 - t0), "rounds_subdomain0": rounds,
                          "eval_checksum": float(np.sum(np.log(vals)))}), flush=True)


if __name__ == "__main__":
    main()
