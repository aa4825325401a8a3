"""Wall time of the full BASELINE configs 1-4 through the public API on one GPU.

For each config: fit_parallel (all subdomains, all adaptive rounds) and
GlobalSurrogate.evaluate at the config's evaluation points, host arrays in and
out (the call a user makes), after one warm-up run.  The CPU reference times
for the same configs are in SURVEY.md §8d / Appendix B (C2 ~3 min, C3 ~20 min
on 8 cores) and the bench's CPU arm (C4).

    python tools/config_times.py C1 C2 C3 [--form residual|gram|auto] [--kernel block|pair|lean|auto]
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

    import argparse

    from paper_2605_16564_b200 import engine as E

    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["C1", "C2", "C3"])
    ap.add_argument("--form", default="auto")
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--tau", type=float, default=None)
    args = ap.parse_args()
    E.set_options(cd_form=args.form, cd_kernel=args.kernel)
    if args.tau is not None:
        E.set_options(tile_tau=args.tau)
    names = args.names
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
        print(json.dumps({"config": name, "form": args.form, "kernel": args.kernel,
                          "cd_s": rep.device["kernel_seconds"]["cd"],
                          "kernel_seconds": rep.device["kernel_seconds"],
                          "subdomains": part.n_subdomains, "cells": int(wl.field.mesh.n_cells),
                          "fit_s": t1 - t0, "eval_points": int(len(wl.eval_points)), "eval_s": t2 - t1,
                          "fits_per_s": part.n_subdomains / (t1 - t0), "rounds_subdomain0": rounds,
                          "eval_checksum": float(np.sum(np.log(vals)))}), flush=True)


if __name__ == "__main__":
    main()
