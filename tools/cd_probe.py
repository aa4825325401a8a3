"""Small CD probe for profiling one kernel choice on a BASELINE-shaped batch.

    python tools/cd_probe.py C2 --kernel block --iters 300 [--rounds 1] [--form residual]

Fits the config's subdomains with the solver capped at --iters sweeps (the CD
launch is then short enough for ncu --set full) and prints the CD seconds.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2605_16564_b200 as pam
    from paper_2605_16564_b200 import engine as E
    from paper_2605_16564_b200 import workloads

    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["C2", "C3", "C4"])
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--form", default="residual")
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--lib", default=None, help="alternative libpam_b200.so build (A/B of kernel variants)")
    args = ap.parse_args()
    if args.lib:
        from paper_2605_16564_b200 import _native
        _native.LIB_PATH = Path(args.lib).resolve()
    E.set_options(cd_form=args.form, cd_kernel=args.kernel)
    wl = {"C2": workloads.config2, "C3": workloads.config3,
          "C4": lambda: workloads.config4(with_refined_eval=False)}[args.config]()
    cfg = dataclasses.replace(wl.config, max_rounds=args.rounds,
                              elastic=dataclasses.replace(wl.config.elastic, max_iters=args.iters))
    for _ in range(args.repeat):
        sur, rep = pam.fit_parallel(wl.field, wl.partition, cfg, wl.spec)
        print(json.dumps({"config": args.config, "kernel": args.kernel, "form": args.form, "iters": args.iters,
                          "cd_s": rep.device["kernel_seconds"]["cd"],
                          "cd_bytes": rep.device.get("cd_bytes")}), flush=True)


if __name__ == "__main__":
    main()
