"""K4 evaluation microbenchmark (BASELINE config 5 evaluation shape).

65,536 unit boxes tiling [0,64]x[0,32]x[0,32], each with an M-entry jittered
lattice dictionary and seeded coefficients, evaluated at
1e8 seeded uniform points through GlobalSurrogate.evaluate_device (locate +
owner sort + fused Shepard/exp kernel).  Coefficients are random: evaluation
cost does not depend on their values.  Prints one JSON line with points/s,
point-centre pairs/s and the FP64 roofline fraction under SURVEY §8d's flop
convention (M_owner*(3d+4+E) per point, E = 20).

    python tools/eval_bench.py --m 256 --points 1e8 --reps 3
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--points", type=float, default=1e8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--layers", type=int, default=32)
    args = ap.parse_args()

    import torch

    from paper_2605_16564_b200 import _native as nat
    from paper_2605_16564_b200.geometry import build_mesh
    from paper_2605_16564_b200.partition import DeviceSurrogate, GlobalSurrogate, make_partition
    from paper_2605_16564_b200.workloads import C5_LATTICE

    L = args.layers
    S = 64 * 32 * L
    g = np.array(C5_LATTICE[args.m])
    M = int(np.prod(g))
    rng = np.random.default_rng(5)
    # lattice in the unit box, x fastest, jittered by U(-1/4, 1/4) h and clamped
    h = 1.0 / g
    ax = [(np.arange(n) + 0.5) / n for n in g]
    Z, Y, X = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    lat = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)  # (M, 3)
    # subdomain order of make_partition: x fastest, then y, then z
    sidx = np.arange(S)
    lo = np.stack([sidx % 64, (sidx // 64) % 32, sidx // (64 * 32)], axis=1).astype(float)
    jit = (rng.random((S, M, 3)) - 0.5) * 0.5 * h
    cen = np.clip(lo[:, None, :] + lat[None] + jit, lo[:, None, :], lo[:, None, :] + 1.0)
    widths = np.full(S * M, float(h.mean()))
    beta = rng.standard_normal(S * M)
    dev = nat.device()
    off = np.arange(S, dtype=np.int64) * M
    ds = DeviceSurrogate(3, nat.to_dev(off), nat.to_dev(np.full(S, M, dtype=np.int32)),
                         nat.to_dev(cen.reshape(-1)), nat.to_dev(widths), nat.to_dev(beta),
                         torch.ones(S, dtype=torch.int32, device=dev))
    part = make_partition(build_mesh(3, (64, 32, L), ((0.0, 64.0), (0.0, 32.0), (0.0, float(L)))), 64, 32, L)
    gs = GlobalSurrogate(partition=part, locals=tuple([None] * S))
    gs.attach_device(ds)
    P = int(args.points * L / 32)
    gen = torch.Generator(device=dev).manual_seed(50)
    pts = torch.rand((P, 3), dtype=torch.float64, device=dev, generator=gen) * torch.tensor([64.0, 32.0, float(L)],
                                                                             dtype=torch.float64, device=dev)
    out = torch.empty(P, dtype=torch.float64, device=dev)
    work = torch.empty(int(nat.lib().pam_eval_workspace_bytes(P, S)), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    gs.evaluate_device(pts, out=out, work=work)  # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        gs.evaluate_device(pts, out=out, work=work)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    t = float(np.median(times))
    pairs = P * M
    flops = pairs * 33 + P * 20
    peak = nat.measure_fp64_peak() / 1e12  # measured DFMA peak (FMA = 2), like bench.py
    print(json.dumps({"workload": f"C5 eval: {S} boxes x M={M}, {P} uniform points", "seconds": t,
                      "points_per_s": P / t, "pairs_per_s": pairs / t, "gflops_convention": flops / t / 1e9,
                      "fp64_peak_tflops": peak, "frac": flops / t / 1e12 / peak,
                      "times": times, "checksum": float(out.sum().item())}), flush=True)


if __name__ == "__main__":
    main()
