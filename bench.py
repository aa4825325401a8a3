#!/usr/bin/env python
"""bench.py — B200 PAM hot-path benchmark (BASELINE.json metric).

Workload: BASELINE config 4, the SPE10-shaped 3D field (60x220x85 = 1,122,000
cells, 20x10x2 ft), 6x22x17 = 2,244 subdomains of 500 cells, per-cell
dictionaries, 2 adaptive refinement levels (3 rounds, up to 1,100 centres),
the reference 2D-preset solver (lam1=4.59e-4, lam2=1e-4, tol=1e-6,
max_iters=4000); evaluation at all 1,122,000 cell centres and all 8,976,000
2x-refined cell centres.  A step = fit every subdomain (all rounds) +
evaluate all 10,098,000 points.

value     subdomain fits/s (whole job), inputs resident in HBM;
evals     RBF evaluations/s of the evaluation pass alone (same steps);
e2e       the same through the public API with host buffers
          (fit_parallel(FieldData) + GlobalSurrogate.evaluate(numpy points));
roofline  the dominant kernel (batched CD): algorithmic design-matrix bytes
          / CD device time vs the measured HBM copy bandwidth;
cpu_baseline  the CPU oracle port on this host's cores, bounded sample.

--impl reference times the reference's CPU algorithm (the bit-exact oracle
port: numpy + the C restatement of the numba CD core) on all host cores.
Multi-GPU (torchrun): one full SPE10-shaped realisation per rank (seed 4 +
rank), no collective on the data path; scaling "weak".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "subdomain fits/s + RBF evals/s at SPE10 shape; % of HBM/FP64 roofline"
UNIT = "subdomain-fits/s"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
                for b, name in REASON_BITS.items():
                    if bits & b and name != "gpu_idle":
                        reasons.add(name)
                if len(parts) > 3:
                    power.append(float(parts[3]))
            except ValueError:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------
# CPU arm: the REFERENCE itself (baseline/_ref, unmodified, numba CD) on the
# host cores -- the reference arm and the cpu_baseline leg.  Without the
# installed reference the bit-exact oracle port (oracle/) stands in.

REF_DIR = ROOT / "baseline" / "_ref"
_CPU = {}


def cpu_kind() -> str:
    return "reference" if (REF_DIR / "fieldfit").is_dir() else "port"


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cpu_init(kind: str, seed: int):
    """Pool initializer: build the C4 field and the partition once per worker
    (outside every timed region) and JIT the reference's CD core."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import pam_oracle as O
    from paper_2605_16564_b200 import workloads

    wl = workloads.config4(seed=seed, with_refined_eval=False)
    mesh = wl.field.mesh
    boxes, _, _ = O.partition_boxes(mesh.counts, mesh.bounds, wl.shape)
    _CPU.update(kind=kind, wl=wl, boxes=boxes)
    if kind == "reference":
        sys.path.insert(0, str(REF_DIR))
        import fieldfit.elastic_net as en

        assert en._HAVE_NUMBA, "the reference arm must run the numba CD core (elastic_net.py:15-20, 97)"
        W = np.abs(np.random.default_rng(0).standard_normal((8, 4)))
        en.fit(W / W.sum(1, keepdims=True), np.ones(8), en.ElasticNetConfig(max_iters=5))  # JIT compile


def _cpu_fit_one(args):
    """Fit subdomain s of C4 (3 adaptive rounds) + evaluate n_eval points in its box."""
    s, n_eval = args
    from oracle import pam_oracle as O

    wl, boxes, kind = _CPU["wl"], _CPU["boxes"], _CPU["kind"]
    mesh = wl.field.mesh
    lo, hi, op = boxes[s]
    rows = O.subdomain_rows(mesh.centroids, boxes[s])
    cen = mesh.centroids[rows]
    c = wl.config
    pts = np.asarray(lo) + np.random.default_rng(s).random((n_eval, 3)) * (np.asarray(hi) - np.asarray(lo))
    if kind == "reference":
        from fieldfit.adaptive import AdaptiveConfig as RA, fit_adaptive
        from fieldfit.elastic_net import ElasticNetConfig as REN
        from fieldfit.fields import SubdomainField
        from fieldfit.geometry import Box
        from fieldfit.rbf import RbfDictionary

        e = c.elastic
        rcfg = RA(k_top=c.k_top, m_max=c.m_max, eps_tol=c.eps_tol, eta=c.eta, m_q=c.m_q, max_rounds=c.max_rounds,
                  offsets=c.offsets, quad_order=c.quad_order,
                  elastic=REN(lam1=e.lam1, lam2=e.lam2, tol=e.tol, max_iters=e.max_iters))
        sub = SubdomainField(box=Box(lo=lo, hi=hi, open_hi=op), cell_indices=rows, centroids=cen,
                             values=wl.field.values[rows], cell_size=mesh.cell_size)
        t0 = time.perf_counter()
        sur, _ = fit_adaptive(sub, RbfDictionary(centers=cen, widths=np.full(rows.size, wl.spec.sigma)), rcfg)
        t_fit = time.perf_counter() - t0
        t0 = time.perf_counter()
        sur.evaluate(pts)
        t_eval = time.perf_counter() - t0
    else:
        cfg = dict(lam1=c.elastic.lam1, lam2=c.elastic.lam2, tol=c.elastic.tol, max_iters=c.elastic.max_iters,
                   k_top=c.k_top, m_max=c.m_max, eta=c.eta, m_q=c.m_q, max_rounds=c.max_rounds, offsets=c.offsets)
        t0 = time.perf_counter()
        od = O.fit_adaptive(cen, wl.field.values[rows], mesh.cell_size, lo, hi, cen,
                            np.full(rows.size, wl.spec.sigma), cfg)
        t_fit = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.surrogate_eval(pts, od["centers"], od["widths"], od["beta"])
        t_eval = time.perf_counter() - t0
    return t_fit, t_eval, n_eval


class CpuArm:
    """One process pool over all host cores, workers initialised once."""

    def __init__(self, threads: int, seed: int = 4):
        import multiprocessing as mp

        self.threads = threads
        self.kind = cpu_kind()
        self.pool = ProcessPoolExecutor(max_workers=threads, mp_context=mp.get_context("spawn"),
                                        initializer=_cpu_init, initargs=(self.kind, seed))
        # distinct subdomains across steps: a seeded permutation of all 2,244
        self.order = np.random.default_rng(2244).permutation(2244)
        self.next = 0
        list(self.pool.map(_cpu_fit_one, [(int(s), 8) for s in self.take(threads)]))  # start + init all workers

    def take(self, n):
        out = [self.order[(self.next + k) % 2244] for k in range(n)]
        self.next += n
        return out

    def step(self, n_sub: int, n_eval: int):
        subs = self.take(n_sub)
        t0 = time.perf_counter()
        res = list(self.pool.map(_cpu_fit_one, [(int(s), n_eval) for s in subs]))
        wall = time.perf_counter() - t0
        return {"wall_s": wall, "n_sub": n_sub, "fit_core_s": sum(r[0] for r in res),
                "eval_core_s": sum(r[1] for r in res), "n_eval": sum(r[2] for r in res)}

    def close(self):
        self.pool.shutdown()


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = host_threads()
    arm = CpuArm(threads)
    for _ in range(args.warmup):
        arm.step(threads, 200)
    steps = [arm.step(threads, 2000) for _ in range(args.steps)]
    arm.close()
    wall = sum(r["wall_s"] for r in steps)
    n_fit = sum(r["n_sub"] for r in steps)
    value = n_fit / wall
    fit_core = sum(r["fit_core_s"] for r in steps) / n_fit
    evals = sum(r["n_eval"] for r in steps) / sum(r["eval_core_s"] for r in steps) * threads
    distinct = min(2244, threads * (args.steps + args.warmup + 1))
    sample = (f"{threads} C4 subdomains per step (one per core, full 3-round adaptive fit, <= 4000 sweeps "
              f"per round) + 2000 evaluations each; {distinct} distinct subdomains over the run; "
              f"{'the unmodified reference (baseline/_ref, numba CD)' if arm.kind == 'reference' else 'the bit-exact oracle port'}"
              f" in {threads} processes, field built once per worker outside the timed steps")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "C4 SPE10-shaped 60x220x85, 6x22x17 subdomains, 2 refinement levels",
                   "sample": sample},
        "evals": {"value": evals, "unit": "points/s"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": arm.kind, "sample": sample,
                         "cpu_model": cpu_model(), "fit_core_s_per_subdomain": fit_core},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2605_16564_b200 as pam
    from paper_2605_16564_b200 import _native as nat
    from paper_2605_16564_b200 import engine as E
    from paper_2605_16564_b200 import workloads
    from paper_2605_16564_b200.partition import stage_field

    wl = workloads.config4(seed=4 + rank, with_refined_eval=True)
    part = wl.partition
    field = wl.field
    n_sub = part.n_subdomains
    P = wl.eval_points.shape[0]
    stage_field(field)
    d_eval = torch.from_numpy(wl.eval_points).cuda()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def step(record=None):
        sur, rep = pam.fit_parallel(field, part, wl.config, wl.spec)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sur.evaluate_device(d_eval)
        e1.record(stream)
        if record is not None:
            record.append((rep, e0, e1))
        return sur, rep

    warm = None
    for _ in range(args.warmup):
        warm = step()
    if warm is None:
        warm = step()
    # evaluation work: point-centre pairs = sum over points of the owner's M
    m_sizes = np.array([len(l.dictionary) for l in warm[0].locals], dtype=np.int64)
    _, edges = part.grid
    own = np.zeros(P, dtype=np.int64)
    stride = 1
    for k in range(3):
        idx = np.clip(np.searchsorted(edges[k], wl.eval_points[:, k], side="right") - 1, 0, part.shape[k] - 1)
        own += stride * idx
        stride *= part.shape[k]
    eval_pairs = int(m_sizes[own].sum())
    fp64_peak = nat.measure_fp64_peak()
    barrier()
    lib = nat.lib()
    lib.reset_counters()
    sampler = ClockSampler(local)
    sampler.start()
    recs = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    start.record(stream)
    for _ in range(args.steps):
        step(recs)
    end.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = lib.launches
    elapsed = start.elapsed_time(end) / 1e3
    eval_s = sum(e0.elapsed_time(e1) for _, e0, e1 in recs) / 1e3
    cd_s = sum(r.device["kernel_seconds"]["cd"] for r, _, _ in recs)
    cd_bytes = sum(r.device["cd_bytes"] for r, _, _ in recs)
    cd_flops = sum(r.device["cd_flops"] for r, _, _ in recs)
    cd_dense = sum(r.device.get("cd_dense_bytes", 0) for r, _, _ in recs)
    cd_launches = sum(r.device["cd_launches"] for r, _, _ in recs)
    kt = {}
    for r, _, _ in recs:
        for k, v in r.device["kernel_seconds"].items():
            kt[k] = kt.get(k, 0.0) + v
    if world > 1:
        t = torch.tensor([elapsed, eval_s], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed, eval_s = float(t[0]), float(t[1])

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        vals_host = torch.from_numpy(np.array(field.values)).pin_memory().numpy()
        pts_host = torch.from_numpy(wl.eval_points).pin_memory().numpy()
        mesh = field.mesh

        def e2e_step():
            fld = pam.FieldData(mesh=mesh, values=vals_host)  # fresh object: no device cache
            sur, rep = pam.fit_parallel(fld, part, wl.config, wl.spec)
            out = sur.evaluate(pts_host)
            m = sum(len(l.dictionary) for l in sur.locals)
            return out, m

        e2e_step()
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        n_entries = 0
        for _ in range(args.steps):
            _, n_entries = e2e_step()
        s1.record(stream)
        barrier()
        e_el = s0.elapsed_time(s1) / 1e3
        if world > 1:
            t = torch.tensor([e_el], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_el = float(t[0])
        h2d = field.values.nbytes + wl.eval_points.nbytes
        d2h = P * 8 + n_entries * (3 * 8 + 8 + 4 + 8)
        e2e = {"value": world * n_sub * args.steps / e_el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "evals_included": True,
               "ms_per_step": e_el / args.steps * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        arm = CpuArm(threads)
        r = arm.step(threads, 2000)
        arm.close()
        cpu = {"value": r["n_sub"] / r["wall_s"], "unit": UNIT, "cores": threads, "kind": arm.kind,
               "sample": f"{threads} distinct C4 subdomains (full 3-round adaptive fit, one per core) + 2000 "
                         f"evals each, {'the unmodified reference (baseline/_ref, numba)' if arm.kind == 'reference' else 'the oracle port'}, "
                         f"{r['wall_s']:.1f} s wall",
               "cpu_model": cpu_model(), "fit_core_s_per_subdomain": r["fit_core_s"] / r["n_sub"],
               "evals_per_s": r["n_eval"] / r["eval_core_s"] * threads}

    hbm, src = peaks()
    achieved = cd_bytes / cd_s / 1e9 if cd_s > 0 else 0.0
    line = {
        "metric": METRIC,
        "value": world * n_sub * args.steps / elapsed,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded SPE10-shaped stand-in; SPE10 file absent)",
        "config": {
            "workload": "C4 SPE10-shaped 60x220x85 cells (20x10x2 ft), 6x22x17=2244 subdomains x 500 cells, "
                        "per-cell dictionary, 2 refinement levels (k_top=100, m_q=3, eta=0.5, m_max=600, "
                        "3 rounds), lam1=4.59e-4 lam2=1e-4 tol=1e-6 max_iters=4000; eval at 1,122,000 cell "
                        "centres + 8,976,000 2x-refined centres",
            "subdomains_per_gpu": n_sub, "eval_points_per_gpu": P,
            "l2": "inputs larger than L2 (design matrices ~10 GB per round)",
            "parallelism": f"replica-per-gpu x{world}",
            "tile_tau": E.tile_tau(),
            "cd_kernel": cd_kernel_name(),
        },
        "evals": {"value": world * P * args.steps / eval_s, "unit": "points/s",
                  "ms_per_step": eval_s / args.steps * 1e3},
        "roofline": {"kernel": cd_kernel_name(), "bound": "hbm",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "peak_source": src, "traffic": None,
                     "algorithmic_bytes_per_launch": cd_bytes / max(cd_launches, 1),
                     "avg_launch_s": cd_s / max(cd_launches, 1),
                     "fp64_gflops": cd_flops / cd_s / 1e9 if cd_s > 0 else 0.0,
                     "dense_equivalent_bytes_per_launch": cd_dense / max(cd_launches, 1),
                     "tile_tau": E.tile_tau(),
                     "step_share": cd_s / elapsed if elapsed else None},
        # FP64-pipe bound: the issued FP64 instructions per point-centre pair
        # (15, pinned from SASS: 3 DADD + 3 DFMA distance, 2 DFMA + 1 DADD
        # exponent reduction, 3 DFMA polynomial, 1 DMUL scale, 2 accumulations)
        # against the measured DFMA issue rate (peak flop/s / 2).  The SURVEY 8d
        # flop convention (E = 20 per exp, 33 flops per pair) is kept beside it.
        "eval_roofline": {"kernel": "eval_kernel (locate + owner sort + one-pass Shepard sum, table-driven FP64 exp)",
                          "bound": "fp64", "unit": "FP64 instr/s",
                          "fp64_instr_per_pair": 15,
                          "pairs_per_step": eval_pairs,
                          "achieved": eval_pairs * 15 / (eval_s / args.steps),
                          "peak": fp64_peak / 2, "peak_source": "measured (pam_probe_fp64: DFMA/s)",
                          "frac": eval_pairs * 15 / (eval_s / args.steps) / (fp64_peak / 2),
                          "convention": "issued FP64-pipe fraction (SASS-pinned 15 FP64 instructions per pair)",
                          "survey_flop_frac": eval_pairs * 33 / (eval_s / args.steps) / fp64_peak,
                          "survey_flop_convention": "M_owner*(3d+4+E) per point, E=20 (overstates: the exp issues 11)"},
        "kernel_seconds_per_step": {k: v / args.steps for k, v in kt.items()},
        "cd_rounds": [{**d, "achieved_gbs": d["bytes"] / d["seconds"] / 1e9 if d["seconds"] else None,
                       "max_over_mean_fit": d["max_fit_bytes"] / d["mean_fit_bytes"] if d["mean_fit_bytes"] else None}
                      for d in recs[-1][0].device.get("cd_rounds", [])],
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if args.traffic:
        line["roofline"]["traffic"] = float(args.traffic)
    else:
        tr = committed_traffic(line["roofline"]["kernel"])
        if tr is not None:
            line["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
            line["roofline"]["traffic_source"] = tr["source"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def cd_kernel_name() -> str:
    """The CD kernel the C4 batch dispatches to under the current engine options (cd.cu)."""
    from paper_2605_16564_b200 import engine as E

    o = E.OPTIONS
    if o.tile_tau == 0:
        return "cd_kernel (dense column stream, TMA)"
    if o.cd_kernel in ("auto", "dual"):
        # C4: 2,244 fits of 500 rows >= 8 fits per SM (cd.cu cd_dispatch_tiles)
        return "cd_dual_kernel (lean tile stream, two fits per warp, TMA)"
    if o.cd_kernel == "pair":
        return "cd_pipe_kernel (column pairs, TMA)"
    return "cd_tile_kernel (lean single-column tile stream, TMA)"


def committed_traffic(kernel: str):
    """DRAM bytes per CD launch measured by ncu for this kernel (profiles/cd_traffic.json)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "cd_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    return d if d.get("kernel") == kernel else None


def run_c5(args):
    """BASELINE config 5 (throughput sweep): 64 x 32 x layers unit boxes, 1000
    samples each, a jittered M-centre lattice, planar interfaces; fit, then
    evaluate n_eval = 1e8 * layers / 32 uniform points over the slab.

    Strong scaling (the job is fixed): under N ranks, rank r fits the balanced
    box range r (parallel.balanced_ranges) on its GPU with inputs generated on
    the device for that range, the fitted dictionaries are allgathered over
    NCCL (parallel.gather_device_dictionaries), and every rank evaluates its
    share of the points with the full surrogate.  Time = max over ranks.
    """
    import torch

    from paper_2605_16564_b200 import _native as nat
    from paper_2605_16564_b200 import engine as E
    from paper_2605_16564_b200 import parallel, workloads
    from paper_2605_16564_b200.geometry import build_mesh
    from paper_2605_16564_b200.partition import DeviceSurrogate, GlobalSurrogate, make_partition

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    layers = args.c5_layers
    n_total = 64 * 32 * layers
    a, b = parallel.balanced_ranges(np.ones(n_total), world)[rank]
    n_sub = b - a
    n_eval = int(1e8 * layers / 32)
    pa, pb = parallel.balanced_ranges(np.ones(n_eval), world)[rank]
    if args.c5_gen == "device" or world > 1:  # pam_c5_generate_f64 for this rank's boxes
        p = workloads.config5_device(M=args.m, n_sub=n_sub, first_box=a)
    else:
        p = workloads.config5(M=args.m, n_sub=n_sub, n_eval=0)
    eval_all = np.random.default_rng(50).random((n_eval, 3)) * np.array([64.0, 32.0, float(layers)])
    dev = nat.device()
    d_pts = torch.from_numpy(np.ascontiguousarray(p.points).reshape(-1)).to(dev)
    d_vals = torch.from_numpy(p.values).to(dev)
    d_eval = torch.from_numpy(eval_all[pa:pb]).to(dev)
    del eval_all
    part = make_partition(build_mesh(3, (64, 32, layers), ((0.0, 64.0), (0.0, 32.0), (0.0, float(layers)))),
                          64, 32, layers)
    stream = torch.cuda.current_stream()
    # shards whose design matrices exceed the HBM budget (the full 65,536-box
    # sweep on one GPU: ~134 GB at M = 256) go through the chunked fit_packed path
    cap = E.dictionary_capacity(p.dict_m, min(p.config.k_top, 1000), p.config.m_q, p.config.m_max,
                                p.config.max_rounds)
    chunked = int(E.device_bytes(np.diff(p.row_off), cap).sum()) > E.w_budget_bytes()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def step(rec=None):
        if chunked:
            torch.cuda.empty_cache()  # hand the previous step's chunk buffers back before sizing chunks
            res = E.fit_packed(3, p.row_off, p.points, p.values, p.box_lo, p.box_hi, p.config, p.dict_m,
                               p.centres, p.widths, p.cell_size)
            m = np.asarray(res.m_final, dtype=np.int64)
            off = np.concatenate([[0], np.cumsum(m)[:-1]]).astype(np.int64)
            parts = (nat.to_dev(off), nat.to_dev(m.astype(np.int32)), nat.to_dev(np.concatenate(res.centres).reshape(-1)),
                     nat.to_dev(np.concatenate(res.widths)), nat.to_dev(np.concatenate(res.beta)))
            form = "gram (chunked)"
        else:
            eng = E.FitEngine(3, p.cell_size, p.row_off, d_pts, d_vals, p.box_lo, p.box_hi, [p.config] * n_sub,
                              init_centres=p.centres, init_widths=p.widths, init_m=p.dict_m)
            res = eng.run()
            parts = (eng.d_dict_off, eng.d_m_cur, eng.d_centres, eng.d_widths, eng.d_beta)
            eng.d_W = None
            form = eng.form
        g = parallel.gather_device_dictionaries(*parts, 3)  # NCCL allgatherv when world > 1
        ds = DeviceSurrogate(3, *g, torch.ones(n_total, dtype=torch.int32, device=dev))
        gs = GlobalSurrogate(partition=part, locals=tuple([None] * n_total))
        gs.attach_device(ds)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gs.evaluate_device(d_eval)
        e1.record(stream)
        if rec is not None:
            rec.append((res, e0, e1, form))

    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    recs = []
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    s0.record(stream)
    for _ in range(args.steps):
        step(recs)
    s1.record(stream)
    barrier()
    clocks = sampler.stop()
    el = s0.elapsed_time(s1) / 1e3
    ev = sum(x.elapsed_time(y) for _, x, y, _ in recs) / 1e3
    cd = sum(r.kernel_seconds["cd"] for r, _, _, _ in recs)
    streamed = sum(int(np.sum(rec.stream_doubles[rec.ran] * (rec.sweeps[rec.ran].astype(np.int64) + 1)))
                   for r, _, _, _ in recs for rec in r.rounds) * 8
    if world > 1:
        t = torch.tensor([el, ev, cd], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        el, ev, cd = (float(x) for x in t)
        tb = torch.tensor([float(streamed)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tb)
        streamed = float(tb[0])
    sweeps = [int(np.mean(rec.sweeps)) for rec in recs[0][0].rounds]
    hbm, src = peaks()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": n_total * args.steps / el, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded C5 generator)",
            "config": {"workload": f"C5 throughput sweep: {n_total} unit boxes x 1000 samples, M={args.m}, "
                                   f"{n_eval} eval points, boxes sharded over {world} rank(s)",
                       "cd_form": recs[0][3], "mean_sweeps": sweeps, "generator": "device" if
                       (args.c5_gen == "device" or world > 1) else "host",
                       "parallelism": f"shard x{world} + NCCL allgatherv of the dictionaries"},
            "evals": {"value": n_eval * args.steps / ev, "unit": "points/s"},
            "roofline": {"kernel": f"cd ({recs[0][3]} form)", "bound": "hbm",
                         "achieved": streamed / cd / 1e9 / world, "peak": hbm, "unit": "GB/s",
                         "frac": streamed / cd / 1e9 / world / hbm, "peak_source": src},
            "kernel_seconds_per_step": {k: sum(r.kernel_seconds[k] for r, _, _, _ in recs) / args.steps
                                        for k in recs[0][0].kernel_seconds},
            "clocks": clocks,
        }), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4", choices=["C4", "C5"])
    ap.add_argument("--m", type=int, default=256, help="C5: centres per subdomain")
    ap.add_argument("--c5-layers", type=int, default=4, help="C5: z-layers of the 64x32 box grid")
    ap.add_argument("--c5-gen", default="host", choices=["host", "device"],
                    help="C5 inputs: numpy generator (as the parity tests) or the on-device generator")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per CD launch from an ncu --set full capture (profiles/)")
    ap.add_argument("--tile-tau", type=float, default=None, help="CD tile-drop threshold (0 = dense stream)")
    ap.add_argument("--cd-kernel", default=None, choices=["auto", "lean", "dual", "pair", "block"])
    args = ap.parse_args()
    from paper_2605_16564_b200 import engine as E

    if args.tile_tau is not None:
        E.set_options(tile_tau=args.tile_tau)
    if args.cd_kernel is not None:
        E.set_options(cd_kernel=args.cd_kernel)
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            raise SystemExit(f"WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}")
    elif args.gpus > 1:
        return spawn_ranks(args)
    if args.config == "C5":
        return run_c5(args)
    return run_ours(args)


def _rank_main(local_rank, world, port, argv):
    os.environ.update(RANK=str(local_rank), LOCAL_RANK=str(local_rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.argv = [sys.argv[0]] + argv
    rc = main()
    if rc:
        raise SystemExit(rc)


def spawn_ranks(args):
    """`python bench.py --gpus N` without torchrun: one process per GPU (torch.multiprocessing),
    rendezvous on 127.0.0.1; rank 0 prints the JSON line."""
    import socket

    import torch.multiprocessing as tmp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    tmp.spawn(_rank_main, args=(args.gpus, port, sys.argv[1:]), nprocs=args.gpus, join=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
