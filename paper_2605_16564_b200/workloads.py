"""Seeded synthetic workloads for BASELINE.json's five configurations.

No public dataset is available offline (the SPE10 file is absent),
so every configuration is a seeded synthetic field with the shapes, sizes
and value distributions BASELINE.json states.  All generation is numpy
``default_rng(seed)`` on the host; the same arrays feed the GPU path, the
CPU oracle and the reference arm.

Pinned solver/refinement choices: the reference's 2D
preset ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=4000)
(tests/test_acceptance.py:32), no overlap (the decomposition is half-open),
"L levels" = max_rounds L+1 and m_max = L*k_top*m_q with k_top ~ 20% of the
cells per subdomain, m_q = 3, eta = 0.5, in-cell offsets
((0,0),(-1/4,0),(1/4,0)) (tests/test_acceptance.py:33) and their 3D analogue.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .adaptive import AdaptiveConfig
from .elastic_net import ElasticNetConfig
from .fields import FieldData
from .geometry import build_mesh
from .partition import DictionarySpec, make_partition

PRESET_ELASTIC = ElasticNetConfig(lam1=4.59e-4, lam2=1e-4, tol=1e-6, max_iters=4000)
IN_CELL_2D = ((0.0, 0.0), (-0.25, 0.0), (0.25, 0.0))
IN_CELL_3D = ((0.0, 0.0, 0.0), (-0.25, 0.0, 0.0), (0.25, 0.0, 0.0))


@dataclass
class Workload:
    name: str
    field: FieldData
    shape: tuple  # partition grid
    config: AdaptiveConfig
    spec: DictionarySpec
    eval_points: np.ndarray
    notes: dict = field(default_factory=dict)

    @property
    def partition(self):
        return make_partition(self.field.mesh, *self.shape)


def _refined(levels, k_top, m_q=3, elastic=PRESET_ELASTIC, offsets=IN_CELL_2D):
    return AdaptiveConfig(k_top=k_top, m_max=levels * k_top * m_q, eta=0.5, m_q=m_q,
                          max_rounds=levels + 1, elastic=elastic, offsets=offsets)


def _grf_2d(n, corr, rng):
    """Periodic Gaussian random field with C(r) = exp(-r^2/(2 corr^2)) on [0,1]^2 (FFT)."""
    k = np.fft.fftfreq(n, d=1.0 / n) * 2 * np.pi
    kx, ky = np.meshgrid(k, k, indexing="xy")
    spec = np.exp(-0.5 * (kx**2 + ky**2) * corr**2)
    noise = rng.standard_normal((n, n))
    f = np.fft.ifft2(np.fft.fft2(noise) * np.sqrt(spec)).real
    return (f - f.mean()) / f.std()


def config1() -> Workload:
    """2D step 64x64, 2x2 subdomains, 16x16 lattice per subdomain, no refinement."""
    mesh = build_mesh(2, (64, 64), ((0.0, 1.0), (0.0, 1.0)))
    x = mesh.centroids[:, 0]
    fld = FieldData(mesh=mesh, values=np.where(x < 0.5, 1.0, 100.0))
    ev = build_mesh(2, (128, 128), ((0.0, 1.0), (0.0, 1.0))).centroids
    return Workload("C1-step2d", fld, (2, 2), AdaptiveConfig(m_max=0, elastic=PRESET_ELASTIC),
                    DictionarySpec(sigma=0.5 / 16, lattice=16), ev,
                    {"true_field": lambda p: np.where(p[:, 0] < 0.5, 1.0, 100.0)})


def config2(seed: int = 2, n_eval: int = 100_000) -> Workload:
    """2D inclusions 256^2: 20 seeded disks, 8x8 subdomains, 2 refinement levels."""
    rng = np.random.default_rng(seed)
    mesh = build_mesh(2, (256, 256), ((0.0, 1.0), (0.0, 1.0)))
    c = mesh.centroids
    vals = np.ones(mesh.n_cells)
    centres = rng.random((20, 2))
    radii = rng.uniform(0.03, 0.10, 20)
    logk = rng.uniform(-2.0, 3.0, 20)
    for (cx, cy), r, u in zip(centres, radii, logk):  # later disks overwrite
        vals[(c[:, 0] - cx) ** 2 + (c[:, 1] - cy) ** 2 < r * r] = 10.0**u
    ev = rng.random((n_eval, 2))
    cells = 1024
    return Workload("C2-inclusions", FieldData(mesh=mesh, values=vals), (8, 8),
                    _refined(2, cells * 20 // 100), DictionarySpec(sigma=1.0 / 256), ev)


def config3(seed: int = 3, eval_n: int = 1024) -> Workload:
    """2D facies 512^2: thresholded GRF, 16x16 subdomains, 3 refinement levels."""
    rng = np.random.default_rng(seed)
    mesh = build_mesh(2, (512, 512), ((0.0, 1.0), (0.0, 1.0)))
    g = _grf_2d(512, 0.05, rng).ravel()  # row-major (y, x) == cell order
    cuts = np.percentile(g, [20, 40, 60, 80])
    facies = np.searchsorted(cuts, g)
    logk = np.array([-3.0, -1.5, 0.0, 1.5, 3.0])[facies]
    ev = build_mesh(2, (eval_n, eval_n), ((0.0, 1.0), (0.0, 1.0))).centroids
    return Workload("C3-facies", FieldData(mesh=mesh, values=10.0**logk), (16, 16),
                    _refined(3, 1024 * 20 // 100), DictionarySpec(sigma=1.0 / 512), ev)


SPE10_COUNTS = (60, 220, 85)
SPE10_CELL = (20.0, 10.0, 2.0)  # ft
SPE10_SHAPE = (6, 22, 17)  # subdomains of 10 x 10 x 5 cells


def spe10_like_field(seed: int = 4, counts=SPE10_COUNTS, cell=SPE10_CELL) -> FieldData:
    """SPE10-shaped synthetic permeability (mD) on 60x220x85 cells of 20x10x2 ft.

    Layers z < 35: log10 k ~ N(0,1) with anisotropic Gaussian correlation
    (200, 100, 4) ft (FFT synthesis).  Layers z >= 35: sinuous channels
    100-300 ft wide along y with k = 10^U[2,4] per channel in a per-layer
    background k = 10^U[-3,1].  Cell order x fastest, then y, then z.
    """
    rng = np.random.default_rng(seed)
    nx, ny, nz = counts
    dx, dy, dz = cell
    mesh = build_mesh(3, counts, tuple((0.0, n * d) for n, d in zip(counts, cell)))
    logk = np.empty((nz, ny, nx))
    nz_top = 35
    # anisotropic GRF on the top layers (periodic FFT on the full 3D block)
    kx = np.fft.fftfreq(nx, d=dx) * 2 * np.pi
    ky = np.fft.fftfreq(ny, d=dy) * 2 * np.pi
    kz = np.fft.fftfreq(nz_top, d=dz) * 2 * np.pi
    KZ, KY, KX = np.meshgrid(kz, ky, kx, indexing="ij")
    spec = np.exp(-0.5 * ((KX * 200.0) ** 2 + (KY * 100.0) ** 2 + (KZ * 4.0) ** 2))
    noise = rng.standard_normal((nz_top, ny, nx))
    f = np.fft.ifftn(np.fft.fftn(noise) * np.sqrt(spec)).real
    logk[:nz_top] = (f - f.mean()) / f.std()
    # fluvial layers
    X = (np.arange(nx) + 0.5) * dx
    Y = (np.arange(ny) + 0.5) * dy
    XX, YY = np.meshgrid(X, Y, indexing="xy")  # (ny, nx)
    for z in range(nz_top, nz):
        layer = np.full((ny, nx), rng.uniform(-3.0, 1.0))
        for _ in range(int(rng.integers(2, 6))):
            x0 = rng.uniform(0, nx * dx)
            amp = rng.uniform(100.0, 400.0)
            lam = rng.uniform(800.0, 2000.0)
            phase = rng.uniform(0, 2 * np.pi)
            width = rng.uniform(100.0, 300.0)
            centre = x0 + amp * np.sin(2 * np.pi * YY / lam + phase)
            layer[np.abs(XX - centre) < 0.5 * width] = rng.uniform(2.0, 4.0)
        logk[z] = layer
    return FieldData(mesh=mesh, values=10.0 ** logk.ravel())


def config4(seed: int = 4, with_refined_eval: bool = True) -> Workload:
    """SPE10-shaped 3D: 1,122,000 cells, 6x22x17 subdomains of 500 cells, 2 levels."""
    fld = spe10_like_field(seed)
    mesh = fld.mesh
    sigma = float(np.prod(SPE10_CELL) ** (1.0 / 3.0))
    pts = [mesh.centroids]
    if with_refined_eval:
        pts.append(build_mesh(3, tuple(2 * n for n in SPE10_COUNTS), mesh.bounds).centroids)
    ev = np.concatenate(pts)
    return Workload("C4-spe10-shaped", fld, SPE10_SHAPE,
                    _refined(2, 500 * 20 // 100, offsets=IN_CELL_3D), DictionarySpec(sigma=sigma), ev,
                    {"n_centroids": mesh.n_cells})


# ---------------------------------------------------------------------------
# C5: throughput sweep on independent subdomains (sample points are not cell
# centroids, so it is expressed at the subdomain level, like the reference
# oracle procedure: SubdomainField + RbfDictionary + fit_adaptive per box).

C5_LATTICE = {64: (4, 4, 4), 128: (8, 4, 4), 256: (8, 8, 4), 512: (8, 8, 8)}
C5_GRID = (64, 32, 32)


@dataclass
class PackedSubdomains:
    """Packed ragged batch for the subdomain-level batched API."""

    dim: int
    row_off: np.ndarray  # (S+1,)
    points: np.ndarray  # (sum N, dim)
    values: np.ndarray  # (sum N,)
    box_lo: np.ndarray  # (S, dim)
    box_hi: np.ndarray
    dict_m: np.ndarray  # (S,)
    centres: np.ndarray  # (sum M, dim)
    widths: np.ndarray  # (sum M,)
    cell_size: tuple
    config: AdaptiveConfig
    eval_points: np.ndarray | None = None
    grid: tuple = C5_GRID
    device: dict | None = None  # device-resident copies (config5_device): points, values, centres


def config5(M: int = 256, n_sub: int = 65536, n_pts: int = 1000, n_eval: int = 100_000_000,
            seed: int = 5) -> PackedSubdomains:
    """65,536 unit boxes tiling [0,64]x[0,32]x[0,32]; 1000 uniform samples per box,
    a jittered M-centre lattice, 1-4 random planar interfaces with levels 10^U[-3,3]."""
    rng = np.random.default_rng(seed)
    gx, gy, gz = C5_GRID
    total = gx * gy * gz
    if n_sub > total:
        raise ValueError("n_sub exceeds the 64x32x32 tiling")
    idx = np.arange(n_sub)
    lo = np.stack([idx % gx, (idx // gx) % gy, idx // (gx * gy)], axis=1).astype(float)
    hi = lo + 1.0
    u = rng.random((n_sub, n_pts, 3))
    pts = lo[:, None, :] + u  # in [lo, lo+1): half-open
    # interfaces
    vals = np.empty((n_sub, n_pts))
    n_planes = rng.integers(1, 5, n_sub)
    for s in range(n_sub):
        k = int(n_planes[s])
        nrm = rng.standard_normal((k, 3))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        through = lo[s] + rng.random((k, 3))
        side = np.einsum("pkd,kd->pk", pts[s][:, None, :] - through[None, :, :], nrm) > 0
        region = (side.astype(np.int64) << np.arange(k)[None, :]).sum(1)
        levels = 10.0 ** rng.uniform(-3.0, 3.0, 1 << k)
        vals[s] = levels[region]
    g = C5_LATTICE[M]
    h = np.array([1.0 / g[0], 1.0 / g[1], 1.0 / g[2]])
    axes = [(np.arange(g[k]) + 0.5) * h[k] for k in range(3)]
    base = np.stack(np.meshgrid(*axes[::-1], indexing="ij")[::-1], axis=-1).reshape(-1, 3)
    jit = rng.uniform(-0.25, 0.25, (n_sub, M, 3)) * h[None, None, :]
    cen = np.clip(lo[:, None, :] + base[None] + jit, lo[:, None, :], hi[:, None, :])
    sigma = float(h.mean())
    ev = None
    if n_eval:
        ev = rng.random((n_eval, 3)) * np.array([gx, gy, gz], dtype=float)
    cfg = AdaptiveConfig(m_max=0, elastic=PRESET_ELASTIC, max_rounds=1)
    return PackedSubdomains(
        dim=3, row_off=np.arange(n_sub + 1, dtype=np.int64) * n_pts,
        points=pts.reshape(-1, 3), values=vals.reshape(-1), box_lo=lo, box_hi=hi,
        dict_m=np.full(n_sub, M, dtype=np.int64), centres=cen.reshape(-1, 3),
        widths=np.full(n_sub * M, sigma), cell_size=(0.1, 0.1, 0.1), config=cfg, eval_points=ev)


def config5_device(M: int = 256, n_sub: int = 65536, n_pts: int = 1000, seed: int = 5,
                   host_copy: bool = True, first_box: int = 0) -> PackedSubdomains:
    """BASELINE config 5 inputs generated on the GPU (``pam_c5_generate_f64``).

    Same distributions as :func:`config5` (unit boxes of the 64x32x32 tiling,
    uniform samples, 1-4 planar interfaces with levels 10^U[-3,3], jittered
    lattice) from a counter-based random stream, so the data differ from the
    numpy generator's but are deterministic for a seed; the full 65,536-box
    sweep is generated in well under a second instead of minutes on the host.
    Host copies are made unless ``host_copy=False`` (then only ``device``).
    ``first_box``: generate boxes first_box .. first_box + n_sub - 1 of the
    tiling (a rank's shard; a box's data do not depend on the range).
    """
    from . import _native as nat

    torch = nat.torch_mod()
    gx, gy, gz = C5_GRID
    if first_box + n_sub > gx * gy * gz:
        raise ValueError("boxes beyond the 64x32x32 tiling")
    g = C5_LATTICE[M]
    dev = nat.device()
    d_pts = torch.empty(n_sub * n_pts * 3, dtype=torch.float64, device=dev)
    d_vals = torch.empty(n_sub * n_pts, dtype=torch.float64, device=dev)
    d_cen = torch.empty(n_sub * M * 3, dtype=torch.float64, device=dev)
    nat.check(nat.lib().pam_c5_generate_f64(first_box, n_sub, n_pts, g[0], g[1], g[2], gx, gy, seed, nat.ptr(d_pts),
                                            nat.ptr(d_vals), nat.ptr(d_cen), nat.stream_ptr()),
              "pam_c5_generate_f64")
    idx = first_box + np.arange(n_sub)
    lo = np.stack([idx % gx, (idx // gx) % gy, idx // (gx * gy)], axis=1).astype(float)
    h = np.array([1.0 / g[0], 1.0 / g[1], 1.0 / g[2]])
    cfg = AdaptiveConfig(m_max=0, elastic=PRESET_ELASTIC, max_rounds=1)
    host = (lambda t: t.cpu().numpy()) if host_copy else (lambda t: None)
    pts, vals, cen = host(d_pts), host(d_vals), host(d_cen)
    return PackedSubdomains(
        dim=3, row_off=np.arange(n_sub + 1, dtype=np.int64) * n_pts,
        points=None if pts is None else pts.reshape(-1, 3), values=vals, box_lo=lo, box_hi=lo + 1.0,
        dict_m=np.full(n_sub, M, dtype=np.int64), centres=None if cen is None else cen.reshape(-1, 3),
        widths=np.full(n_sub * M, float(h.mean())), cell_size=(0.1, 0.1, 0.1), config=cfg,
        device={"points": d_pts, "values": d_vals, "centres": d_cen})


WORKLOADS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4}
