"""Reference-side binding of the B200 seams (the file a ``fieldfit`` maintainer
adds as ``fieldfit/_b200.py``).

Binds ``libpam_b200.so`` with ctypes -- the reference's own FFI for this path
(it is pure Python + numba) -- and exposes drop-in replacements with the exact
signatures and in-place semantics of the reference functions:

    cd_sweeps_b200    <->  fieldfit.elastic_net._cd_sweeps_jit  (elastic_net.py:113-161)
    shepard_eval_b200 <->  fieldfit.rbf.shepard_eval             (rbf.py:152-167)

``install(fieldfit)`` swaps them in at the reference's seams:
``elastic_net.py:97`` dispatches to ``_cd_sweeps_jit`` whenever numba is
present, and ``LocalSurrogate.evaluate`` (rbf.py:190-192) calls the module
global ``shepard_eval``.  Nothing else in the reference changes.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB = Path(os.environ.get("PAM_B200_LIB", Path(__file__).resolve().parents[1] / "paper_2605_16564_b200" /
                          "libpam_b200.so"))

_P, _I64, _D, _I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int32
_lib = ctypes.CDLL(str(LIB))
_lib.pam_cd_sweeps_host_f64.restype = ctypes.c_int
_lib.pam_cd_sweeps_host_f64.argtypes = [_P, _I64, _I64, _P, _P, _D, _D, _D, _I64, _P, _P, _P, _P, _P]
_lib.pam_shepard_eval_host_f64.restype = ctypes.c_int
_lib.pam_shepard_eval_host_f64.argtypes = [ctypes.c_int, _I64, _P, _I64, _P, _P, _P, _P, _P]
_lib.pam_last_error.restype = ctypes.c_char_p

PAM_ERR_DEGENERATE = 4
CALLS = {"cd_sweeps": 0, "shepard_eval": 0}


def _f64(a, order="C"):
    return np.require(np.asarray(a, dtype=np.float64), requirements=[order[0], "A"])


def cd_sweeps_b200(W, col_sq, denom, lam1, lam2, tol, max_iters, beta, r, history):
    """_cd_sweeps_jit on the GPU: updates beta, r, history in place; returns (sweeps, converged)."""
    assert W.flags.f_contiguous and W.dtype == np.float64  # fit() passes np.asfortranarray(W)
    for a in (beta, r, history):
        assert a.flags.c_contiguous and a.dtype == np.float64 and a.flags.writeable
    n, m = W.shape
    cs, dn = _f64(col_sq), _f64(denom)
    sweeps, conv = _I64(0), _I32(0)
    rc = _lib.pam_cd_sweeps_host_f64(W.ctypes.data, n, m, cs.ctypes.data, dn.ctypes.data, float(lam1),
                                     float(lam2), float(tol), int(max_iters), beta.ctypes.data, r.ctypes.data,
                                     history.ctypes.data, ctypes.byref(sweeps), ctypes.byref(conv))
    if rc != 0:
        raise RuntimeError(f"pam_cd_sweeps_host_f64: {_lib.pam_last_error().decode()} (status {rc})")
    CALLS["cd_sweeps"] += 1
    return int(sweeps.value), bool(conv.value)


def shepard_eval_b200(points, dictionary, beta):
    """shepard_eval(points, dictionary, beta) on the GPU, same checks and exceptions."""
    beta = np.asarray(beta, dtype=float)
    if beta.ndim != 1 or beta.shape[0] != len(dictionary):
        raise ValueError(
            f"coefficient length {beta.shape} does not match dictionary size {len(dictionary)}"
        )
    pts = np.asarray(points, dtype=float)
    if pts.ndim == 1:
        pts = pts[:, None] if dictionary.dim == 1 else pts[None, :]
    if pts.shape[1] != dictionary.dim:
        raise ValueError(f"points have dim {pts.shape[1]}, dictionary has dim {dictionary.dim}")
    pts = _f64(pts)
    c, w, b = _f64(dictionary.centers), _f64(dictionary.widths), _f64(beta)
    out = np.empty(pts.shape[0])
    if pts.shape[0] == 0:
        return out
    bad = _I64(-1)
    rc = _lib.pam_shepard_eval_host_f64(dictionary.dim, pts.shape[0], pts.ctypes.data, len(dictionary),
                                        c.ctypes.data, w.ctypes.data, b.ctypes.data, out.ctypes.data,
                                        ctypes.byref(bad))
    if rc == PAM_ERR_DEGENERATE:
        raise FloatingPointError("Shepard denominator degenerate")
    if rc != 0:
        raise RuntimeError(f"pam_shepard_eval_host_f64: {_lib.pam_last_error().decode()} (status {rc})")
    CALLS["shepard_eval"] += 1
    return out


def _install_in_worker(pkg_name):
    import importlib

    install(importlib.import_module(pkg_name))


def install(fieldfit_pkg) -> None:
    """Swap the seams of an imported reference package (``import fieldfit``).

    ``fit_parallel(workers > 1)`` fans out over a ProcessPoolExecutor
    (partition.py:188-195) whose default start method on Linux is fork; a CUDA
    context does not survive fork, so the pool is switched to spawn with an
    initializer that installs the same seams in every worker process.
    """
    import functools
    import importlib
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    en = importlib.import_module(fieldfit_pkg.__name__ + ".elastic_net")
    rbf = importlib.import_module(fieldfit_pkg.__name__ + ".rbf")
    part = importlib.import_module(fieldfit_pkg.__name__ + ".partition")
    en._cd_sweeps_jit = cd_sweeps_b200
    rbf.shepard_eval = shepard_eval_b200
    fieldfit_pkg.shepard_eval = shepard_eval_b200
    part.ProcessPoolExecutor = functools.partial(
        ProcessPoolExecutor, mp_context=mp.get_context("spawn"), initializer=_install_in_worker,
        initargs=(fieldfit_pkg.__name__,))
