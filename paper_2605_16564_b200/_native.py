"""ctypes binding of the sm_100a C-ABI library (``include/pam_b200.h``).

This is the only door from Python into the compute path.  There is no CPU
fallback: if the shared library is missing, fails to load, or no CUDA device
is present, every compute entry point raises :class:`NativeUnavailable`.

Device memory, streams and host<->device copies are handled with PyTorch
(plumbing only); tensors are passed to the library as raw pointers.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import NumericalError

LIB_PATH = Path(__file__).resolve().parent / "libpam_b200.so"

ABI_VERSION = 3  # PAM_ABI_VERSION of include/pam_b200.h

# status codes (pam_b200.h)
PAM_OK = 0
PAM_ERR_CUDA = 1
PAM_ERR_ARG = 2
PAM_ERR_OUTSIDE = 3
PAM_ERR_DEGENERATE = 4
PAM_ERR_NONPOSITIVE = 5
PAM_ERR_UNSUPPORTED = 6
PAM_ERR_NONFINITE = 7
PAM_ERR_CLAIMED = 8

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_ptr = ctypes.c_void_p

# name -> (restype, argtypes); every symbol declared in include/pam_b200.h
SIGNATURES = {
    "pam_abi_version": (ctypes.c_int, []),
    "pam_last_error": (ctypes.c_char_p, []),
    "pam_cd_max_rows": (_i64, []),
    "pam_err_reset": (ctypes.c_int, [_ptr, _ptr]),
    "pam_log_values_f64": (ctypes.c_int, [_ptr, _i64, _ptr, _ptr, _ptr]),
    "pam_assemble_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32, ctypes.c_int,
         _ptr, _ptr],
    ),
    "pam_cd_workspace_bytes": (_i64, [_i64, _i64, _i64, _i32, _i32]),
    "pam_cd_f64": (
        ctypes.c_int,
        [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32,
         _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_cd_ex_f64": (
        ctypes.c_int,
        [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32,
         _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, ctypes.c_int, _ptr, _ptr],
    ),
    "pam_assemble_tiles_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32, _dbl, _ptr,
         _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr],
    ),
    "pam_cd_tiles_f64": (
        ctypes.c_int,
        [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
         _ptr, _i32, _i32, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32, _ptr, _ptr],
    ),
    "pam_gram_f64": (
        ctypes.c_int,
        [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_cd_gram_f64": (
        ctypes.c_int,
        [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32,
         _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_residual_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
         _i32, _ptr, _i32, _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_mark_f64": (ctypes.c_int, [_i64, _ptr, _ptr, _ptr, _ptr, _i32, _ptr, _ptr, _ptr]),
    "pam_enrich_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _i32, _ptr, _ptr, _i32, _ptr, _ptr, _ptr, _ptr,
         _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i32, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_eval_workspace_bytes": (_i64, [_i64, _i64]),
    "pam_locate_f64": (ctypes.c_int, [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr]),
    "pam_locate_boxes_f64": (ctypes.c_int, [ctypes.c_int, _i64, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr]),
    "pam_eval_boxes_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
         _ptr, _ptr],
    ),
    "pam_eval_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
         _ptr, _ptr, _ptr],
    ),
    "pam_shepard_eval_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _i64, _ptr, _ptr, _ptr, _i32, _ptr, _ptr, _ptr],
    ),
    "pam_row_normalize_f64": (ctypes.c_int, [_i64, _i64, _ptr, ctypes.c_int, _ptr, _ptr, _ptr]),
    "pam_gather_cells_f64": (
        ctypes.c_int,
        [ctypes.c_int, _ptr, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_probe_fp64": (ctypes.c_int, [_i64, _ptr, _ptr]),
    "pam_dict_scatter_f64": (ctypes.c_int, [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                                            _ptr, _ptr]),
    "pam_c5_generate_f64": (ctypes.c_int, [_i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, ctypes.c_uint64, _ptr,
                                           _ptr, _ptr, _ptr]),
    "pam_p1_values_f64": (ctypes.c_int, [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr]),
    "pam_csr_spmv_f64": (ctypes.c_int, [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr]),
    "pam_pcg_workspace_bytes": (_i64, [_i64]),
    "pam_pcg_f64": (ctypes.c_int, [_i64, _ptr, _ptr, _ptr, _ptr, _ptr, _dbl, _i64, _ptr, _ptr, _ptr, _ptr,
                                   _ptr]),
    "pam_format_entries_host": (_i64, [ctypes.c_int, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _i64]),
    "pam_cd_sweeps_host_f64": (
        ctypes.c_int,
        [_ptr, _i64, _i64, _ptr, _ptr, _dbl, _dbl, _dbl, _i64, _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
    "pam_shepard_eval_host_f64": (
        ctypes.c_int,
        [ctypes.c_int, _i64, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr],
    ),
}


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing: there is no CPU fallback."""


_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None):
    """Load libpam_b200.so and bind every declared symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - broken build
            raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError = missing export
            fn.restype = res
            fn.argtypes = args
        if lib.pam_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libpam_b200.so ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


class _CountingLib:
    """Proxy over the ctypes library that counts kernel launches per entry point.

    bench.py reports ``gpu_launches`` from these counters; KERNELS_PER_CALL is
    the number of kernels each entry point enqueues (csrc/*.cu).
    """

    KERNELS_PER_CALL = {
        "pam_err_reset": 1, "pam_log_values_f64": 1, "pam_assemble_f64": 1, "pam_cd_f64": 1,
        "pam_cd_ex_f64": 1, "pam_residual_f64": 2, "pam_mark_f64": 1, "pam_enrich_f64": 1,
        "pam_locate_f64": 1, "pam_locate_boxes_f64": 2, "pam_eval_f64": 5, "pam_eval_boxes_f64": 6, "pam_shepard_eval_f64": 1,
        "pam_row_normalize_f64": 1, "pam_gather_cells_f64": 1, "pam_dict_scatter_f64": 1, "pam_assemble_tiles_f64": 3,
        "pam_cd_tiles_f64": 1, "pam_gram_f64": 2, "pam_cd_gram_f64": 1, "pam_probe_fp64": 1,
        "pam_p1_values_f64": 1, "pam_csr_spmv_f64": 1, "pam_pcg_f64": 3, "pam_c5_generate_f64": 2,  # + 5 per PCG iteration
    }

    def __init__(self, raw):
        self._raw = raw
        self.launches = 0
        self.calls = {}

    def __getattr__(self, name):
        fn = getattr(self._raw, name)
        k = self.KERNELS_PER_CALL.get(name)
        if k is None:
            return fn

        def call(*args):
            self.launches += k
            self.calls[name] = self.calls.get(name, 0) + 1
            return fn(*args)

        return call

    def reset_counters(self):
        self.launches = 0
        self.calls = {}


_counting = None


def lib():
    global _counting
    raw = load_library()
    if _counting is None or _counting._raw is not raw:
        _counting = _CountingLib(raw)
    return _counting


# ---------------------------------------------------------------------------
# torch plumbing

_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch  # deferred: importing the package must not need a GPU

        _torch = torch
    return _torch


def device():
    """The CUDA device every kernel runs on; raises when there is none."""
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise NativeUnavailable("a CUDA device is required: the PAM hot path has no CPU fallback")
    lib()  # fail loudly if the extension is absent
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    torch = torch_mod()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def to_dev(a, dtype=None):
    """numpy/sequence -> contiguous device tensor (float64/int64/int32)."""
    torch = torch_mod()
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if not arr.flags.writeable:
        arr = arr.copy()
    t = torch.from_numpy(arr)
    return t.to(device(), non_blocking=False)


def check(rc: int, what: str, index: int | None = None):
    """Raise the reference-equivalent Python exception for a status code."""
    if rc == PAM_OK:
        return
    msg = lib().pam_last_error().decode(errors="replace")
    if rc == PAM_ERR_CUDA:
        raise RuntimeError(f"{what}: CUDA error: {msg}")
    if rc == PAM_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg or 'shape outside the kernel envelope'}")
    if rc == PAM_ERR_ARG:
        raise ValueError(f"{what}: invalid argument {msg}")
    raise RuntimeError(f"{what}: status {rc} (index {index})")


class ErrorWord:
    """Device int64[2] {code, first index} written by the kernels."""

    def __init__(self):
        torch = torch_mod()
        self.t = torch.empty(2, dtype=torch.int64, device=device())
        self.reset()

    def reset(self):
        check(lib().pam_err_reset(ptr(self.t), stream_ptr()), "pam_err_reset")

    def read(self):
        code, idx = (int(v) for v in self.t.cpu().tolist())
        return code, idx


def raise_data_error(code: int, index: int, context: str = ""):
    """Map a device error word onto the reference's exceptions."""
    if code == 0:
        return
    if code == PAM_ERR_NONPOSITIVE:
        raise ValueError(f"field value at cell {index} is not positive{context}")
    if code == PAM_ERR_DEGENERATE:
        raise FloatingPointError("Shepard denominator degenerate")
    if code == PAM_ERR_OUTSIDE:
        raise ValueError(f"point index {index}{context} lies outside all boxes")
    if code == PAM_ERR_UNSUPPORTED:
        raise NumericalError(f"dictionary capacity exceeded in subdomain {index}")
    raise RuntimeError(f"device error {code} at index {index}")


def measure_fp64_peak(iters: int = 200_000) -> float:
    """Measured FP64 peak (flop/s, FMA = 2) of this GPU via pam_probe_fp64."""
    torch = torch_mod()
    dev = device()
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    check(lib().pam_probe_fp64(1000, ptr(out), stream_ptr()), "pam_probe_fp64")  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    check(lib().pam_probe_fp64(iters, ptr(out), stream_ptr()), "pam_probe_fp64")
    e1.record()
    e1.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    return sms * 4 * 256 * 8 * iters * 2.0 / sec


def available() -> bool:
    """True when the library loads and a CUDA device is present."""
    try:
        device()
        return True
    except NativeUnavailable:
        return False
