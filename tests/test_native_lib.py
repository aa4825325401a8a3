"""CPU checks of the C-ABI boundary: the library loads, exports exactly what
include/pam_b200.h declares, and the product refuses to run without a GPU
(no CPU fallback)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2605_16564_b200 import _native

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pam_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pam_\w+)\s*\(", text)))


def test_library_exists_and_loads():
    lib = _native.load_library()
    assert lib.pam_abi_version() == _native.ABI_VERSION == 3
    assert lib.pam_cd_max_rows() >= 2**31 - 1  # no row envelope (elastic_net.py has none)
    assert lib.pam_cd_workspace_bytes(10, 5000, 700, 500, 1) == 256
    assert lib.pam_cd_workspace_bytes(1, 20000, 100, 20000, 0) == 256 + 8 * 20000
    assert lib.pam_cd_workspace_bytes(4, 4000, 1000, 1000, 4) == 256 + 576 * 1000 + 96 * 4  # blocked CD


def test_every_declared_symbol_is_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pam_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # the ctypes table binds every declared symbol, and nothing undeclared
    assert sorted(_native.SIGNATURES) == syms


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "-lelf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # TMA bulk copies in the CD kernel


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_2605_16564_b200 as pam

    d = pam.RbfDictionary(centers=np.zeros((2, 1)), widths=np.ones(2))
    with pytest.raises(_native.NativeUnavailable):
        pam.shepard_features(np.zeros((3, 1)), d)
    with pytest.raises(_native.NativeUnavailable):
        pam.fit(np.eye(2), np.ones(2), pam.ElasticNetConfig())


def test_no_environment_switches_in_native_code():
    """Kernel selection is explicit (C-ABI arguments / engine options), never getenv."""
    for p in (ROOT / "paper_2605_16564_b200" / "csrc").glob("*.cu*"):
        assert "getenv" not in p.read_text(), p


def test_reference_side_binding_loads():
    """integration/fieldfit_b200.py (the ctypes file a fieldfit maintainer adds) binds the seams."""
    from integration import fieldfit_b200 as b

    assert b._lib.pam_cd_sweeps_host_f64 is not None and b._lib.pam_shepard_eval_host_f64 is not None
    assert callable(b.install)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2605_16564_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "from oracle" not in src and "import oracle" not in src, p
