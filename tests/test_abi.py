"""CPU checks of the drop-in boundary: libfsg.so loads, exports exactly the
C ABI declared in include/fsg.h, and fails loudly without a GPU (no CPU
fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2206_01683_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsg.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsg_[a-z_0-9]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = C.CDLL(_abi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"declared in fsg.h but not exported: {missing}"


def test_binding_covers_the_header():
    assert sorted(_abi.SIGNATURES) == header_symbols()


def test_abi_version_and_defaults():
    L = _abi.lib()
    assert L.fsg_abi_version() == 1
    cfg = _abi.fsg_config()
    L.fsg_config_default(C.byref(cfg))
    assert list(cfg.dims) == [64, 64, 64]  # SessionConfig default (session.hpp:13)
    assert cfg.frame_mode == 2             # TranslationYaw (session.hpp:17)
    # units.hpp:25 ; test_lattice.cpp:276
    assert abs(L.fsg_tau(0.02, 0.004, 0.00089) - (0.5 + 3.0 * 0.00089 * 0.004 / (0.02 * 0.02))) < 1e-14


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_cuda_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    from paper_2206_01683_b200 import CoupledSession, FsgError, SessionConfig
    with pytest.raises(FsgError, match="no CUDA device"):
        CoupledSession(SessionConfig(dims=(16, 16, 16)))


def test_invalid_config_rejected_before_touching_the_device():
    """InputError cases of the reference (units.hpp:56-68, lattice.hpp:66-69)."""
    from paper_2206_01683_b200 import CoupledSession, InputError, SessionConfig
    with pytest.raises(InputError, match="tau"):
        CoupledSession(SessionConfig(dims=(16, 16, 16), nu=0.1, dx=0.02))
    with pytest.raises(InputError, match=">= 8"):
        CoupledSession(SessionConfig.lattice_units((4, 8, 8), 0.8))
    with pytest.raises(InputError, match="positive"):
        CoupledSession(SessionConfig(dims=(8, 8, 8), nu=0.0))
