"""C-ABI surface (CPU): the library loads, exports every symbol declared in
include/hykin_b200.h, and refuses to run without a B200 (no CPU fallback)."""
import ctypes as C
import re

import pytest

from paper_2505_03360_b200 import _abi


def test_library_exports_every_header_symbol():
    lib = C.CDLL(_abi.LIB_PATH)
    names = _abi.exported_symbols_from_header()
    assert len(names) >= 12
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_status_codes_match_header():
    text = open(_abi.HEADER).read()
    codes = dict(re.findall(r"(HK_[A-Z_]+) = (\d+)", text))
    for k, v in codes.items():
        assert getattr(_abi, k) == int(v), k


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _abi.lib()
    h = C.c_void_p()
    assert lib.hk_ctx_create(0, C.byref(h)) == _abi.HK_CUDA


def test_python_mirror_names():
    import paper_2505_03360_b200 as hk

    for n in ("precompute_kernel", "spectral_collision", "make_velocity_grid", "config_error",
              "aliasing_config_error", "numerical_consistency_error", "degenerate_state_error"):
        assert hasattr(hk, n), n
    assert issubclass(hk.aliasing_config_error, hk.config_error)
    with pytest.raises(hk.config_error):
        hk.make_velocity_grid(1, 8.0)
