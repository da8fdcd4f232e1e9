"""The C-ABI library loads on any box and exports every symbol include/*.h declares;
the operator path has no CPU fallback."""
import ctypes

import numpy as np
import pytest

from paper_1803_11385_b200 import _lib


def test_library_exports_every_declared_symbol():
    names = _lib.declared_symbols()
    assert len(names) >= 35
    missing = []
    for n in names:
        try:
            getattr(_lib.lib, n)
        except AttributeError:
            missing.append(n)
    assert not missing, f"declared but not exported: {missing}"


def test_version_and_math_mode():
    assert b"sm_100a" in _lib.lib.hc_version()
    assert _lib.lib.hc_set_math(7) == _lib.HC_ERR_INVALID_ARGUMENT
    assert _lib.lib.hc_get_math() == _lib.HC_MATH_EXACT


def test_null_handles_are_invalid_arguments():
    info = np.zeros(6, np.int64)
    st = _lib.lib.hc_psh_info(None, info.ctypes.data_as(ctypes.c_void_p))
    assert st == _lib.HC_ERR_INVALID_ARGUMENT


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1803_11385_b200 import ops
    with pytest.raises(_lib.HashConvCudaError):
        ops.matmul(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32))
