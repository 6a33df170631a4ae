"""Host-side checks of the C-ABI library (no GPU needed): it loads and exports every function
include/locc.h declares; the binding refuses to run without it (no fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "locc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(locc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("locc_load_weights", "locc_query", "locc_set_shapes", "locc_create", "locc_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2304_09439_b200 import build as b
    path = b.build()
    L = ctypes.CDLL(path)
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    from paper_2304_09439_b200 import locc
    assert set(locc.EXPORTS) == set(declared_functions())
    assert locc.version().startswith("locc-b200")


def test_status_strings_and_no_device_error():
    from paper_2304_09439_b200 import locc
    L = locc.lib()
    assert L.locc_status_string(-7) == b"LOCC_E_STATE"
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present: covered by the gpu tests")
    with pytest.raises(locc.LoccError):
        locc.Locc()  # no CUDA device here: must fail loudly, never fall back to the CPU


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2304_09439_b200 import locc
    monkeypatch.setattr(locc, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(locc, "_lib", None)
    with pytest.raises(ImportError):
        locc.lib()


def test_buffer_checks_before_the_library_is_called():
    """The binding checks dtype and length of every caller buffer: a wrong dtype or a
    buffer shorter than the call needs raises before any pointer reaches the library."""
    import numpy as np
    from paper_2304_09439_b200.locc import _ptr
    assert _ptr(None, np.float32, 10) is None
    a = np.zeros(10, np.float32)
    assert _ptr(a, np.float32, 10) == a.ctypes.data
    with pytest.raises(ValueError):
        _ptr(a, np.float32, 11)
    with pytest.raises(TypeError):
        _ptr(np.zeros(10, np.int64), np.int32, 10)
    import torch
    t = torch.zeros(3, 2, dtype=torch.int32)
    assert _ptr(t, np.int32, 6) == t.data_ptr()
    with pytest.raises(TypeError):
        _ptr(t.to(torch.int64), np.int32, 6)
    with pytest.raises(ValueError):
        _ptr(t, np.int32, 7)
    with pytest.raises(ValueError):
        _ptr(torch.zeros(4, 4).t(), np.float32, 16)  # non-contiguous


def test_nccl_unique_id_without_gpu():
    """NCCL is loaded at run time (dlopen) and the handshake id needs no GPU: 128 bytes, fresh each call."""
    from paper_2304_09439_b200 import locc
    a, b = locc.comm_unique_id(), locc.comm_unique_id()
    assert len(a) == 128 and a != b
