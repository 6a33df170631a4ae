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
