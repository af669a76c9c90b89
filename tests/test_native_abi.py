"""CPU-side checks of the C ABI library: it loads and exports every symbol include/*.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "surriga_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sg_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("sg_assemble", "sg_surrogate", "sg_result_copy", "sg_result_free", "sg_last_error"):
        assert s in syms


def test_library_loads_and_exports_all_symbols():
    from paper_1904_06971_b200 import _lib

    L = ctypes.CDLL(_lib.LIB_PATH)  # RTLD_NOW semantics: unresolved symbols fail here
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_lib.SYMBOLS) <= set(declared_symbols())
    assert _lib.lib().sg_version().startswith(b"surriga_b200")
    assert _lib.lib().sg_max_degree() >= 4


def test_no_device_call_fails_loudly_without_gpu():
    import numpy as np
    import pytest

    import paper_1904_06971_b200 as pkg

    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    disc = pkg.make_discretization(pkg.unit_square(), 1, (4, 4))
    with pytest.raises(Exception):
        pkg.assemble(pkg.FormKind.POISSON, disc)
