"""CPU-side checks of the drop-in boundary: libmce_b200.so loads and exports
every entry point include/mce_b200.h declares (no compute calls here)."""

from __future__ import annotations

import ctypes
import os
import re

from paper_2212_01473_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "mce_b200.h")


def declared_functions() -> list[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mce_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("mce_graph_from_edges", "mce_degeneracy_order", "mce_reorder",
                     "mce_enumerate", "mce_graph_free", "mce_last_error"):
        assert required in names


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), f"{name} declared in mce_b200.h but not exported"
        assert isinstance(getattr(L, name), ctypes._CFuncPtr)


def test_ctypes_binding_covers_the_header():
    assert set(_lib.EXPORTS) == set(declared_functions())


def test_struct_layouts_match_header():
    # mce_run_config: 6 ints, 3 int64, int, int64, int64, double (natural alignment)
    assert ctypes.sizeof(_lib.RunConfigC) == 6 * 4 + 3 * 8 + 8 + 8 + 8 + 8
    assert ctypes.sizeof(_lib.RunResultC) == 10 * 8 + 8 * _lib.HIST_MAX


def test_last_error_is_callable_without_a_device():
    assert isinstance(_lib.lib().mce_last_error(), bytes)
