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


def _c_layout(struct: str, fields: list[str]) -> list[int]:
    """sizeof + offsetof of every field, as gcc lays out the header's struct."""
    import subprocess
    import tempfile

    body = "\n".join(f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields)
    src = (f'#include <stddef.h>\n#include <stdio.h>\n#include "mce_b200.h"\n'
           f'int main(void) {{ printf("%zu\\n", sizeof({struct})); {body} return 0; }}\n')
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        with open(c, "w") as fh:
            fh.write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        return [int(x) for x in subprocess.run([exe], capture_output=True, text=True,
                                               check=True).stdout.split()]


def test_struct_layouts_match_header():
    for struct, cls in (("mce_run_config", _lib.RunConfigC), ("mce_run_result", _lib.RunResultC)):
        names = [f[0] for f in cls._fields_]
        want = _c_layout(struct, names)
        got = [ctypes.sizeof(cls)] + [getattr(cls, f).offset for f in names]
        assert got == want, struct


def test_last_error_is_callable_without_a_device():
    assert isinstance(_lib.lib().mce_last_error(), bytes)


def test_worker_metric_columns_match_header():
    import re

    text = open(os.path.join(ROOT, "include", "mce_b200.h")).read()
    assert int(re.search(r"#define MCE_WM_COLS (\d+)", text).group(1)) == _lib.WM_COLS
