"""CPU-side checks of the boundary: libdtr.so loads and exports every symbol
include/dtr.h declares; host-only entry points behave (no GPU compute here)."""
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dtr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dtr_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2006_09616_b200 as P
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(P.lib, s), s
    assert sorted(P.EXPORTS) == syms


def test_strerror_and_version():
    import paper_2006_09616_b200 as P
    assert P.lib.dtr_version() == 1
    for code in range(9):
        assert P.lib.dtr_strerror(code)


def test_workspace_sizes():
    import paper_2006_09616_b200 as P
    dims = np.array([264, 391, 0, 264, 391, 1, 264, 391, 4], dtype=np.uint32)
    cta = P.workspace_bytes(dims, P.ENGINE_CTA)
    grid = P.workspace_bytes(dims, P.ENGINE_GRID)
    assert cta > 0 and grid > 0
    one = P.workspace_bytes(dims[:3], P.ENGINE_CTA)
    assert cta > one
    # invalid heuristic / engine
    import pytest
    with pytest.raises(P.DtrError):
        P.workspace_bytes(np.array([10, 10, 9], dtype=np.uint32), P.ENGINE_CTA)


def test_cell_and_row_layout():
    import paper_2006_09616_b200 as P
    assert P.CELL_DTYPE.itemsize == 64 and P.RESULT_DTYPE.itemsize == 96 and P.TRACE_DTYPE.itemsize == 32


def test_product_path_does_not_import_oracle():
    """The product package never imports oracle/ (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2006_09616_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/ (shares no code", ""), f


def test_header_struct_layouts_match_the_binding(tmp_path):
    """sizeof / offsetof of every struct in include/dtr.h (compiled by gcc) equal
    the numpy dtypes the binding marshals."""
    import subprocess
    import paper_2006_09616_b200 as P
    structs = {"dtr_cell": P.CELL_DTYPE, "dtr_result": P.RESULT_DTYPE, "dtr_evict_rec": P.TRACE_DTYPE,
               "dtr_adversary": P.ADV_DTYPE}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dtr.h"', "int main(void) {"]
    for s, dt in structs.items():
        lines.append(f'  printf("{s} sizeof %zu\\n", sizeof({s}));')
        for f in dt.names:
            lines.append(f'  printf("{s} {f} %zu\\n", offsetof({s}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)]).decode().split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for s, dt in structs.items():
        assert got[(s, "sizeof")] == dt.itemsize, s
        for f in dt.names:
            assert got[(s, f)] == dt.fields[f][1], (s, f)


def test_adversary_workspace_validation():
    import pytest
    import paper_2006_09616_b200 as P
    b = np.zeros(2, dtype=P.ADV_DTYPE)
    b["n"] = 100
    b["budget"] = 8
    b["heuristic"] = [8, 21]
    import ctypes as C
    nb = C.c_uint64(0)
    assert P.lib.dtr_adversary_workspace_bytes(C.c_void_p(b.ctypes.data), 2, C.byref(nb)) == 0 and nb.value > 256
    for field, bad in (("budget", 2), ("n", 0), ("heuristic", 9)):
        c = b.copy()
        c[field][0] = bad
        assert P.lib.dtr_adversary_workspace_bytes(C.c_void_p(c.ctypes.data), 2, C.byref(nb)) == 1   # DTR_E_INVAL
