"""The C-ABI library loads without a GPU and exports every symbol include/ficco.h declares."""
import ctypes
import pathlib
import re

import pytest

from paper_2512_10236_b200 import runtime

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared_symbols() -> set[str]:
    text = (ROOT / "include" / "ficco.h").read_text()
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(ficco_\w+)\s*\(", text, flags=re.M))


def test_header_declares_the_runtime_exports():
    assert declared_symbols() == set(runtime.EXPORTED)


def test_library_loads_and_exports_everything():
    if not runtime.LIB_PATH.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = runtime.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.ficco_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors == the C compiler's view of include/ficco.h (sizes and field offsets)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    fields = {"ficco_copy_op": runtime.CopyOp, "ficco_tile": runtime.Tile, "ficco_operand": runtime.Operand,
              "ficco_plan_desc": runtime.PlanDesc}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "ficco.h"', "int main(void) {"]
    for cname, py in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["return 0; }"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.split("\n") if line)
    for cname, py in fields.items():
        assert int(out[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_errors_without_gpu_are_reported_not_raised_in_c():
    if not runtime.LIB_PATH.exists():
        pytest.skip("library not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = runtime.load_library()
    n = ctypes.c_int()
    rc = lib.ficco_device_info(0, ctypes.byref(n), None, None)
    assert rc == -2 and lib.ficco_last_error()
