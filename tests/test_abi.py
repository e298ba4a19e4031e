"""CPU-side checks of the boundary: the C-ABI library loads and exports every function
include/kk_spgemm.h declares; host-only entry points behave without a GPU."""
import ctypes
import os

import pytest

from paper_2103_11991_b200 import _ffi


def test_library_exports_header_symbols():
    lib = _ffi.load()
    names = _ffi.header_functions()
    assert {"kk_spgemm_symbolic", "kk_spgemm_numeric", "kk_spgemm_create", "kk_spgemm_destroy"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n


def test_status_strings():
    for s in range(8):
        assert _ffi.status_string(s).startswith("KK_")


def test_opts_default():
    o = _ffi.kk_spgemm_opts_default()
    assert (o.sort_rows, o.compression, o.validate, o.num_streams) == (1, -1, 0, 2)


def test_struct_layout_matches_header(tmp_path):
    """The ctypes structs have the sizes and field offsets the C compiler gives the header."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"kk_csr_t": _ffi.kk_csr_t, "kk_spgemm_opts_t": _ffi.kk_spgemm_opts_t,
               "kk_spgemm_stats_t": _ffi.kk_spgemm_stats_t, "kk_kernel_time_t": _ffi.kk_kernel_time_t}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "kk_spgemm.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(_ffi.__file__)), "include")
    subprocess.run([cc, "-I", inc, str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_create_fails_cleanly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_ffi.KKError) as e:
        _ffi.kk_spgemm_create(0)
    assert e.value.status in (_ffi.KK_ERR_CUDA, _ffi.KK_ERR_INVALID_ARG)


def test_no_oracle_in_product_package():
    pkg = os.path.dirname(_ffi.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(root, f)).read()
                for bad in ("import oracle", "from oracle", "kk_oracle", "kko_"):
                    assert bad not in src, (f, bad)
