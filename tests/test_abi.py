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


def test_struct_layout_matches_header():
    # kk_csr_t: 3 x int64 + 2 enums + 3 pointers = 24 + 8 + 24
    assert ctypes.sizeof(_ffi.kk_csr_t) == 56
    assert ctypes.sizeof(_ffi.kk_spgemm_stats_t) == 8 * 3 + 4 * 6 + 8 * 32 + 16


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
