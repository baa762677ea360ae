"""The C-ABI library loads and exports every symbol include/bs.h declares (no GPU needed)."""
import ctypes
import os
import subprocess
import tempfile

import pytest

from paper_2506_01576_b200 import bs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    L = bs.lib()
    syms = bs.header_symbols()
    assert len(syms) >= 16
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_struct_sizes_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "bs.h"\n#include <stdio.h>\n'
                   'int main(void){printf("%zu %zu %zu\\n", sizeof(bs_layout), sizeof(bs_launch), sizeof(bs_info));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    a, b, c = map(int, subprocess.check_output([str(exe)]).split())
    assert a == ctypes.sizeof(bs.bs_layout)
    assert b == ctypes.sizeof(bs.bs_launch)
    assert c == ctypes.sizeof(bs.bs_info)


def test_layout_default_and_version():
    lay = bs.bs_layout_default()
    assert lay.struct_size == ctypes.sizeof(bs.bs_layout)
    assert lay.key_bytes == 8 and lay.out_bytes == 8
    assert lay.variant == bs.KARY and lay.k == 5 and lay.leaf_chunk == 0
    # schedule and L2 hints are resolved by bs_build from the array size (include/bs.h)
    assert lay.kary_mode == 8 and lay.cache_hints == 0x100
    assert "sm_100a" in bs.bs_version()


def test_argument_validation_without_gpu():
    """Validation happens before any CUDA call, so it works on a CPU-only box."""
    L = bs.lib()
    h = ctypes.c_void_p()
    lay = bs.bs_layout_default()
    dummy = ctypes.c_uint64(0)
    # n == 0 (P:65 needs n >= 1)
    assert L.bs_build(ctypes.addressof(dummy), 0, ctypes.byref(lay), ctypes.byref(h)) == bs.BS_ERR_INVALID
    assert "n == 0" in bs.bs_last_error()
    bad = bs.bs_layout_default(key_bytes=3)
    assert L.bs_build(ctypes.addressof(dummy), 1, ctypes.byref(bad), ctypes.byref(h)) == bs.BS_ERR_INVALID
    bad = bs.bs_layout_default(k=34)
    assert L.bs_build(ctypes.addressof(dummy), 1, ctypes.byref(bad), ctypes.byref(h)) == bs.BS_ERR_INVALID
    bad = bs.bs_layout_default(leaf_chunk=12)
    assert L.bs_build(ctypes.addressof(dummy), 1, ctypes.byref(bad), ctypes.byref(h)) == bs.BS_ERR_INVALID
    bad = bs.bs_layout_default(out_bytes=4)
    assert L.bs_build(ctypes.addressof(dummy), 1 << 31, ctypes.byref(bad), ctypes.byref(h)) == bs.BS_ERR_INVALID
    bad = bs.bs_layout_default()
    bad.struct_size = 4
    assert L.bs_build(ctypes.addressof(dummy), 1, ctypes.byref(bad), ctypes.byref(h)) == bs.BS_ERR_INVALID
    bad = bs.bs_layout_default()
    bad.reserved[0] = 1
    assert L.bs_build(ctypes.addressof(dummy), 1, ctypes.byref(bad), ctypes.byref(h)) == bs.BS_ERR_INVALID
    assert L.bs_build(None, 1, ctypes.byref(lay), ctypes.byref(h)) == bs.BS_ERR_INVALID
    assert L.bs_lookup(None, None, 0, None, None) == bs.BS_ERR_INVALID
    L.bs_destroy(None)   # NULL-safe


def test_graft_entry_build_compiles_everything():
    import __graft_entry__ as g
    g.build()
    assert os.path.exists(bs.LIB_PATH)
