"""The C-ABI library loads on CPU and exports every entry point that
include/trisplat_b200.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from conftest import REPO


def declared_functions():
    src = open(os.path.join(REPO, "include", "trisplat_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(ts_\w+)\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("ts_forward", "ts_backward", "ts_context_create", "ts_context_destroy",
                 "ts_error_string", "ts_debug_copy"):
        assert must in names


def test_library_exports_all_declared_symbols():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2505_19175_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) <= set(declared_functions())
    lib2 = _lib.load()
    assert lib2.ts_version().decode().startswith("trisplat_b200")
    assert lib2.ts_error_string(-5).decode() == "non-finite triangle parameters"


def test_abi_struct_sizes():
    from paper_2505_19175_b200 import _lib
    assert ctypes.sizeof(_lib.TsCamera) == 5 * 8 + 12 * 8 + 8
    assert ctypes.sizeof(_lib.TsOptions) == 16 + 16 + 24 + 16
    assert ctypes.sizeof(_lib.TsSoup) == 40
    assert ctypes.sizeof(_lib.TsForwardOut) == 56
    assert ctypes.sizeof(_lib.TsForwardResult) == 56
