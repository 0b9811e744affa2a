"""The C-ABI library loads on a CPU-only host and exports every symbol include/nsdgt.h declares."""
import ctypes
import os
import re

import paper_1307_4569_b200 as nsdgt
from paper_1307_4569_b200 import nsdgt as binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "nsdgt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(dgt_[a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_symbols_exported():
    names = declared_functions()
    assert "dgt_plan" in names and "dgt_execute" in names and "dgt_destroy" in names
    lib = ctypes.CDLL(binding.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(binding.EXPORTS) == names


def test_strerror_and_version():
    assert nsdgt.version().startswith("nsdgt")
    lib = binding._lib
    for code in (0, 2, 4, 5, 6, 7, 8):
        assert lib.dgt_strerror(code)
    assert b"unknown" in lib.dgt_strerror(99)


def test_null_pointer_errors_without_gpu():
    lib = binding._lib
    assert lib.dgt_execute(None, None, None, 1, None) == binding.DGT_EINVAL
    assert lib.dgt_plan_query(None, None) == binding.DGT_EINVAL
    h = ctypes.c_void_p()
    assert lib.dgt_plan(ctypes.byref(h), 36, 6, 6, 1, 2, None, 1, 0, 0, 0, 0, 0, None) == binding.DGT_EINVAL
    assert lib.dgt_launches_per_execute(None, 4) == 0


def test_no_oracle_import_in_product():
    """The product package never imports the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1307_4569_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, fn
                assert "dgt_oracle" not in txt, fn
