"""The C-ABI boundary: libmemo.so loads without a GPU and exports every entry
point include/memo.h declares; struct layouts in the ctypes mirror match."""
import ctypes as C
import os
import re

from paper_2407_12117_b200 import _abi
from paper_2407_12117_b200 import executor as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "memo.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(memo_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(_abi.lib, n)]
    assert not missing, missing


def test_version_and_error_plumbing():
    assert b"memo-b200" in _abi.lib.memo_version()
    rc = _abi.lib.memo_token_split_of(C.c_double(2.0), C.c_uint64(10), C.c_uint64(128),
                                      C.byref(_abi.TokenSplitC()))
    assert rc == _abi.MEMO_ERR_INPUT
    assert b"alpha" in _abi.lib.memo_last_error()


def test_struct_sizes_match_header():
    # sizes computed from the C declarations (x86-64 SysV)
    assert C.sizeof(_abi.ModelConfigC) == 10 * 8 + 8 + 10 * 8
    assert C.sizeof(_abi.HardwareConfigC) == 40
    assert C.sizeof(_abi.ScheduleEventC) == 32
    assert C.sizeof(_abi.SwapPlanC) == 56
    assert C.sizeof(E.ExecOptionsC) == 104
    o = E.default_options()
    assert o.token_granularity == 128 and o.swap_enabled == 1 and o.alignment == 512
