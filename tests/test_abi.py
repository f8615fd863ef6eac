"""The C-ABI library: loads, exports every symbol include/wsort.h declares,
and behaves sanely without a GPU (no compute calls happen here)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1407_6603_b200 import _native

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "wsort.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(ws_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding_table():
    assert header_symbols() == sorted(_native.EXPORTS)


def test_header_constants_match_binding():
    text = HEADER.read_text()
    consts = dict((k, int(v)) for k, v in re.findall(r"#define\s+(WS_\w+)\s+(-?\d+)", text))
    for name, value in consts.items():
        if hasattr(_native, name):
            assert getattr(_native, name) == value, name
    for name in ("WS_INGEST_KEEP_TOKENS", "WS_INGEST_DEVICE_PTR", "WS_INGEST_RESIDENT",
                 "WS_INGEST_UNORDERED"):
        assert consts[name] == getattr(_native, name)


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_errors_without_device():
    lib = _native.load_library()
    assert lib.ws_version() >= 10000
    n = ctypes.c_int32(-1)
    assert lib.ws_device_count(ctypes.byref(n)) == 0
    if n.value == 0:
        h = ctypes.c_void_p()
        rc = lib.ws_create(ctypes.byref(h), 0)
        assert rc == _native.WS_ERR_CUDA
        assert b"CUDA" in lib.ws_last_error() or b"device" in lib.ws_last_error()
        with pytest.raises(RuntimeError):
            _native.Handle()


def test_closed_form_host_function():
    cf = _native.stats_closed_form
    assert cf(0, 0, 0, True) == (0, 0, 0)
    assert cf(1, 0, 0, False) == (0, 0, 0)
    assert cf(5, 3, 2, True) == (10, 3, 4)
    # sorted 5 words, early exit: one pass of 4 comparisons (test_engine.py:62-69)
    assert cf(5, 0, 0, False) == (4, 0, 1)
    # descending: K = n-1 -> full schedule
    assert cf(6, 15, 5, False) == (15, 15, 5)
    with pytest.raises(ValueError):
        cf(5, -1, 0, True)
    with pytest.raises(ValueError):
        cf(5, 0, 9, False)


def test_trivial_blocks_need_no_device():
    # n < 2 and width-0 blocks are answered without touching the GPU
    rows = [np.zeros((1, 4), np.uint8), np.zeros((0, 3), np.uint8), np.zeros((7, 0), np.uint8)]
    stats, perms = _native.sort_blocks(rows, naive=True, want_perms=True)
    assert stats.tolist() == [[0, 0, 0], [0, 0, 0], [21, 0, 6]]
    assert perms[2].tolist() == list(range(7))
    stats, _ = _native.sort_blocks([np.zeros((7, 0), np.uint8)], naive=False)
    assert stats.tolist() == [[6, 0, 1]]


def test_product_fails_loudly_without_gpu():
    from paper_1407_6603_b200 import sort_text, tokenize

    if _native.device_count() == 0:
        with pytest.raises(RuntimeError):
            tokenize(b"no gpu here")
        with pytest.raises(RuntimeError):
            sort_text(b"b a")
