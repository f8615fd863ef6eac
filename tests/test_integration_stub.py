"""The reference-side ctypes stub printed in INTEGRATION.md, executed as
written against this library: it must reproduce _bubble_rows exactly."""

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_1407_6603_b200 import _native, synth

ROOT = Path(__file__).resolve().parent.parent


def stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    src = next(b for b in blocks if "def bubble_rows" in b)
    return src.replace('ctypes.CDLL("libwsort_b200.so")', f'ctypes.CDLL({str(_native.LIB_PATH)!r})')


def test_stub_is_present_and_binds_the_abi():
    src = stub_source()
    assert "ws_sort_rows" in src and "ws_last_error" in src
    assert "ws_sort_rows" in _native.EXPORTS


@pytest.mark.gpu
@pytest.mark.parametrize("naive", [True, False])
def test_stub_matches_bubble_rows(naive):
    ns: dict = {}
    exec(compile(stub_source(), "INTEGRATION.md", "exec"), ns)
    for width, n, order in ((3, 2000, "random"), (9, 700, "descending"), (12, 1500, "dups"), (1, 5, "sorted")):
        rows = synth.bucket_case(width, n, width, order)
        ref = rows.copy()
        want = oracle.sort_rows_fast(ref, naive)[0]
        got = ns["bubble_rows"](rows, naive)
        assert tuple(got) == tuple(want) and np.array_equal(rows, ref)
