"""GPU parity against the reference's golden vectors and the pinned CPU oracle.

Every test here runs the CUDA path through the C ABI (libwsort_b200.so) and
compares with (a) fixtures frozen from the reference itself
(tests/golden/make_golden.py) and (b) the oracle (oracle/), which
tests/test_oracle.py pins against the same fixtures. Integer/byte work:
bit-exact equality is the only bar.
"""

import hashlib

import numpy as np
import pytest

from conftest import config_text
from oracle import oracle
from paper_1407_6603_b200 import _native, synth
from paper_1407_6603_b200.ingest import tokenize
from paper_1407_6603_b200.pipeline import DeviceCorpus, sort_text

pytestmark = pytest.mark.gpu


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def test_tokenize_matches_reference_kats(golden_tokenize):
    for case in golden_tokenize:
        text = bytes.fromhex(case["text"])
        assert [w.hex() for w in tokenize(text)] == case["tokens"], text[:80]


@pytest.mark.parametrize("naive", [True, False])
def test_sort_rows_matches_reference_stats(golden_stats, naive):
    key = "naive" if naive else "early-exit"
    for c in golden_stats:
        rows = synth.bucket_case(c["seed"], c["n"], c["width"], c["order"], c["alpha"])
        stats, _ = _native.sort_blocks([rows], naive)
        assert [int(x) for x in stats[0]] == c[key], c
        if naive:
            assert sha(rows.tobytes()) == c["sorted_sha"], c


def test_sort_blocks_batched_matches_reference(golden_stats):
    # every case of the fixture in ONE segmented call (widths repeat)
    cases = golden_stats[:120]
    rows = [synth.bucket_case(c["seed"], c["n"], c["width"], c["order"], c["alpha"]) for c in cases]
    stats, perms = _native.sort_blocks(rows, True, want_perms=True)
    for c, r, s, p in zip(cases, rows, stats, perms):
        assert [int(x) for x in s] == c["naive"], c
        assert sha(r.tobytes()) == c["sorted_sha"], c
        orig = synth.bucket_case(c["seed"], c["n"], c["width"], c["order"], c["alpha"])
        assert np.array_equal(orig[p.astype(np.int64)], r)
        # stable: equal rows keep corpus order
        if len(p) > 1:
            same = np.all(r[1:] == r[:-1], axis=1)
            assert np.all(p[1:][same] > p[:-1][same])


@pytest.mark.parametrize("cfg", ["0", "1", "2", "3", "4_prefix200k"])
def test_config_payload_and_stats(golden_configs, cfg):
    rec = golden_configs[cfg]
    text = config_text(rec)
    assert sha(text) == rec["text_sha"]
    # fused end-to-end call
    payload = sort_text(text)
    assert len(payload) == rec["payload_bytes"]
    assert sha(payload) == rec["payload_sha"]
    # phase-by-phase with stats
    dc = DeviceCorpus()
    dc.ingest(text)
    assert dc.histogram() == {int(k): v for k, v in rec["hist"].items()}
    dc.sort(want_stats=True)
    naive = dc.stats(naive=True)
    early = dc.stats(naive=False)
    for L, v in rec["per_length_stats"].items():
        assert list(naive[int(L)]) == v["naive"], (L, naive[int(L)], v)
        assert list(early[int(L)]) == v["early-exit"], (L, early[int(L)], v)
    assert sha(dc.payload()) == rec["payload_sha"]


def test_config4_full_matches_oracle():
    text = synth.generate(4)
    want, info = oracle.sort_text(text, mode="fast")
    got = sort_text(text)
    assert len(got) == len(want)
    assert got == want
    dc = DeviceCorpus()
    dc.ingest(text)
    dc.sort(want_stats=True)
    naive = dc.stats(naive=True)
    early = dc.stats(naive=False)
    for L, (n, inv, K, c, s, p) in info.items():
        assert naive[L] == (c, s, p), L
        P = min(K + 1, n - 1) if n >= 2 else 0
        assert early[L] == ((P * (n - 1) - P * (P - 1) // 2, inv, P) if n >= 2 else (0, 0, 0)), L
