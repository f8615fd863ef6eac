"""The CPU oracle pinned against golden vectors frozen from the reference.

The fixtures in tests/golden/ were produced by running the unmodified
reference package in the build container (tests/golden/make_golden.py). If
these pass, the oracle restates the reference exactly on: the tokenizer KATs
(ingest.py:15,26-28), 324 buckets of _bubble_rows stats in both variants
(engine.py:89-114), and the full payload + per-length stats of configs 0-3
and a 200k-word prefix of config 4.
"""

import hashlib

import numpy as np
import pytest

from conftest import config_text
from oracle import oracle
from paper_1407_6603_b200 import synth


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def test_tokenize_matches_reference(golden_tokenize):
    for case in golden_tokenize:
        text = bytes.fromhex(case["text"])
        assert [w.hex() for w in oracle.tokenize(text)] == case["tokens"]


def test_bubble_rows_matches_reference(golden_stats):
    for c in golden_stats:
        rows = synth.bucket_case(c["seed"], c["n"], c["width"], c["order"], c["alpha"])
        for naive, key in ((True, "naive"), (False, "early-exit")):
            r = rows.copy()
            assert list(oracle.bubble_rows(r, naive)) == c[key], c
            if naive:
                assert sha(r.tobytes()) == c["sorted_sha"]


def test_fast_path_matches_reference(golden_stats):
    for c in golden_stats:
        rows = synth.bucket_case(c["seed"], c["n"], c["width"], c["order"], c["alpha"])
        for naive, key in ((True, "naive"), (False, "early-exit")):
            r = rows.copy()
            st, inv, k = oracle.sort_rows_fast(r, naive)
            assert list(st) == c[key], c
            assert sha(r.tobytes()) == c["sorted_sha"]


@pytest.mark.parametrize("cfg", ["0", "1", "2", "3", "4_prefix200k"])
def test_config_payload_and_stats(golden_configs, cfg):
    rec = golden_configs[cfg]
    text = config_text(rec)
    assert sha(text) == rec["text_sha"], "synthetic generator drifted"
    payload, info = oracle.sort_text(text, mode="fast")
    assert len(payload) == rec["payload_bytes"]
    assert sha(payload) == rec["payload_sha"]
    assert {L: v[0] for L, v in info.items()} == {int(k): v for k, v in rec["hist"].items()}
    for L, v in rec["per_length_stats"].items():
        n, inv, K, c, s, p = info[int(L)]
        assert [c, s, p] == v["naive"]
        P = min(K + 1, n - 1) if n >= 2 else 0
        early = [P * (n - 1) - P * (P - 1) // 2, inv, P] if n >= 2 else [0, 0, 0]
        assert early == v["early-exit"]


def test_bubble_mode_pipeline_matches_reference(golden_configs):
    # the literal O(n^2) restatement, end to end (config 0: largest bucket ~7.6k)
    rec = golden_configs["0"]
    payload, info = oracle.sort_text(config_text(rec), mode="bubble", threads=4)
    assert sha(payload) == rec["payload_sha"]
    for L, v in rec["per_length_stats"].items():
        assert list(info[int(L)][3:6]) == v["naive"]


def test_closed_form_matches_bubble_random():
    rng = np.random.default_rng(0)
    for t in range(300):
        n = int(rng.integers(0, 60))
        w = int(rng.integers(1, 5))
        rows = rng.integers(97, 100, size=(n, w), dtype=np.uint8)
        for naive in (True, False):
            a, b = rows.copy(), rows.copy()
            assert oracle.bubble_rows(a, naive) == oracle.sort_rows_fast(b, naive)[0]
            assert np.array_equal(a, b)
