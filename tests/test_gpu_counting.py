"""Distinct-word counting (dedupe.cu): texts that repeat their vocabulary take
it in payload mode, high-cardinality texts keep the sort paths, and both give
the oracle's bytes (the reference's printed payload, cli.py:97, depends only on
which words a bucket holds and how often)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_1407_6603_b200 import _native, synth
from paper_1407_6603_b200._runtime import default_handle
from paper_1407_6603_b200.pipeline import BatchSorter, TextSorter, sort_text

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def counted_payload(text: bytes) -> tuple[bytes, int]:
    out = sort_text(text)
    return out, default_handle().counted_classes()


def want_of(text: bytes) -> bytes:
    return oracle.sort_text(text, mode="fast", max_len=2048)[0]


def test_repeated_vocabulary_is_counted():
    text = synth.generate(4, words=2_000_000, seed=11)  # ~16 MB, Zipf over a 200k-word vocabulary
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert mask == 0b1111, mask  # every lane class counted


def test_smaller_sample_of_the_vocabulary():
    """400k words of the same vocabulary: the short classes see too many
    distinct words for their budget (sorted), the long ones are counted."""
    text = synth.generate(4, words=400_000, seed=11)
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert mask != 0, mask


def test_config1_is_counted():
    text = synth.generate(1)  # 1.38 MB, Zipf over 20k words
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert mask & 1, mask


def test_high_cardinality_keeps_the_sort_paths():
    text = synth.generate(2)  # 1M mostly unique words
    got, mask = counted_payload(text)
    assert got == want_of(text)
    # lengths 1-2 have few possible words but 3-5 do not: class 0 as a whole is sorted
    assert mask == 0, mask


def test_descending_config3():
    text = synth.generate(3)
    got, mask = counted_payload(text)
    assert got == want_of(text)


def test_mixed_classes():
    """Short words repeat (class 0 counted) while the 6-10 character words are
    all distinct (class 1 over its table budget: sorted)."""
    rng = np.random.default_rng(3)
    short = [b"the", b"of", b"and", b"a", b"to", b"in", b"is", b"You", b"that", b"it", b"he7"]
    uniq = synth.random_words(17, 120_000, max_len=10, min_len=6)
    words = [short[i] for i in rng.integers(0, len(short), 400_000)] + list(uniq)
    order = rng.permutation(len(words))
    text = b" ".join(words[i] for i in order)
    assert len(text) >= 1 << 20
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert mask & 1 and not mask & 2, mask


def test_one_bucket_over_budget_sends_its_class_to_the_sort():
    """A class is counted only if every bucket of it stayed in budget."""
    rng = np.random.default_rng(4)
    rep5 = [b"aaaaa", b"bbbbb", b"Ccccc", b"9dddd"]
    uniq4 = synth.random_words(23, 60_000, max_len=4, min_len=4)  # > 4096 distinct, > n / 16
    words = [rep5[i] for i in rng.integers(0, 4, 300_000)] + list(uniq4)
    order = rng.permutation(len(words))
    text = b"\n".join(words[i] for i in order)
    assert len(text) >= 1 << 20
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert not mask & 1, mask


def test_late_overflow_after_a_passing_probe():
    """The probe sees a bucket's first keys only: a text that starts with one
    repeated word and then turns into distinct words passes it, the counting
    launch gives the class up later, and the class is sorted without the early
    launches (which ran for nobody)."""
    uniq6 = synth.random_words(31, 150_000, max_len=6, min_len=6)
    uniq3 = synth.random_words(37, 1000, max_len=3, min_len=3)  # within the 3-character bucket's budget
    text = b" ".join([b"Repeat"] * 20_000 + [b"the"] * 20_000 + list(uniq6) + list(uniq3) + [b"tail"] * 9000)
    assert len(text) >= 1 << 20
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert not mask & 2, mask  # class 1 (the 6-character bucket) ran out of budget
    assert mask & 1, mask      # class 0 repeats enough


def test_long_words_and_heavy_runs():
    """One word filling whole output tiles, runs of one, and words beyond 32
    characters (never counted) side by side."""
    rng = np.random.default_rng(6)
    words = [b"w"] * 300_000 + [b"Zebra"] * 70_000 + [b"q" * 32] * 5000 + [b"L" * 40, b"M" * 33] * 50
    words += list(synth.random_words(29, 3000, max_len=21, min_len=11))
    order = rng.permutation(len(words))
    text = b" ".join(words[i] for i in order)
    assert len(text) >= 1 << 20
    got, mask = counted_payload(text)
    assert got == want_of(text)
    assert mask & 1, mask


def test_resident_and_batch_paths():
    text = synth.generate(4, words=1_500_000, seed=7)
    want = want_of(text)
    ts = TextSorter(len(text))
    ts.load(text)
    for _ in range(3):  # repeated calls on one handle: the table pool is zeroed per call
        n = ts.run()
        assert ts.payload(n) == want
    assert ts.handle.counted_classes() == 0b1111
    # device-resident: the text stays from the last call
    n = ts.handle.sort_resident(len(text))
    p, size = ts.handle.output_device()
    assert size == n == len(want)
    assert _native.device_bytes(p, size) == want
    assert ts.handle.counted_classes() == 0b1111
    ts.close()
    bs = BatchSorter(len(text), inflight=3)
    bs.load(text)
    sizes = bs.run(6)
    for i, n in enumerate(sizes[-3:]):
        assert bs.payload((len(sizes) - 3 + i) % 3, n) == want
    bs.close()


SMALL = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
from oracle import oracle
from paper_1407_6603_b200 import synth
from paper_1407_6603_b200._runtime import default_handle
from paper_1407_6603_b200.pipeline import sort_text
rng = np.random.default_rng(1)
cases = [b"a", b"b a", b"pear Apple fig pear", b"word " * 1000, b"z" * 40 + b" z z",
         synth.generate(0), synth.prefix(synth.generate(4, words=50_000, seed=2), 20_000),
         b" ".join(synth.random_words(5, 3000, max_len=32)),
         b" ".join([b"ab", b"abc", b"abcdef", b"abcdefghijk", b"a" * 22] * 700)]
counted = 0
for t in cases:
    want = oracle.sort_text(t, mode="fast", max_len=2048)[0]
    assert sort_text(t) == want, t[:40]
    counted += default_handle().counted_classes() != 0
assert counted >= 5, counted
print("ok")
"""


def test_small_texts_through_the_counting_path():
    """WSORT_DEDUPE_MIN=0 and no small-corpus kernel: buckets of a few words
    (tables of 2n slots), single-word buckets, empty classes."""
    env = dict(os.environ, WSORT_DEDUPE_MIN="0", WSORT_NO_TINY="1")
    r = subprocess.run([sys.executable, "-c", SMALL.format(root=str(ROOT))], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
