"""The reference's own test strategy (pkg/tests/*.py), restated against this
package's mirror of the `wordsort` API, running on the GPU.

Each test names the reference test it restates. Deliberate deviations (tests
that encode CPU-thread assumptions) are listed at the bottom.
"""

import random
import string
import subprocess
import sys
import threading
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_1407_6603_b200.cli import main
from paper_1407_6603_b200.engine import (
    SchedulePolicy, SortConfig, SortStats, SortVariant, bubble_sort_bucket, sort_all_parallel,
    sort_all_sequential,
)
from paper_1407_6603_b200.ingest import WORD_RE, load_text, preprocess_stats, tokenize
from paper_1407_6603_b200.store import (
    LayoutKind, build_buckets, build_flat, build_store, emit_sorted,
)
from paper_1407_6603_b200.verify import oracle_sorted, verify_words

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
ALNUM = (string.ascii_letters + string.digits).encode()
ALNUM_SET = frozenset(ALNUM)


def make_corpus(seed, count, max_len=12, min_len=1):
    rng = random.Random(seed)
    return [bytes(rng.choices(ALNUM, k=rng.randint(min_len, max_len))) for _ in range(count)]


class TaggedWord(bytes):
    def __new__(cls, value, tag):
        self = super().__new__(cls, value)
        self.tag = tag
        return self


words_st = st.lists(
    st.text(alphabet=string.ascii_letters + string.digits, min_size=1, max_size=12).map(str.encode),
    max_size=80)


# --- test_ingest.py -----------------------------------------------------------

def test_load_text(tmp_path):
    p = tmp_path / "f.txt"
    p.write_bytes(b"a\r\nb\rc\n")
    assert load_text(p) == b"a\r\nb\rc\n"
    with pytest.raises(OSError):
        load_text(tmp_path / "nope.txt")


@pytest.mark.parametrize("text,expected", [
    (b"HAMLET, PRINCE!", [b"HAMLET", b"PRINCE"]), (b"don't", [b"don", b"t"]), (b"", []),
    (b"...", []), (b"a1b2 3", [b"a1b2", b"3"]), (b"caf\xc3\xa9", [b"caf"]),
    (b"caf\xc3\xa9s", [b"caf", b"s"]),
])
def test_tokenize_examples(text, expected):
    assert tokenize(text) == expected


@settings(max_examples=60, deadline=None)
@given(st.binary(max_size=300))
def test_tokenize_properties(data):
    words = tokenize(data)
    assert all(len(w) >= 1 and all(b in ALNUM_SET for b in w) for w in words)
    assert tokenize(bytes(data)) == words
    assert tokenize(b" ".join(words)) == words


@settings(max_examples=60, deadline=None)
@given(st.binary(max_size=200), st.integers(0, 200),
       st.sampled_from([b"!", b" ", b"\x00", b"\xff", b"'", b"\n"]))
def test_tokenize_separator_insertion_invariance(data, pos, sep):
    valid = [i for i in range(len(data) + 1)
             if not (0 < i < len(data) and data[i - 1] in ALNUM_SET and data[i] in ALNUM_SET)]
    pos = valid[pos % len(valid)]
    assert sorted(tokenize(data[:pos] + sep + data[pos:])) == sorted(tokenize(data))


def test_preprocess_stats(tmp_path):
    p = tmp_path / "f.txt"
    p.write_bytes(b"some words here and there")
    t = preprocess_stats(p)
    assert t.load_strip_seconds >= 0 and t.bucket_build_seconds >= 0
    p.write_bytes(b"")
    assert preprocess_stats(p).load_strip_seconds >= 0
    with pytest.raises(OSError):
        preprocess_stats(tmp_path / "nope.txt")


# --- test_store.py --------------------------------------------------------------

def test_build_flat_examples():
    m = build_flat([b"ab", b"cd"])
    assert m.blocks[2].tobytes() == b"abcd" and m.count_for_length(2) == 2
    assert m.blocks[2].dtype == np.uint8
    m = build_flat([b"x"])
    assert m.blocks[1].tobytes() == b"x" and m.lmax == 1
    m = build_flat([b"abc", b"def", b"gh"])
    assert m.blocks[3].shape == (2, 3) and m.blocks[3].flags["C_CONTIGUOUS"]
    assert m.blocks[3].nbytes == 6 and m.blocks[2].nbytes == 2
    assert emit_sorted(build_flat([])) == []


@settings(max_examples=40, deadline=None)
@given(words_st)
def test_layouts_hold_same_words_per_bucket(words):
    ragged, flat = build_buckets(words), build_flat(words)
    assert ragged.lengths() == flat.lengths()
    for L in ragged.lengths():
        assert ragged.words_for_length(L) == flat.words_for_length(L)


@settings(max_examples=40, deadline=None)
@given(words_st)
def test_emit_sorted_matches_oracle_and_multiset(words):
    for layout in LayoutKind:
        store = build_store(words, layout)
        sort_all_sequential(store, SortVariant.NAIVE)
        assert emit_sorted(store) == oracle_sorted(words)


def test_build_flat_any_bytes_and_empty_words():
    # like the reference, empty words form a (k, 0) block (store.py:94-95);
    # its words_for_length(0) cannot split them (range step 0) in either package
    words = [b"\xff\x00", b"", b"\x80", b"", b"zz"]
    m = build_flat(words)
    assert m.blocks[0].shape == (2, 0)
    assert m.words_for_length(2) == [b"\xff\x00", b"zz"]
    st = sort_all_sequential(m, SortVariant.NAIVE)
    assert st == SortStats(1 + 1, 1, 1 + 1)  # (0,b"") pair + (ff00, zz) swapped once
    assert m.words_for_length(2) == [b"zz", b"\xff\x00"] and m.words_for_length(1) == [b"\x80"]


# --- test_engine.py --------------------------------------------------------------

def sort_single_bucket(words, layout, variant):
    store = build_store(words, layout)
    (length,) = store.lengths()
    stats = bubble_sort_bucket(store, length, variant)
    return store.words_for_length(length), stats


@pytest.mark.parametrize("layout", list(LayoutKind))
def test_engine_kats(layout):
    out, s = sort_single_bucket([b"cab", b"abc", b"bca"], layout, SortVariant.NAIVE)
    assert out == [b"abc", b"bca", b"cab"] and s.comparisons == 3
    words = [b"aa", b"bb", b"cc", b"dd", b"ee"]
    out, s = sort_single_bucket(words, layout, SortVariant.EARLY_EXIT)
    assert out == words and (s.passes, s.comparisons, s.swaps) == (1, 4, 0)
    words = [bytes([c]) * 3 for c in random.Random(7).sample(range(97, 123), 5)]
    assert sort_single_bucket(words, layout, SortVariant.NAIVE)[1].comparisons == 10
    for variant in SortVariant:
        for w in ([], [b"zz"]):
            assert sort_all_sequential(build_store(w, layout), variant) == SortStats(0, 0, 0)


@settings(max_examples=30, deadline=None)
@given(st.integers(0, 200), st.integers())
def test_comparison_laws(n, seed):
    rng = random.Random(seed)
    words = [bytes(rng.choices(b"abcd", k=4)) for _ in range(n)]
    for layout in LayoutKind:
        s = sort_all_sequential(build_store(words, layout), SortVariant.NAIVE)
        assert s.comparisons == n * (n - 1) // 2
        e = sort_all_sequential(build_store(words, layout), SortVariant.EARLY_EXIT)
        assert e.comparisons <= n * (n - 1) // 2 and e.swaps <= e.comparisons


@pytest.mark.parametrize("layout", list(LayoutKind))
def test_early_exit_sorted_is_n_minus_1(layout):
    for n in range(2, 40):
        words = sorted(bytes([97 + i % 26, 97 + i // 26]) for i in range(n))
        assert sort_single_bucket(words, layout, SortVariant.EARLY_EXIT)[1].comparisons == n - 1


@pytest.mark.parametrize("variant", list(SortVariant))
def test_stability_ragged_tagged_duplicates(variant):
    rng = random.Random(11)
    words = [TaggedWord(bytes(rng.choices(b"ab", k=3)), tag=i) for i in range(200)]
    store = build_buckets(list(words))
    bubble_sort_bucket(store, 3, variant)
    bucket = store.buckets[3]
    assert all(isinstance(w, TaggedWord) for w in bucket)
    for prev, cur in zip(bucket, bucket[1:]):
        assert prev <= cur
        if prev == cur:
            assert prev.tag < cur.tag


@pytest.mark.parametrize("variant", list(SortVariant))
def test_flat_and_ragged_stats_identical(variant):
    for seed in range(10):
        words = make_corpus(seed, 300, max_len=6)
        assert (sort_all_sequential(build_buckets(words), variant)
                == sort_all_sequential(build_flat(words), variant))
    for layout in LayoutKind:
        assert sort_all_sequential(build_store([b"same"] * 500, layout), variant).swaps == 0


def test_aggregate_is_sum_over_buckets():
    store = build_buckets([b"b", b"a", b"xx", b"zz", b"yy"])
    assert sort_all_sequential(store, SortVariant.NAIVE).comparisons == 4


# --- test_parallel.py ----------------------------------------------------------

@pytest.mark.parametrize("layout", list(LayoutKind))
@pytest.mark.parametrize("variant", list(SortVariant))
@pytest.mark.parametrize("schedule", list(SchedulePolicy))
@pytest.mark.parametrize("threads", [1, 2, 3, 8, 16])
def test_parallel_equals_sequential(layout, variant, schedule, threads):
    words = make_corpus(threads * 100 + 1, 300)
    seq = build_store(words, layout)
    seq_stats = sort_all_sequential(seq, variant)
    par = build_store(words, layout)
    stats = sort_all_parallel(par, SortConfig(layout, variant, threads, schedule))
    assert emit_sorted(par) == oracle_sorted(words) == emit_sorted(seq)
    assert stats == seq_stats


def test_concurrent_calls_on_disjoint_stores():
    words_a, words_b = make_corpus(1, 3000), make_corpus(2, 3000)
    store_a = build_store(words_a, LayoutKind.RAGGED)
    store_b = build_store(words_b, LayoutKind.FLAT)
    results, errors = {}, []

    def run(name, store, layout):
        try:
            results[name] = sort_all_parallel(store, SortConfig(layout, SortVariant.NAIVE, 4))
        except BaseException as exc:  # surfaced below
            errors.append(exc)

    ts = [threading.Thread(target=run, args=("a", store_a, LayoutKind.RAGGED)),
          threading.Thread(target=run, args=("b", store_b, LayoutKind.FLAT))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
    assert emit_sorted(store_a) == oracle_sorted(words_a)
    assert emit_sorted(store_b) == oracle_sorted(words_b)


# --- test_acceptance.py ------------------------------------------------------------

def test_criterion_1_oracle_equivalence():
    rng = random.Random(2024)
    for i in range(150):
        words = make_corpus(rng.randrange(2**31), rng.randint(0, 500), max_len=12)
        expected = oracle_sorted(words)
        for layout in LayoutKind:
            for variant in SortVariant:
                store = build_store(words, layout)
                sort_all_parallel(store, SortConfig(layout, variant, 4))
                assert emit_sorted(store) == expected, (i, layout, variant)


def test_criterion_2_3_comparison_laws():
    rng = random.Random(2)
    for n in range(0, 201, 7):
        words = [bytes(rng.choices(ALNUM, k=6)) for _ in range(n)]
        for layout in LayoutKind:
            assert sort_all_sequential(build_store(words, layout),
                                       SortVariant.NAIVE).comparisons == n * (n - 1) // 2
    for n in range(2, 201, 7):
        words = sorted(bytes(rng.choices(ALNUM, k=5)) for _ in range(n))
        for layout in LayoutKind:
            assert sort_all_sequential(build_store(words, layout),
                                       SortVariant.EARLY_EXIT).comparisons == n - 1


def test_criterion_6_cli_determinism(tmp_path):
    corpus = b" ".join(make_corpus(66, 48_000, max_len=40))
    path = tmp_path / "big.txt"
    path.write_bytes(corpus)
    outputs = set()
    for i in range(20):
        out = tmp_path / f"out_{i}.txt"
        assert main(["sort", str(path), "--threads", "16", "--output", str(out)]) == 0
        outputs.add(out.read_bytes())
    assert len(outputs) == 1
    words = make_corpus(66, 48_000, max_len=40)
    assert outputs.pop() == b"".join(w + b"\n" for w in oracle_sorted(words))


def test_criterion_9_tokenizer_properties():
    rng = random.Random(9)
    seps = b" \t\n.,?!'\"-\x00\x80\xff"
    for _ in range(2000):
        data = rng.randbytes(rng.randint(0, 120))
        words = tokenize(data)
        assert all(len(w) >= 1 and all(b in ALNUM_SET for b in w) for w in words)
        valid = [i for i in range(len(data) + 1)
                 if not (0 < i < len(data) and data[i - 1] in ALNUM_SET and data[i] in ALNUM_SET)]
        pos = valid[rng.randrange(len(valid))]
        spliced = data[:pos] + bytes([seps[rng.randrange(len(seps))]]) + data[pos:]
        assert sorted(tokenize(spliced)) == sorted(words)


# --- test_cli.py ---------------------------------------------------------------------

def run_cli(capsys, *argv):
    status = main([str(a) for a in argv])
    out, err = capsys.readouterr()
    return status, out, err


def test_cli(capsys, tmp_path):
    p = tmp_path / "in.txt"
    p.write_bytes(b"b a cc")
    assert run_cli(capsys, "sort", p, "--threads", 1)[:2] == (0, "a\nb\ncc\n")
    p.write_bytes(b"")
    assert run_cli(capsys, "sort", p)[:2] == (0, "")
    status, out, err = run_cli(capsys, "sort", tmp_path / "nope.txt")
    assert status == 1 and "error" in err and out == ""
    p.write_bytes(b" ".join(make_corpus(14, 300)))
    assert run_cli(capsys, "sort", p, "--layout", "ragged")[1] == run_cli(capsys, "sort", p)[1]
    with pytest.raises(SystemExit):
        main(["sort", str(p), "--bogus"])
    p.write_bytes(b"a bb a")
    status, out, _ = run_cli(capsys, "preprocess", p)
    lines = out.splitlines()
    assert status == 0 and "words,3" in lines and "lmax,2" in lines and "hist,1,2" in lines
    status, out, _ = run_cli(capsys, "verify", p, "--sizes", "0,50")
    assert status == 0 and "OK (3 words)" in out and "OK (50 words)" in out


def test_console_entry_point_subprocess(tmp_path):
    p = tmp_path / "in.txt"
    p.write_bytes(b"pear Apple fig")
    proc = subprocess.run([sys.executable, "-m", "paper_1407_6603_b200.cli", "sort", str(p),
                           "--threads", "1"], capture_output=True, cwd=str(ROOT))
    assert proc.returncode == 0, proc.stderr
    assert proc.stdout == b"fig\npear\nApple\n"


def test_verify_words_all_layouts():
    assert verify_words(make_corpus(5, 400)) is None


# Deliberate deviations from the reference suite (CPU-thread assumptions):
#  * test_parallel.py::test_worker_count_capped_by_bucket_count -- the GPU
#    path spawns no worker threads (one segmented launch replaces the pool).
#  * test_acceptance.py criterion 7/8 and test_bench.py strip<sort -- timing
#    relations of the CPU implementation.
# test_bench.py (speedup / efficiency arithmetic, CSV / JSON / plot reports,
# the timing matrix and the `bench` subcommand) is restated in
# tests/test_harness.py against paper_1407_6603_b200/harness.py.


@pytest.mark.parametrize("case", ["config1", "long_words", "chunked"])
def test_preprocess_device_histogram(tmp_path, case, capsys):
    # `wordsort preprocess` prints words / lmax / hist from the device's bucket
    # counts (cli.py:171-181); they must equal the reference tokenizer's
    from collections import Counter

    from paper_1407_6603_b200 import synth
    from paper_1407_6603_b200.ingest import preprocess_device

    if case == "config1":
        text = synth.generate(1)
    elif case == "long_words":
        text = b"x" * 40 + b" a bb " + b"Q" * 33 + b"!" + b"q" * 40 + b" " + b"z" * 200
    else:  # > 16 MiB: chunked upload overlapped with the ingest
        text = synth.generate(4, words=2_400_000, seed=3)
    p = tmp_path / "in.txt"
    p.write_bytes(text)
    want = Counter(len(w) for w in WORD_RE.findall(text))
    pre = preprocess_device(p)
    assert pre.hist == dict(want) and pre.words == sum(want.values())
    assert pre.lmax == max(want)
    assert pre.timings.load_strip_seconds > 0 and pre.timings.bucket_build_seconds >= 0
    status, out, _ = run_cli(capsys, "preprocess", p)
    lines = out.splitlines()
    assert status == 0 and f"words,{sum(want.values())}" in lines and f"lmax,{max(want)}" in lines
    assert [ln for ln in lines if ln.startswith("hist,")] == [f"hist,{L},{want[L]}" for L in sorted(want)]
