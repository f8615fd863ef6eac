"""GPU edge cases: empty/ragged inputs, chunk/tile boundaries, long words,
separators, bucket sizes around every tile size and merge level."""

import numpy as np
import pytest

from oracle import oracle
from paper_1407_6603_b200 import _native, synth
from paper_1407_6603_b200.ingest import tokenize
from paper_1407_6603_b200.pipeline import DeviceCorpus, sort_text

pytestmark = pytest.mark.gpu


def check_text(text: bytes, stats: bool = True):
    want, info = oracle.sort_text(text, mode="fast", max_len=2048)
    assert sort_text(text) == want
    assert tokenize(text) == oracle.tokenize(text)
    if stats:
        dc = DeviceCorpus()
        dc.ingest(text)
        dc.sort(want_stats=True)
        naive = dc.stats(naive=True)
        early = dc.stats(naive=False)
        for L, (n, inv, K, c, s, p) in info.items():
            assert naive[L] == (c, s, p), L
            P = min(K + 1, n - 1) if n >= 2 else 0
            exp = (P * (n - 1) - P * (P - 1) // 2, inv, P) if n >= 2 else (0, 0, 0)
            assert early[L] == exp, L
        assert dc.payload() == want


@pytest.mark.parametrize("text", [
    b"", b" ", b"...", b"\x00\x80\xff", b"a", b"a b", b"b a cc", b"pear Apple fig",
    b"word " * 1000, b"z" * 4096, b"z" * 4097, b"q" * 5000 + b" " + b"r" * 33,
])
def test_small_texts(text):
    check_text(text)


def test_separator_bytes():
    rng = np.random.default_rng(5)
    seps = np.frombuffer(b" \t\n.,?!'\"-\x00\x80\xff\x7f@[`{/:", dtype=np.uint8)
    al = np.frombuffer(synth.ALNUM, dtype=np.uint8)
    for n in (1, 15, 16, 17, 31, 33, 4095, 4096, 4097, 12293, 100_003):
        t = al[rng.integers(0, 62, n)]
        m = rng.random(n) < 0.25
        t[m] = seps[rng.integers(0, len(seps), int(m.sum()))]
        check_text(t.tobytes())


def test_words_crossing_chunk_boundaries():
    # words straddling the 16/32-byte (thread), warp and 4/8 KiB (CTA chunk:
    # ordered / payload ingest) edges
    parts = []
    for edge in (16, 32, 512, 1024, 4096, 8192, 16384):
        pad = b"x " * ((edge - 7) // 2)
        parts.append(pad + b" ab" + b"C" * 9 + b"d" * 30 + b" ")
    check_text(b"".join(parts) * 3)


def test_word_spanning_whole_chunks_payload_mode():
    # a word covering several whole 8 KiB payload-mode chunks (no start or end
    # inside them) next to words that start / end exactly on chunk edges
    big = b"W" * 20000
    text = b"ab " * 2730 + b"c" + big + b" " + b"d" * 8191 + b" e" + b" f" * 9000
    want, _ = oracle.sort_text(text, mode="fast", max_len=40000)
    assert sort_text(text) == want
    for shift in range(1, 40, 7):
        t = b" " * shift + text
        assert sort_text(t) == want


def test_long_words_around_the_scan_bound():
    # the ingest measures a long word up to a bound (256 bytes past its
    # thread's segment) and leaves longer ones to the post-ingest length fix;
    # words around that bound, and short words that start in a chunk's last
    # segment and end past it (which that segment cannot tell from long
    # ones), at every alignment and next to chunk edges, in a text above the
    # tiny-path limit
    rng = np.random.default_rng(17)
    fill = b" ".join(synth.random_words(7, 120_000, max_len=12, min_len=1))
    parts = [fill[:300_000]]
    for L in (20, 33, 200, 255, 256, 257, 280, 287, 288, 289, 300, 511, 1000, 5000, 70_000):
        for off in (0, 1, 15, 16, 31):
            parts.append(b" " * (1 + off) + bytes(rng.choice(list(b"abcXYZ"), size=L)))
    for edge in (4096, 8192):  # ordered and payload chunk edges
        for short in (3, 20, 40):
            pos = sum(len(p) for p in parts)
            gap = (-pos - short // 2) % edge
            parts.append(b" " * max(gap, 1) + b"k" * short)
    parts.append(b" " + fill[300_000:])
    text = b"".join(parts)
    assert len(text) > 600_000
    want, _ = oracle.sort_text(text, mode="fast", max_len=80_000)
    assert sort_text(text) == want
    for shift in (1, 9):
        assert sort_text(b" " * shift + text) == want
    dc = DeviceCorpus()
    dc.ingest(text)
    dc.sort(want_stats=True)
    assert dc.payload() == want


@pytest.mark.parametrize("L", [1, 7, 8, 9, 16, 17, 24, 25, 32, 33, 40, 64, 65, 100, 1000])
def test_single_length_buckets(L):
    words = synth.random_words(L, 300, max_len=L, min_len=L)
    check_text(b" ".join(words))


def test_mixed_long_words():
    rng = np.random.default_rng(11)
    words = synth.random_words(3, 2000, max_len=90, min_len=1, alphabet=b"abAB01")
    words += [bytes(rng.choice(list(b"ab"), size=int(L))) for L in rng.integers(33, 300, 200)]
    rng.shuffle(words)
    check_text(b"\n".join(words))


def test_l1_bucket_all_symbols():
    al = list(synth.ALNUM)
    rng = np.random.default_rng(1)
    check_text(b" ".join(bytes([al[i]]) for i in rng.integers(0, 62, 20000)))


@pytest.mark.parametrize("n", [2047, 2048, 2049, 4095, 4096, 4097, 8191, 8193,
                               16385, 65537, 262145])
@pytest.mark.parametrize("order", ["random", "descending", "sorted", "dups"])
def test_bucket_sizes_around_tiles(n, order):
    for width in (5, 12):  # lanes 1 (T=4096) and 2 (T=2048)
        rows = synth.bucket_case(n + width, n, width, order)
        ref = rows.copy()
        (c, s, p), inv, K = oracle.sort_rows_fast(ref, naive=True)
        got = rows.copy()
        stats, perms = _native.sort_blocks([got], True, want_perms=True)
        assert np.array_equal(got, ref)
        assert tuple(int(x) for x in stats[0]) == (c, s, p)
        assert np.array_equal(rows[perms[0].astype(np.int64)], ref)
        early, _ = _native.sort_blocks([rows.copy()], False)
        P = min(K + 1, n - 1)
        assert tuple(int(x) for x in early[0]) == (P * (n - 1) - P * (P - 1) // 2, inv, P)


def test_wide_rows_generic_path():
    for width in (33, 40, 64, 65, 200):
        for order in ("random", "descending", "dups"):
            rows = synth.bucket_case(width, 3000, width, order)
            ref = rows.copy()
            st = oracle.bubble_rows(ref, naive=False) if width < 64 else oracle.sort_rows_fast(ref, False)[0]
            stats, _ = _native.sort_blocks([rows], False)
            assert np.array_equal(rows, ref)
            assert tuple(int(x) for x in stats[0]) == tuple(st)


def test_arbitrary_bytes_rows():
    # flat blocks may hold any byte values (0x00, 0xff, ...): unsigned order
    rng = np.random.default_rng(2)
    for width in (1, 3, 8, 9, 31):
        rows = rng.integers(0, 256, size=(5000, width), dtype=np.uint8)
        rows[::7] = 0xFF
        rows[::11] = 0
        ref = rows.copy()
        st = oracle.sort_rows_fast(ref, True)[0]
        stats, _ = _native.sort_blocks([rows], True)
        assert np.array_equal(rows, ref) and tuple(int(x) for x in stats[0]) == st


def test_chunked_h2d_long_word_redo():
    # > 16 MiB host text is copied in pieces overlapped with ingest; a word
    # longer than a piece forces the non-chunked re-ingest path
    rng = np.random.default_rng(21)
    body = b" ".join(synth.random_words(4, 2_000_000, max_len=12))
    giant = b"Q" * (20 << 20)
    text = body[: 9 << 20] + b" " + giant + b" " + body[9 << 20:] + b" " + giant + b"R"
    want, _ = oracle.sort_text(text, mode="fast", max_len=64)
    assert sort_text(text) == want


def test_chunked_h2d_matches_unchunked():
    text = synth.generate(4, words=4_000_000)
    assert len(text) > (16 << 20)
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want


def test_unordered_ingest_payload_and_state_errors():
    # WS_INGEST_UNORDERED (the payload-only path of ws_sort_text /
    # ws_sort_resident) reserves bucket runs per chunk with atomics: same
    # sorted payload, but stats / permutations must be refused
    for text in (synth.generate(0, seed=3), synth.generate(4, words=300_000, seed=4),
                 b"q" * 5000 + b" " + b"r" * 33 + b" a" * 7000):
        want, _ = oracle.sort_text(text, mode="fast", max_len=8192)
        h = _native.Handle(0)
        h.ingest_text(text, unordered=True)
        h.sort(False)
        assert h.emit_lines().tobytes() == want
        with pytest.raises(RuntimeError, match="corpus order"):
            h.sort(True)
        h.ingest_text(text)  # a later ordered ingest restores stats
        h.sort(True)
        assert h.emit_lines().tobytes() == want
        h.close()


def test_sort_texts_batch_matches_single_calls():
    # ws_sort_texts: many corpora with several in flight, each output equal to
    # its own ws_sort_text result (distinct corpora, repeated output buffers)
    texts = [synth.generate(0, seed=s) for s in range(5)] + [b"", b"b a", synth.generate(4, words=200_000, seed=9)]
    wants = [oracle.sort_text(t, mode="fast")[0] for t in texts]
    h = _native.Handle(0)
    for inflight in (1, 2, 3, 4):
        arrs = [np.frombuffer(t, dtype=np.uint8) if t else np.zeros(0, np.uint8) for t in texts]
        cap = max(len(t) for t in texts) + 1
        outs_pool = [np.empty(cap, dtype=np.uint8) for _ in range(inflight)]
        outs = [outs_pool[i % inflight] for i in range(len(texts))]
        # a slot finishes corpus i before i + inflight reuses its buffer: check
        # each result right after the batch only for the last corpus per slot
        sizes = h.sort_texts(arrs, outs, inflight)
        assert sizes == [len(w) for w in wants]
        for i in range(max(0, len(texts) - inflight), len(texts)):
            assert outs[i][: sizes[i]].tobytes() == wants[i]
        # distinct buffers: every output checked
        outs2 = [np.empty(cap, dtype=np.uint8) for _ in texts]
        sizes2 = h.sort_texts(arrs, outs2, inflight)
        assert all(o[:sz].tobytes() == w for o, sz, w in zip(outs2, sizes2, wants))
    with pytest.raises(ValueError):
        h.sort_texts([arrs[0]], [np.empty(3, dtype=np.uint8)], 2)
    h.close()


def test_ordered_ingest_chunked_stats_and_permutation():
    # > 16 MiB host text: chunked upload + ordered reserve ingest + reorder;
    # the stats and a bucket permutation must match corpus order exactly
    text = synth.generate(4, words=2_500_000, seed=12)
    assert len(text) > (16 << 20)
    want, info = oracle.sort_text(text, mode="fast")
    dc = DeviceCorpus()
    dc.ingest(text)
    dc.sort(want_stats=True)
    naive = dc.stats(naive=True)
    for L, (n, inv, K, c, s, p) in info.items():
        assert naive[L] == (c, s, p), L
    assert dc.payload() == want
    # the permutation of the L=3 bucket sorts the corpus-order words of length 3
    words3 = [w for w in oracle.tokenize(text) if len(w) == 3]
    lengths, counts, _ = dc.handle.buckets()
    b = lengths.index(3)
    perm = dc.handle.permutation(b, counts[b])
    assert [words3[i] for i in perm] == sorted(words3)


def _rand_words(rng, n, L, alphabet=synth.ALNUM):
    al = np.frombuffer(alphabet, dtype=np.uint8)
    return [bytes(r) for r in al[rng.integers(0, len(al), size=(n, L))]]


def test_sample_sort_shared_prefixes_and_skew():
    # payload-mode sample sort of the multi-lane classes: a splitter prefix
    # shared by thousands of distinct words (a prefix-equal slot beyond a tile:
    # the block odd-even fallback), a bucket half made of one word, uniform
    # random buckets, and bucket sizes around the tile and slot sizes
    rng = np.random.default_rng(77)
    words = [b"Qwertyuiopa" + w for w in _rand_words(rng, 6000, 5)]          # L = 16
    words += [b"Zz" * 6 + w for w in _rand_words(rng, 3000, 10)]              # L = 22
    words += [b"samewordx"] * 4000 + _rand_words(rng, 4000, 9)                # L = 9
    for L, n in ((12, 1791), (13, 1792), (14, 1793), (7, 3839), (8, 3840), (10, 3841),
                 (25, 20000), (32, 9000), (6, 50000)):
        words += _rand_words(rng, n, L)
    rng.shuffle(words)
    text = b" ".join(words)
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want


def test_sample_sort_descending_and_sorted_inputs():
    rng = np.random.default_rng(78)
    for L in (6, 11, 22):
        ws = sorted(_rand_words(rng, 30000, L, b"abcdefghijklmnopqrstuvwxyz"))
        for seq in (ws, ws[::-1]):
            text = b"\n".join(seq)
            want, _ = oracle.sort_text(text, mode="fast")
            assert sort_text(text) == want


def test_payload_mode_raw_byte_words():
    # word lists with arbitrary bytes (raw 8-bit keys) sorted without stats:
    # class 0 by the radix passes, the wider classes by the sample sort with
    # 8-byte prefixes (shared prefixes, 0x00 / 0xff bytes, many duplicates)
    rng = np.random.default_rng(90)
    words = []
    for L, n in ((1, 3000), (3, 9000), (4, 40000), (5, 30000), (8, 20000), (9, 25000),
                 (12, 20000), (17, 8000), (24, 6000), (31, 5000), (32, 4000), (40, 500)):
        rows = rng.integers(0, 256, size=(n, L), dtype=np.uint8)
        rows[::5] = rows[0]                       # duplicates
        rows[::7, : min(L, 9)] = 0xFF             # shared high prefixes
        rows[::11, : min(L, 8)] = 0x00            # shared low prefixes
        words += [bytes(r) for r in rows]
    rng.shuffle(words)
    h = _native.Handle(0)
    h.ingest_words(words)
    h.sort(False)
    want = b"".join(w + b"\n" for w in sorted(words, key=lambda w: (len(w), w)))
    assert h.emit_lines().tobytes() == want
    h.close()


def test_multilane_buckets_beyond_the_sample_budget():
    # buckets larger than the sample sort's splitter budget (class 2: 512
    # slots of 448 keys) take the merge path inside the same class
    rng = np.random.default_rng(91)
    words = _rand_words(rng, 260_000, 12) + _rand_words(rng, 50_000, 14) + _rand_words(rng, 9000, 7)
    words += [b"Repeatedword"] * 20_000
    rng.shuffle(words)
    text = b" ".join(words)
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want


from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=60, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 45), st.sampled_from([b"ab", b"aZ09", synth.ALNUM, b"q"]),
                          st.integers(1, 40)), min_size=0, max_size=12),
       st.sampled_from([b" ", b"\n", b"., ", b"\x00", b"\xff-"]), st.integers(0, 2**31))
def test_payload_and_stats_property(groups, sep, seed):
    # random mixtures of word lengths, alphabets (few symbols = many
    # duplicates), separators and counts: payload mode (radix / sample sort)
    # and stats mode (merge path) must both match the oracle
    rng = np.random.default_rng(seed)
    words = []
    for L, alphabet, count in groups:
        al = np.frombuffer(alphabet, dtype=np.uint8)
        words += [bytes(r) for r in al[rng.integers(0, len(al), size=(count * 37, L))]]
    rng.shuffle(words)
    check_text(sep.join(words))


def test_prefix_equal_slot_with_two_tails():
    # thousands of 9-byte words share their first 8 bytes (one prefix-equal
    # slot) and differ only in the last byte: the slot must be sorted whichever
    # key lands first in it (scatter order is arbitrary)
    h = _native.Handle(0)
    for rep in range(12):
        words = [b"\x00" * 8 + bytes([1 + (i + rep) % 2]) for i in range(6000)]
        words += [bytes([65 + i % 20]) * 9 for i in range(3000)]
        h.ingest_words(words)
        h.sort(False)
        want = b"".join(w + b"\n" for w in sorted(words))
        assert h.emit_lines().tobytes() == want, rep
    h.close()


def _short_word_text(rng, n, L=None, alphabet=synth.ALNUM):
    """n words of length L (or 1..5 at random) over `alphabet`, space-separated."""
    al = np.frombuffer(alphabet, dtype=np.uint8)
    lens = np.full(n, L) if L else rng.integers(1, 6, n)
    buf = np.full(int(lens.sum()) + n, ord(" "), dtype=np.uint8)
    ends = np.cumsum(lens + 1) - 1
    starts = ends - lens
    pos = np.repeat(starts, lens) + (np.arange(int(lens.sum())) - np.repeat(np.cumsum(lens) - lens, lens))
    buf[pos] = al[rng.integers(0, len(al), int(lens.sum()))]
    return buf.tobytes()


def test_radix_one_sweep_tiles_and_reuse():
    # class-0 buckets (<= 5 characters) of 1 .. ~300 radix tiles (5120 keys),
    # exact tile multiples, heavy duplicates; one handle reused across growing
    # and shrinking corpora (look-back status buffer growth, per-launch epochs)
    rng = np.random.default_rng(77)
    T = 5120  # radix.cu: 256 threads x WS_RADIX_E4 (20) keys per tile
    cases = [(1, 5, synth.ALNUM), (4095, 5, synth.ALNUM), (4096, 5, synth.ALNUM),
             (4097, 5, synth.ALNUM), (3 * 4096, 4, synth.ALNUM), (300_000, None, synth.ALNUM),
             (T - 1, 5, synth.ALNUM), (T, 5, synth.ALNUM), (T + 1, 3, synth.ALNUM),
             (5 * T, 4, synth.ALNUM), (5 * T + 1, 5, synth.ALNUM),
             (1_200_000, 5, b"ab"), (1_200_000, 5, synth.ALNUM), (5000, None, b"xyz"),
             (4096 * 7, 3, synth.ALNUM), (2, 5, synth.ALNUM)]
    for n, L, al in cases:
        text = _short_word_text(rng, n, L, al)
        want, _ = oracle.sort_text(text, mode="fast")
        assert sort_text(text) == want, (n, L, al)


def test_fused_payload_sort_then_emit_needs_sort():
    # ws_sort_text writes short-word buckets straight from the last radix pass
    # as payload (no sorted keys): a later emit is refused until ws_sort
    text = synth.generate(4, words=200_000, seed=8)
    want, _ = oracle.sort_text(text, mode="fast")
    h = _native.Handle(0)
    src = np.frombuffer(text, dtype=np.uint8)
    out = np.empty(len(text) + 64, dtype=np.uint8)
    n = h.sort_text(src, out)
    assert out[:n].tobytes() == want
    with pytest.raises(RuntimeError, match="fused sort"):
        h.emit_lines()
    h.sort(False)
    assert h.emit_lines().tobytes() == want
    h.close()


def test_slot_beyond_tile_keeps_input_for_a_second_sort():
    # The sample's positions (i * n / m) all hold the smallest word, every other
    # position a distinct larger word: all splitters are equal, so one slot
    # holds ~n keys, far beyond a slot sort's tile, and takes the in-CTA merge
    # sort. Its merge scratch must not be the input keys: a second ws_sort of
    # the same ingest reads them again (found as a 1-in-60 failure of
    # test_fused_payload_sort_then_emit_needs_sort on unordered ingests).
    rng2 = np.random.default_rng(11)
    n, m = 30_000, 256
    sampled = {i * n // m for i in range(m)}
    letters = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", np.uint8)
    words = []
    for i in range(n):
        words.append(b"000000" if i in sampled else bytes(letters[rng2.integers(0, 26, size=6)]))
    want = b"".join(w + b"\n" for w in sorted(words))
    h = _native.Handle(0)
    h.ingest_words(words)
    for _ in range(3):
        h.sort(False)
        assert h.emit_lines().tobytes() == want
    h.close()


def test_fused_slot_records_repeats_singletons_and_alignment():
    # multi-lane buckets (6..32 characters) whose slot sorts write payload
    # records directly: one word repeated 1..90k times (pattern fill at every
    # 16-byte phase), singleton slots, slots beyond a slot-sort tile (many
    # words sharing a 10-character prefix), mixed with random words
    rng = np.random.default_rng(2026)
    al = np.frombuffer(synth.ALNUM, dtype=np.uint8)
    words = []
    for L in (6, 7, 10, 11, 13, 21, 22, 31, 32):
        for reps in (1, 2, 3, 17, 255, 5000, 90_000 if L in (6, 22) else 1200):
            w = bytes(al[rng.integers(0, len(al), L)])
            words += [w] * reps
        words += [bytes(r) for r in al[rng.integers(0, len(al), size=(4000, L))]]
        pre = bytes(al[rng.integers(0, len(al), min(L - 1, 10))])
        words += [pre + bytes(r) for r in al[rng.integers(0, len(al), size=(3000, L - len(pre)))]]
    order = rng.permutation(len(words))
    text = b" ".join(words[i] for i in order)
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want
    h = _native.Handle(0)
    src = np.frombuffer(text, dtype=np.uint8)
    out = np.empty(len(text) + 64, dtype=np.uint8)
    for shift in range(3):  # the same corpus again on a reused handle
        n = h.sort_text(src, out)
        assert out[:n].tobytes() == want, shift
    h.close()


def test_counted_short_buckets_every_value_and_hot_words():
    # 1- and 2-character buckets are counted, not sorted (payload from
    # whole-key counts): every one of the 62 / 3844 values, hot values with
    # 10^5-10^6 copies (split over CTA parts), absent values, odd counts
    rng = np.random.default_rng(31)
    al = synth.ALNUM
    words = [bytes([c]) for c in al] + [bytes([a, b]) for a in al for b in al]
    words += [b"a"] * 1_000_003 + [b"Zz"] * 123_457 + [b"9"] * 7 + [b"q"] * 65_537
    words += [bytes([al[i % 62]]) * (1 + i % 2) for i in rng.integers(0, 62, 200_000)]
    order = rng.permutation(len(words))
    text = b"\n".join(words[i] for i in order)
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want
    sparse = b" ".join([b"x"] * 5 + [b"Q1"] * 3 + [b"abcdef"])
    assert sort_text(sparse) == oracle.sort_text(sparse, mode="fast")[0]


def test_slot_sort_shared_prefix_200k_is_n_log_n():
    # 200k distinct 14-character tokens sharing their first 10 characters
    # (timestamps / IDs): full-key splitters split them like any other words;
    # before, they all fell into one prefix-equal slot sorted by block
    # odd-even transposition, O((n / T)^2) tile sorts on one CTA.
    import time

    import torch

    from paper_1407_6603_b200._native import Handle

    rng2 = np.random.default_rng(7)
    words = [bytes(b"2024102010" + bytes(r)) for r in
             np.frombuffer(synth.ALNUM, np.uint8)[rng2.integers(0, 62, size=(200_000, 4))]]
    assert len(set(words)) > 190_000
    rng2.shuffle(words)
    text = b" ".join(words)
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want
    h = Handle(0)
    h.ingest_text(text, unordered=True)
    for _ in range(2):
        h.sort_resident(len(text))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.sort_resident(len(text))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    from paper_1407_6603_b200._native import device_bytes

    assert device_bytes(*h.output_device()) == want
    h.close()
    assert dt < 5e-3, f"shared-prefix bucket took {dt * 1e3:.2f} ms"


_MERGE_ROUTE = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
from oracle import oracle
from paper_1407_6603_b200 import synth
from paper_1407_6603_b200.pipeline import sort_text
rng = np.random.default_rng(9)
al = np.frombuffer(synth.ALNUM, np.uint8)
words = []
for L, n in ((7, 30000), (9, 4001), (12, 25000), (16, 7000), (23, 9001), (31, 2500)):
    words += [bytes(r) for r in al[rng.integers(0, 62, size=(n, L))]]
words += [b"Repeatedword"] * 5000 + [b"samewordx"] * 3000
rng.shuffle(words)
text = b" ".join(words)
want, _ = oracle.sort_text(text, mode="fast")
assert sort_text(text) == want
print("ok")
"""


@pytest.mark.parametrize("smax", ["2", "3", "5"])
def test_slot_merge_sort_route(smax):
    # WSORT_SAMPLE_SMAX caps the slots per bucket, so most slots exceed one
    # slot-sort tile and take the in-CTA merge sort (odd and even level counts,
    # a partial last pair, key-equal slots of repeated words)
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, WSORT_SAMPLE_SMAX=smax)
    r = subprocess.run([sys.executable, "-c", _MERGE_ROUTE.format(root=str(root))], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_checked_build_detector_fires():
    # the bounds-check detector of a checked build (WSORT_CHECKED=1) reports a
    # deliberately failing check; in a release build there are no checks
    import os
    import subprocess
    import sys
    from pathlib import Path

    if os.environ.get("WSORT_CHECKED") != "1":
        pytest.skip("release build: run under tools/checked_build.sh + WSORT_CHECKED=1")
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1407_6603_b200 import _native\n"
            "print(_native.debug_checks())\n") % str(Path(__file__).resolve().parent.parent)
    env = dict(os.environ, WSORT_CHECK_SELFTEST="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    fails, where = eval(r.stdout.strip().splitlines()[-1])
    # check_selftest_kernel: 32 threads check threadIdx.x != 0, so thread 0 fails
    assert fails == 1 and where.startswith("emit.cu:"), (fails, where)


def _words_text(rng, lengths, alphabet=synth.ALNUM):
    al = np.frombuffer(alphabet, dtype=np.uint8)
    return b" ".join(bytes(rng.choice(al, size=int(L))) for L in lengths)


@pytest.mark.parametrize("case", ["fits", "one_over_1lane", "one_over_2lane", "long_word", "all_lengths"])
def test_tiny_path_and_its_fallbacks(case):
    # texts <= 512 KiB first try tiny_sort_kernel (one CTA per bucket, right
    # after the ingest); a bucket beyond a CTA (15360 one-word / 7168
    # multi-word keys) or any word longer than 32 sends the call down the
    # class chains. Each case checks the payload of both outcomes, the handle's
    # state after it, and the batch API on the same texts.
    rng = np.random.default_rng(hash(case) % 1000)
    if case == "fits":
        text = _words_text(rng, np.full(15360, 5)) + b" " + _words_text(rng, np.full(7168, 12))
    elif case == "one_over_1lane":
        text = _words_text(rng, np.full(15361, 4))
    elif case == "one_over_2lane":
        text = _words_text(rng, np.full(7169, 11))
    elif case == "long_word":
        text = _words_text(rng, rng.integers(1, 20, 3000)) + b" " + b"L" * 40
    else:
        text = _words_text(rng, rng.integers(1, 33, 20000))
    assert len(text) <= 512 << 10
    want, _ = oracle.sort_text(text, mode="fast")
    assert sort_text(text) == want
    h = _native.Handle(0)
    texts = [np.frombuffer(t, dtype=np.uint8) for t in (text, text[: len(text) // 2])]
    outs = [np.zeros(len(t) + 64, dtype=np.uint8) for t in texts]
    sizes = h.sort_texts(texts, outs, inflight=2)
    for t, o, n in zip(texts, outs, sizes):
        assert o[:n].tobytes() == oracle.sort_text(t.tobytes(), mode="fast")[0]
