"""Seeded synthetic corpora standing in for BASELINE.json configs 0-4.

The paper measures on two Hamlet text files (190 KB and 1.38 MB)
that are not available here; configs 0 and 1 are English-like stand-ins with
the shapes BASELINE.json states, configs 2-4 are the synthetic stress cases
it defines. Every generator is a pure function of (config, seed) built on
numpy's PCG64 ``default_rng``, vectorised so the 16M-word config 4 text is
produced in a few seconds. Nothing here is a copy of any benchmark corpus.

Shapes (BASELINE.json ``configs``):

0. ~190 KB English-like, ~35k tokens, lengths 1-14 (mean ~4.2, ~8% >= 8),
   English letter frequencies, ~10% capitalised first letter, ~6% of tokens
   with one attached punctuation byte, Zipf(s=1.1) over a 5k vocabulary.
1. same generator, ~1.38 MB, ~250k tokens, lengths 1-16, 20k vocabulary.
2. 1M words, lengths uniform 1-20, letters uniform over a-zA-Z, no
   punctuation.
3. 2M words, lengths uniform 3-12, letters uniform a-z, each length bucket
   non-increasing in corpus order (strictly descending is impossible at L=3:
   26**3 < 200k), ~6% attached punctuation.
4. 16M words, lengths Zipfian over 1-32 with P(L=5)=0.4, English letter
   frequencies, Zipf(s=1.0) rank within each length's slice of a 200k
   vocabulary.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BASE_SEED = 1407_6603

# Relative English letter frequencies a..z (percent, standard published table).
ENGLISH_FREQ = np.array(
    [8.167, 1.492, 2.782, 4.253, 12.702, 2.228, 2.015, 6.094, 6.966, 0.153,
     0.772, 4.025, 2.406, 6.749, 7.507, 1.929, 0.095, 5.987, 6.327, 9.056,
     2.758, 0.978, 2.360, 0.150, 1.974, 0.074]
)
ENGLISH_P = ENGLISH_FREQ / ENGLISH_FREQ.sum()
LOWER = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)
LETTERS52 = np.frombuffer(
    b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ", dtype=np.uint8
)
PUNCT = np.frombuffer(b".,;:!?\"'()-", dtype=np.uint8)

# Token-length laws for the English-like configs (index = length).
# 1-7 carry 92% of the mass, >=8 carries 8%; mean ~4.24.
_LEN14 = [0, .06, .18, .22, .16, .12, .09, .09, .030, .020, .013, .008, .005, .003, .001]
_LEN16 = [0, .06, .18, .22, .16, .12, .09, .09, .030, .020, .012, .008, .005, .003, .001,
          .0006, .0004]


@dataclass(frozen=True)
class ConfigSpec:
    index: int
    name: str
    words: int
    description: str


CONFIGS = {
    0: ConfigSpec(0, "english-190KB", 35_000, "English-like ~190 KB, Zipf(1.1) over 5k vocab"),
    1: ConfigSpec(1, "english-1.38MB", 250_000, "English-like ~1.38 MB, Zipf(1.1) over 20k vocab"),
    2: ConfigSpec(2, "uniform-1M", 1_000_000, "1M words, L~U[1,20], letters U[a-zA-Z]"),
    3: ConfigSpec(3, "descending-2M", 2_000_000, "2M words, L~U[3,12], buckets descending"),
    4: ConfigSpec(4, "skewed-16M", 16_000_000, "16M words, Zipf lengths 1-32, P(L=5)=0.4"),
}


def _zipf_sample(rng, n_items: int, s: float, size: int) -> np.ndarray:
    """Ranks 0..n_items-1 with P(r) proportional to 1/(r+1)**s (inverse CDF)."""
    w = 1.0 / np.arange(1, n_items + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return np.minimum(np.searchsorted(cdf, rng.random(size), side="right"), n_items - 1)


def _random_rows(rng, count: int, length: int, alphabet: np.ndarray, p=None) -> np.ndarray:
    idx = rng.choice(len(alphabet), size=(count, length), p=p)
    return alphabet[idx].astype(np.uint8)


def _assemble(lengths: np.ndarray, rows_by_len: dict, token_rows: np.ndarray,
              rng, punct_frac: float, cap_frac: float, newline_every: int) -> bytes:
    """Lay tokens out as text: [punct]word[punct] + one separator byte.

    ``token_rows[i]`` indexes into ``rows_by_len[lengths[i]]``. Attached
    punctuation only ever sits at a word's start or end, so it never splits
    a word (an apostrophe inside "don't" would).
    """
    n = len(lengths)
    pre = np.zeros(n, dtype=np.int64)
    post = np.zeros(n, dtype=np.int64)
    if punct_frac > 0:
        has = rng.random(n) < punct_frac
        at_start = rng.random(n) < 0.3
        pre[has & at_start] = 1
        post[has & ~at_start] = 1
    span = pre + lengths + post + 1
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(span, out=off[1:])
    out = np.empty(int(off[-1]), dtype=np.uint8)
    word_off = off[:-1] + pre
    for L, rows in rows_by_len.items():
        sel = np.nonzero(lengths == L)[0]
        if sel.size == 0:
            continue
        block = rows[token_rows[sel]]
        if cap_frac > 0:
            cap = rng.random(sel.size) < cap_frac
            block = block.copy()
            first = block[:, 0]
            lower = (first >= 97) & (first <= 122)
            block[cap & lower, 0] -= 32
        dst = word_off[sel][:, None] + np.arange(L)[None, :]
        out[dst] = block
    if punct_frac > 0:
        ps = np.nonzero(pre)[0]
        out[off[ps]] = PUNCT[rng.integers(0, len(PUNCT), ps.size)]
        qs = np.nonzero(post)[0]
        out[off[qs] + pre[qs] + lengths[qs]] = PUNCT[rng.integers(0, len(PUNCT), qs.size)]
    sep = np.full(n, 32, dtype=np.uint8)
    if newline_every > 0:
        sep[rng.random(n) < 1.0 / newline_every] = 10
    out[off[1:] - 1] = sep
    return out.tobytes()


def _english_like(rng, n_tokens: int, pmf: list, vocab: int, s: float) -> bytes:
    pmf = np.asarray(pmf, dtype=np.float64)
    pmf = pmf / pmf.sum()
    lengths = rng.choice(len(pmf), size=n_tokens, p=pmf).astype(np.int64)
    rows_by_len, token_rows = {}, np.zeros(n_tokens, dtype=np.int64)
    for L in range(1, len(pmf)):
        slice_n = max(1, int(round(vocab * pmf[L])))
        rows_by_len[L] = _random_rows(rng, slice_n, L, LOWER, ENGLISH_P)
        sel = lengths == L
        token_rows[sel] = _zipf_sample(rng, slice_n, s, int(sel.sum()))
    return _assemble(lengths, rows_by_len, token_rows, rng, punct_frac=0.06,
                     cap_frac=0.10, newline_every=12)


def _uniform_1m(rng) -> bytes:
    n = CONFIGS[2].words
    lengths = rng.integers(1, 21, size=n).astype(np.int64)
    rows_by_len, token_rows = {}, np.zeros(n, dtype=np.int64)
    for L in range(1, 21):
        sel = np.nonzero(lengths == L)[0]
        rows_by_len[L] = _random_rows(rng, sel.size, L, LETTERS52)
        token_rows[sel] = np.arange(sel.size)
    return _assemble(lengths, rows_by_len, token_rows, rng, 0.0, 0.0, 16)


def _descending_2m(rng) -> bytes:
    n = CONFIGS[3].words
    lengths = rng.integers(3, 13, size=n).astype(np.int64)
    rows_by_len, token_rows = {}, np.zeros(n, dtype=np.int64)
    for L in range(3, 13):
        sel = np.nonzero(lengths == L)[0]
        rows = _random_rows(rng, sel.size, L, LOWER)
        keys = rows.view(f"S{L}").ravel()
        order = np.argsort(keys, kind="stable")[::-1]  # non-increasing
        rows_by_len[L] = rows[order]
        token_rows[sel] = np.arange(sel.size)
    return _assemble(lengths, rows_by_len, token_rows, rng, 0.06, 0.0, 16)


def config4_length_pmf() -> np.ndarray:
    """P(L) for L=0..32: 0.4 at L=5, the rest Zipf(s=1) over the other lengths."""
    pmf = np.zeros(33)
    others = np.array([L for L in range(1, 33) if L != 5], dtype=np.float64)
    w = 1.0 / others
    pmf[others.astype(int)] = 0.6 * w / w.sum()
    pmf[5] = 0.4
    return pmf


def _skewed_16m(rng, n_tokens: int) -> bytes:
    pmf = config4_length_pmf()
    lengths = rng.choice(33, size=n_tokens, p=pmf).astype(np.int64)
    vocab = 200_000
    rows_by_len, token_rows = {}, np.zeros(n_tokens, dtype=np.int64)
    for L in range(1, 33):
        slice_n = max(1, int(round(vocab * pmf[L])))
        if L <= 4:
            slice_n = min(slice_n, 26 ** L)
        rows_by_len[L] = _random_rows(rng, slice_n, L, LOWER, ENGLISH_P)
        sel = lengths == L
        token_rows[sel] = _zipf_sample(rng, slice_n, 1.0, int(sel.sum()))
    return _assemble(lengths, rows_by_len, token_rows, rng, 0.0, 0.0, 16)


def generate(config: int, seed: int | None = None, words: int | None = None) -> bytes:
    """Text bytes of BASELINE.json config ``config`` (seed = 14076603 + config).

    ``words`` overrides the token count (used for bounded CPU samples of
    config 4 and for small test cases); it is honoured by configs 0, 1 and 4.
    """
    if config not in CONFIGS:
        raise ValueError(f"unknown config {config}")
    rng = np.random.default_rng(BASE_SEED + config if seed is None else seed)
    if config == 0:
        return _english_like(rng, words or CONFIGS[0].words, _LEN14, 5_000, 1.1)
    if config == 1:
        return _english_like(rng, words or CONFIGS[1].words, _LEN16, 20_000, 1.1)
    if config == 2:
        return _uniform_1m(rng)
    if config == 3:
        return _descending_2m(rng)
    return _skewed_16m(rng, words or CONFIGS[4].words)


def random_words(seed: int, count: int, max_len: int = 12, min_len: int = 1,
                 alphabet: bytes = b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789"
                 ) -> list[bytes]:
    """Seeded list of alphanumeric words (numpy stand-in for the tests' corpora)."""
    rng = np.random.default_rng(seed)
    alpha = np.frombuffer(alphabet, dtype=np.uint8)
    lens = rng.integers(min_len, max_len + 1, size=count)
    flat = alpha[rng.integers(0, len(alpha), size=int(lens.sum()))].tobytes()
    out, pos = [], 0
    for L in lens.tolist():
        out.append(flat[pos:pos + L])
        pos += L
    return out


ALNUM = b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789"
BUCKET_ORDERS = ("random", "sorted", "descending", "dups")


def bucket_case(seed: int, n: int, width: int, order: str, alpha: int = 62) -> np.ndarray:
    """One fixed-width bucket as a C-contiguous uint8 (n, width) array.

    ``order``: random rows; rows sorted ascending; rows non-increasing; or
    rows over a 2-letter alphabet (many exact duplicates). ``alpha`` limits
    the alphabet to the first ``alpha`` bytes of ``ALNUM``.
    """
    rng = np.random.default_rng(seed)
    letters = np.frombuffer(ALNUM[: (2 if order == "dups" else alpha)], dtype=np.uint8)
    rows = letters[rng.integers(0, len(letters), size=(n, width))].astype(np.uint8)
    if order in ("sorted", "descending") and n > 1:
        keys = rows.view(f"S{width}").ravel() if width else None
        idx = np.argsort(keys, kind="stable")
        if order == "descending":
            idx = idx[::-1]
        rows = rows[idx]
    return np.ascontiguousarray(rows)


def stats_case_list() -> list[dict]:
    """The bucket cases whose reference stats are frozen in tests/golden/."""
    cases = []
    sizes = [0, 1, 2, 3, 5, 8, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257,
             511, 512, 513, 1000, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097]
    widths = [1, 3, 5, 8, 9, 16, 17, 24, 32, 33, 40, 64]
    k = 0
    for n in sizes:
        for order in BUCKET_ORDERS:
            cases.append(dict(seed=1000 + k, n=n, width=widths[k % len(widths)],
                              order=order, alpha=62))
            k += 1
    rng = np.random.default_rng(77)
    for j in range(200):
        cases.append(dict(seed=5000 + j, n=int(rng.integers(0, 201)),
                          width=int(rng.integers(1, 41)),
                          order=BUCKET_ORDERS[int(rng.integers(0, 4))],
                          alpha=int(rng.choice([2, 3, 4, 26, 62]))))
    return cases


def prefix(text: bytes, n_words: int) -> bytes:
    """The leading part of a generated text holding its first ``n_words`` tokens.

    Generated texts end every token with exactly one separator byte (space or
    newline) and never put those bytes inside a token, so the cut falls right
    after the ``n_words``-th separator.
    """
    arr = np.frombuffer(text, dtype=np.uint8)
    seps = np.nonzero((arr == 32) | (arr == 10))[0]
    if n_words >= len(seps):
        return text
    return text[: int(seps[n_words - 1]) + 1]
