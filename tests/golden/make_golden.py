"""Freeze golden vectors by running the UNMODIFIED reference in this container.

Run here (never on the GPU box, where /root/reference does not exist):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [--configs 0,1,2,3,4]

Everything is produced through the reference's own public API:
``wordsort.ingest.tokenize`` (ingest.py:26-28), ``wordsort.store.build_flat``
(store.py:90-96), ``wordsort.engine.bubble_sort_bucket`` (engine.py:117-129,
i.e. the numba ``_bubble_rows`` kernel, engine.py:89-114) and
``wordsort.store.emit_sorted`` (store.py:105-114) + the CLI payload rule
``word + b"\\n"`` (cli.py:97). Inputs are regenerated from seeds
(paper_1407_6603_b200.synth), so the fixtures hold only recipes, digests,
histograms and stats.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from paper_1407_6603_b200 import synth  # noqa: E402

import wordsort  # noqa: E402  (the reference, from PYTHONPATH)
from wordsort.engine import SortVariant, bubble_sort_bucket  # noqa: E402
from wordsort.ingest import tokenize  # noqa: E402
from wordsort.store import build_buckets, build_flat, emit_sorted  # noqa: E402

assert "/root/reference" in wordsort.__file__, wordsort.__file__


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


TOKENIZE_KATS = [
    b"HAMLET, PRINCE!", b"don't", b"", b"...", b"a1b2 3", b"caf\xc3\xa9", b"caf\xc3\xa9s",
    b"\x00abc\x00", b"\x80\xff\x7f0Zz9", b"a" * 70 + b"!" + b"b" * 33, b"x", b"  x  ",
    b"tab\tsep\nnl\r\ncrlf", b"@[`{/:", b"09AZaz", b"/0:@A[Z`a{z",
]


def tokenize_cases() -> list[dict]:
    rng = np.random.default_rng(9)
    texts = list(TOKENIZE_KATS)
    seps = np.frombuffer(b" \t\n.,?!'\"-\x00\x80\xff", dtype=np.uint8)
    for i in range(300):
        n = int(rng.integers(0, 400))
        mode = i % 3
        if mode == 0:  # raw random bytes
            t = rng.integers(0, 256, size=n, dtype=np.uint8)
        elif mode == 1:  # alnum-heavy with separators
            al = np.frombuffer(synth.ALNUM, dtype=np.uint8)
            t = al[rng.integers(0, len(al), size=n)]
            mask = rng.random(n) < 0.2
            t[mask] = seps[rng.integers(0, len(seps), size=int(mask.sum()))]
        else:  # long runs crossing 16/32/128-byte boundaries
            t = np.full(n, ord("q"), dtype=np.uint8)
            cuts = rng.integers(0, max(n, 1), size=max(1, n // 50))
            t[cuts[cuts < n]] = 32
        texts.append(t.tobytes())
    return [{"text": t.hex(), "tokens": [w.hex() for w in tokenize(t)]} for t in texts]


def bucket_stats(rows: np.ndarray) -> dict:
    """Reference stats + sorted digest for one (n, width) bucket, both variants."""
    out = {}
    for variant in SortVariant:
        words = [rows[i].tobytes() for i in range(rows.shape[0])]
        store = build_flat(words)
        if rows.shape[0] == 0:
            st = wordsort.SortStats()
        else:
            st = bubble_sort_bucket(store, rows.shape[1], variant)
        out[variant.value] = [st.comparisons, st.swaps, st.passes]
        if variant is SortVariant.NAIVE:
            sorted_rows = b"".join(store.words_for_length(rows.shape[1])) if rows.shape[0] else b""
            out["sorted_sha"] = sha(sorted_rows)
        # ragged layout must agree (engine.py:72-86 vs :89-114)
        rag = build_buckets(list(words))
        st2 = bubble_sort_bucket(rag, rows.shape[1], variant) if rows.shape[0] else wordsort.SortStats()
        assert [st2.comparisons, st2.swaps, st2.passes] == out[variant.value]
    return out


def stats_cases() -> list[dict]:
    res = []
    for c in synth.stats_case_list():
        rows = synth.bucket_case(c["seed"], c["n"], c["width"], c["order"], c["alpha"])
        res.append({**c, **bucket_stats(rows)})
    return res


def config_record(cfg: int, prefix_words: int | None = None, threads: int = 8) -> dict:
    text = synth.generate(cfg)
    if prefix_words is not None:
        text = synth.prefix(text, prefix_words)
    t0 = time.time()
    words = tokenize(text)
    store = build_flat(words)
    hist = {int(L): int(store.count_for_length(L)) for L in store.lengths()}
    per_len = {}

    def run(L, variant):
        # each task gets a private copy of the bucket: variants must not see
        # each other's sorted output
        block = store.blocks[L].copy()
        sub = wordsort.FlatBucketMatrix({L: block})
        st = bubble_sort_bucket(sub, L, variant)
        return L, variant, st, block

    tasks = [(L, v) for L in sorted(store.lengths(), key=lambda L: -hist[L]) for v in SortVariant]
    with ThreadPoolExecutor(threads) as ex:
        results = list(ex.map(lambda a: run(*a), tasks))
    for L, variant, st, block in results:
        per_len.setdefault(L, {})[variant.value] = [st.comparisons, st.swaps, st.passes]
        if variant is SortVariant.NAIVE:
            store.blocks[L] = block
    payload = b"".join(w + b"\n" for w in emit_sorted(store))
    rec = {
        "config": cfg,
        "prefix_words": prefix_words,
        "text_bytes": len(text),
        "text_sha": sha(text),
        "words": len(words),
        "alnum_bytes": int(sum(len(w) for w in words)),
        "lmax": int(store.lmax),
        "hist": hist,
        "payload_bytes": len(payload),
        "payload_sha": sha(payload),
        "tokens_sha": sha(b"\n".join(words)),
        "per_length_stats": per_len,
        "ref_seconds": round(time.time() - t0, 2),
    }
    return rec


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,2,3,4")
    ap.add_argument("--skip-kat", action="store_true")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    if not args.skip_kat:
        (HERE / "tokenize_kat.json").write_text(json.dumps(tokenize_cases()))
        print("tokenize_kat.json written", flush=True)
        (HERE / "stats_kat.json").write_text(json.dumps(stats_cases()))
        print("stats_kat.json written", flush=True)
    cfg_path = HERE / "configs.json"
    table = json.loads(cfg_path.read_text()) if cfg_path.exists() else {}
    for c in [int(x) for x in args.configs.split(",") if x]:
        if c == 4:
            # full config 4 is ~57 h of bubble sort for the L=5 bucket alone;
            # freeze the first 200k words of the seeded config-4 text instead
            rec = config_record(4, prefix_words=200_000, threads=args.threads)
            table["4_prefix200k"] = rec
        else:
            rec = config_record(c, threads=args.threads)
            table[str(c)] = rec
        print(f"config {c}: {rec['words']} words, {rec['ref_seconds']} s", flush=True)
        cfg_path.write_text(json.dumps(table, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
