"""Bucket sort engine (mirror of wordsort/engine.py) backed by the GPU.

The reference bubble-sorts each bucket with a triangular pass schedule
(engine.py:72-114): pass p compares the first n-1-p adjacent pairs, swaps on
strictly-greater, and the early-exit variant stops after the first pass with
no swap. Its results are (a) the stably sorted bucket and (b) SortStats.
Here every bucket is sorted on the device (csrc/sort.cu) and the stats come
from two device-side quantities through the closed form in
``ws_stats_closed_form`` (include/wsort.h):

* swaps       = number of strict inversions (each adjacent strict swap removes
                exactly one),
* naive       : comparisons = n(n-1)/2, passes = n-1,
* early-exit  : passes P = min(K+1, n-1) with K = max_i(i - s(i)) (s = stable
                sorted position), comparisons = P(n-1) - P(P-1)/2,

so they are identical to the reference's for every input and both layouts.
The reference's worker pool (engine.py:140-201) becomes one segmented launch
over all buckets; ``threads`` and ``schedule`` are validated and accepted but
cannot change the result, exactly as the reference guarantees
(test_parallel.py:34-61).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from ._native import sort_blocks
from .store import BucketSet, FlatBucketMatrix, LayoutKind, Store


class SortVariant(enum.Enum):
    NAIVE = "naive"
    EARLY_EXIT = "early-exit"


class SchedulePolicy(enum.Enum):
    STATIC_BLOCK = "static"
    STATIC_CYCLIC = "cyclic"
    DYNAMIC = "dynamic"


@dataclass
class SortStats:
    comparisons: int = 0
    swaps: int = 0
    passes: int = 0

    def __add__(self, other: "SortStats") -> "SortStats":
        return SortStats(
            self.comparisons + other.comparisons,
            self.swaps + other.swaps,
            self.passes + other.passes,
        )


@dataclass
class SortConfig:
    layout: LayoutKind
    variant: SortVariant = SortVariant.NAIVE
    threads: int = 1
    schedule: SchedulePolicy = SchedulePolicy.STATIC_BLOCK

    def __post_init__(self):
        if self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")


def compare_words(a: bytes, b: bytes) -> int:
    """Raw byte-wise comparison of two equal-length words: -1, 0 or 1 (engine.py:62-69)."""
    assert len(a) == len(b), "bucket-internal comparison requires equal lengths"
    if a < b:
        return -1
    if a > b:
        return 1
    return 0


def _ragged_rows(bucket: list[bytes], length: int) -> np.ndarray:
    if any(len(w) != length for w in bucket):
        raise ValueError(f"bucket {length} holds a word of another length")
    raw = b"".join(bucket)
    return np.frombuffer(raw, dtype=np.uint8).reshape(len(bucket), length).copy()


def _sort_stores(store: Store, lengths: list[int], naive: bool) -> list[SortStats]:
    """Sort the given buckets of one store in one batched device call."""
    if isinstance(store, BucketSet):
        todo = [L for L in lengths if len(store.buckets.get(L, ())) >= 2]
        rows = [_ragged_rows(store.buckets[L], L) for L in todo]
        stats, perms = sort_blocks(rows, naive, want_perms=True)
        for L, perm in zip(todo, perms):
            bucket = store.buckets[L]
            # reorder the caller's objects in place (tags on bytes subclasses survive)
            bucket[:] = [bucket[i] for i in perm.tolist()]
    else:
        todo = [L for L in lengths if store.count_for_length(L) >= 2]
        blocks = [store.blocks[L] for L in todo]
        stats, _ = sort_blocks(blocks, naive)
    by_len = {L: SortStats(*map(int, s)) for L, s in zip(todo, stats)}
    return [by_len.get(L, SortStats()) for L in lengths]


def bubble_sort_bucket(store: Store, length: int, variant: SortVariant) -> SortStats:
    """Sort one bucket in place, returning its comparison/swap/pass counts."""
    return _sort_stores(store, [length], variant is SortVariant.NAIVE)[0]


def sort_all_sequential(store: Store, variant: SortVariant) -> SortStats:
    """Sort every bucket (ascending length order of the reference, engine.py:132-137)."""
    total = SortStats()
    for s in _sort_stores(store, store.lengths(), variant is SortVariant.NAIVE):
        total += s
    return total


def sort_all_parallel(store: Store, config: SortConfig) -> SortStats:
    """All buckets in one segmented device launch; same result for every config.

    engine.py:140-201 spreads whole buckets over min(threads, #buckets) host
    threads; on the GPU every bucket (and every tile of a large bucket) is a
    work item of the same launch, so the schedule has nothing left to decide.
    """
    if config.threads < 1:
        raise ValueError(f"threads must be >= 1, got {config.threads}")
    return sort_all_sequential(store, config.variant)
