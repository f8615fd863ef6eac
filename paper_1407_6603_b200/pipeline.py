"""Fused device pipeline: text bytes in, ``wordsort sort`` payload bytes out.

The reference's CLI path (cli.py:83-103) is tokenize -> build_flat ->
sort_all_parallel -> emit_sorted -> b"".join(word + b"\\n"). Here the whole
path after ``load_text`` is one C-ABI call (``ws_sort_text``): H2D of the
text, ingest kernels, segmented sort, emit kernel, D2H of the payload.
``TextSorter`` keeps a handle and page-locked staging buffers for repeated
calls (the bench's end-to-end leg); ``DeviceCorpus`` exposes the individual
phases for device-resident timing.
"""

from __future__ import annotations

import numpy as np

from ._native import Handle, PinnedBuffer
from ._runtime import default_handle, device_index


def payload_bound(n_text: int) -> int:
    """Upper bound of the payload size: every word is followed by a separator or EOF."""
    return n_text + 1


def sort_text(text: bytes) -> bytes:
    """Sorted payload of a corpus, byte-identical to ``wordsort sort`` (cli.py:97)."""
    text = bytes(text)
    h = default_handle()
    src = np.frombuffer(text, dtype=np.uint8) if text else np.zeros(0, np.uint8)
    out = np.empty(payload_bound(len(text)), dtype=np.uint8)
    n = h.sort_text(src, out)
    return out[:n].tobytes()


class TextSorter:
    """Repeated end-to-end sorts through pinned host buffers."""

    def __init__(self, max_text: int, device: int | None = None):
        self.handle = Handle(device_index() if device is None else device)
        self.text = PinnedBuffer(max_text)
        self.out = PinnedBuffer(payload_bound(max_text))

    def load(self, text: bytes) -> int:
        n = len(text)
        if n > self.text.nbytes:
            raise ValueError("text larger than the staging buffer")
        self.text.array[:n] = np.frombuffer(text, dtype=np.uint8)
        self._n = n
        return n

    def run(self) -> int:
        """Sort the loaded text; returns the payload size (payload in self.out)."""
        return self.handle.sort_text(self.text.array[: self._n], self.out.array)

    def payload(self, size: int) -> bytes:
        return self.out.array[:size].tobytes()

    def close(self) -> None:
        self.handle.close()
        self.text.close()
        self.out.close()


class BatchSorter:
    """Serving loop: many corpora through ``ws_sort_texts`` with ``inflight``
    of them in flight, so one corpus crosses PCIe host->device while earlier
    ones sort and come back (each output is byte-identical to ``sort_text``)."""

    def __init__(self, max_text: int, inflight: int = 3, device: int | None = None,
                 outputs: int | None = None):
        """`outputs`: distinct pinned output buffers, used round robin (default
        `inflight`); job i of a run writes buffer i % outputs."""
        self.handle = Handle(device_index() if device is None else device)
        self.inflight = inflight
        self.text = PinnedBuffer(max_text)
        nout = max(inflight, outputs or inflight)
        self.outs = [PinnedBuffer(payload_bound(max_text)) for _ in range(nout)]
        self._n = 0

    def load(self, text: bytes) -> int:
        n = len(text)
        if n > self.text.nbytes:
            raise ValueError("text larger than the staging buffer")
        self.text.array[:n] = np.frombuffer(text, dtype=np.uint8)
        self._n = n
        return n

    def run(self, count: int) -> list[int]:
        """Sort the loaded corpus `count` times as a batch; payload sizes."""
        texts = [self.text.array[: self._n]] * count
        outs = [self.outs[i % len(self.outs)].array for i in range(count)]
        return self.handle.sort_texts(texts, outs, self.inflight)

    def payload(self, slot: int, size: int) -> bytes:
        return self.outs[slot].array[:size].tobytes()

    def close(self) -> None:
        self.handle.close()
        self.text.close()
        for o in self.outs:
            o.close()


class DeviceCorpus:
    """Phase-by-phase access to the device pipeline for one corpus."""

    def __init__(self, handle: Handle | None = None):
        self.handle = handle or Handle(device_index())

    def ingest(self, text: bytes | np.ndarray, keep_tokens: bool = False) -> None:
        self.handle.ingest_text(text, keep_tokens=keep_tokens)

    def ingest_device(self, dev_ptr: int, n: int) -> None:
        self.handle.ingest_text(None, device_ptr=dev_ptr, n=n)

    def histogram(self) -> dict[int, int]:
        lengths, counts, _ = self.handle.buckets()
        return dict(zip(lengths, counts))

    def sort(self, want_stats: bool = False) -> None:
        self.handle.sort(want_stats)

    def stats(self, naive: bool) -> dict[int, tuple[int, int, int]]:
        lengths, _, _ = self.handle.buckets()
        st = self.handle.bucket_stats(naive)
        return {L: tuple(int(x) for x in s) for L, s in zip(lengths, st)}

    def payload(self) -> bytes:
        return self.handle.emit_lines().tobytes()
