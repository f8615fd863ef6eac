"""ctypes binding of libwsort_b200.so (the C ABI declared in include/wsort.h).

This is the only way the package reaches the GPU. There is no CPU fallback:
if the library is missing, or no sm_100a device is visible, every compute
call raises. Error codes map to the exceptions the reference raises for the
same situations (ValueError for bad arguments, RuntimeError for device
failures, MemoryError for allocation failures).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_NAME = "libwsort_b200.so"
LIB_PATH = Path(os.environ.get("WSORT_LIB") or Path(__file__).resolve().parent / LIB_NAME)

WS_OK = 0
WS_ERR_ARG = -1
WS_ERR_CUDA = -2
WS_ERR_OOM = -3
WS_ERR_STATE = -4
WS_INGEST_KEEP_TOKENS = 1
WS_INGEST_DEVICE_PTR = 2
WS_INGEST_RESIDENT = 4
WS_INGEST_UNORDERED = 8

# Every symbol include/wsort.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ws_version", "ws_last_error", "ws_device_count", "ws_create", "ws_destroy",
    "ws_ingest_text", "ws_ingest_words", "ws_ingest_blocks", "ws_buckets", "ws_tokens",
    "ws_sort", "ws_bucket_stats", "ws_permutation", "ws_emit_lines", "ws_emit_rows",
    "ws_sort_text", "ws_sort_rows", "ws_sort_blocks", "ws_stats_closed_form",
    "ws_set_profiling", "ws_profile", "ws_profile_reset", "ws_launch_count", "ws_stream",
    "ws_host_alloc", "ws_host_free", "ws_sort_resident", "ws_output_device", "ws_sort_texts",
    "ws_debug_checks", "ws_checked_build", "ws_counted_classes",
)


class WsPhase(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 32),
        ("launches", ctypes.c_int32),
        ("kind", ctypes.c_int32),
        ("ms", ctypes.c_double),
        ("bytes", ctypes.c_double),
        ("start_ms", ctypes.c_double),
    ]


_lib = None
_lib_lock = threading.Lock()

c_void_p = ctypes.c_void_p
c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u32p = ctypes.POINTER(ctypes.c_uint32)


def _declare(lib) -> None:
    I, V = ctypes.c_int, c_void_p
    sigs = {
        "ws_version": (I, []),
        "ws_last_error": (ctypes.c_char_p, []),
        "ws_device_count": (I, [c_i32p]),
        "ws_create": (I, [ctypes.POINTER(V), ctypes.c_int32]),
        "ws_destroy": (None, [V]),
        "ws_ingest_text": (I, [V, V, ctypes.c_uint64, ctypes.c_int32]),
        "ws_ingest_words": (I, [V, V, V, ctypes.c_uint64]),
        "ws_ingest_blocks": (I, [V, ctypes.c_int32, V, V, V]),
        "ws_buckets": (I, [V, V, V, ctypes.c_int32, c_i32p, c_u64p]),
        "ws_tokens": (I, [V, V, ctypes.c_uint64, c_u64p]),
        "ws_sort": (I, [V, ctypes.c_int32]),
        "ws_bucket_stats": (I, [V, ctypes.c_int32, V, ctypes.c_int32]),
        "ws_permutation": (I, [V, ctypes.c_int32, V, ctypes.c_uint64]),
        "ws_emit_lines": (I, [V, V, ctypes.c_uint64, c_u64p]),
        "ws_emit_rows": (I, [V, V, ctypes.c_uint64, c_u64p]),
        "ws_sort_text": (I, [V, V, ctypes.c_uint64, V, ctypes.c_uint64, c_u64p]),
        "ws_sort_texts": (I, [V, ctypes.c_int32, V, V, V, V, V, ctypes.c_int32]),
        "ws_sort_rows": (I, [V, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, V]),
        "ws_sort_blocks": (I, [ctypes.c_int32, V, V, V, ctypes.c_int32, V, V]),
        "ws_stats_closed_form": (I, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int32, V]),
        "ws_set_profiling": (I, [V, ctypes.c_int32]),
        "ws_profile": (I, [V, ctypes.POINTER(WsPhase), ctypes.c_int32, c_i32p]),
        "ws_profile_reset": (I, [V]),
        "ws_launch_count": (I, [V, c_u64p]),
        "ws_counted_classes": (I, [V, c_i32p]),
        "ws_stream": (I, [V, ctypes.POINTER(V)]),
        "ws_host_alloc": (I, [ctypes.c_uint64, ctypes.POINTER(V)]),
        "ws_host_free": (I, [V]),
        "ws_sort_resident": (I, [V, ctypes.c_uint64, c_u64p]),
        "ws_output_device": (I, [V, ctypes.POINTER(V), c_u64p]),
        "ws_debug_checks": (I, [c_u64p, c_i32p, c_i32p]),
        "ws_checked_build": (I, []),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load_library(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes library; raise loudly if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`); "
                "there is no CPU fallback"
            )
        lib = ctypes.CDLL(str(p))
        _declare(lib)
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    return load_library().ws_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == WS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == WS_ERR_ARG:
        raise ValueError(msg)
    if rc == WS_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(arr) -> int:
    """Address of a numpy array's (or bytes-like) first byte."""
    if isinstance(arr, np.ndarray):
        return arr.ctypes.data
    raise TypeError(type(arr))


class _DeviceSpan:
    """A raw device byte range exposed through __cuda_array_interface__."""

    def __init__(self, address: int, size: int):
        self.__cuda_array_interface__ = {"shape": (size,), "typestr": "|u1",
                                         "data": (address, False), "version": 3}


def device_bytes(address: int, size: int) -> bytes:
    """Copy `size` bytes at device address `address` (e.g. ws_output_device)
    back to the host; the caller's work on the library stream must be done."""
    if size == 0:
        return b""
    import torch

    t = torch.as_tensor(_DeviceSpan(address, size), device="cuda")
    return t.cpu().numpy().tobytes()


CHECK_UNITS = ("ingest", "sort", "radix", "emit")


def debug_checks() -> tuple[int, str]:
    """(failed bounds checks since the last call, 'unit:line' of the first) of
    a checked build (WS_CHECKED=1); (0, '') otherwise. Synchronizes the device."""
    f = ctypes.c_uint64(0)
    u = ctypes.c_int32(-1)
    ln = ctypes.c_int32(0)
    check(load_library().ws_debug_checks(ctypes.byref(f), ctypes.byref(u), ctypes.byref(ln)),
          "ws_debug_checks")
    where = f"{CHECK_UNITS[u.value]}.cu:{ln.value}" if f.value and u.value >= 0 else ""
    return int(f.value), where


def checked_build() -> bool:
    return bool(load_library().ws_checked_build())


def device_count() -> int:
    n = ctypes.c_int32(0)
    check(load_library().ws_device_count(ctypes.byref(n)))
    return int(n.value)


class PinnedBuffer:
    """Page-locked host bytes (cudaMallocHost) exposed as a uint8 numpy array."""

    def __init__(self, nbytes: int):
        lib = load_library()
        p = c_void_p()
        check(lib.ws_host_alloc(max(int(nbytes), 1), ctypes.byref(p)), "ws_host_alloc")
        self._p = p
        self.nbytes = int(nbytes)
        buf = (ctypes.c_uint8 * max(self.nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=np.uint8, count=self.nbytes)

    @property
    def address(self) -> int:
        return int(self._p.value)

    def close(self) -> None:
        if self._p is not None and self._p.value:
            self.array = None
            load_library().ws_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Handle:
    """One device context: stream + device buffers (include/wsort.h ws_handle)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = c_void_p()
        check(self.lib.ws_create(ctypes.byref(h), int(device)), "ws_create")
        self._h = h

    @property
    def h(self):
        if self._h is None:
            raise RuntimeError("handle closed")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            self.lib.ws_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- ingest -----------------------------------------------------------
    def ingest_text(self, text, keep_tokens: bool = False, device_ptr: int | None = None,
                    n: int | None = None, unordered: bool = False) -> None:
        """`unordered`: payload-only ingest (WS_INGEST_UNORDERED) - words of
        one length may sit in any order before the sort; sort(stats=True)
        and permutation() then raise."""
        flags = (WS_INGEST_KEEP_TOKENS if keep_tokens else 0) | (WS_INGEST_UNORDERED if unordered else 0)
        if device_ptr is not None:
            check(self.lib.ws_ingest_text(self.h, c_void_p(device_ptr), int(n),
                                          flags | WS_INGEST_DEVICE_PTR), "ws_ingest_text")
            return
        if isinstance(text, np.ndarray):
            data, size = ptr(text), text.nbytes
        else:
            text = bytes(text)
            data, size = ctypes.cast(ctypes.c_char_p(text), c_void_p).value, len(text)
            self._keep = text  # keep the bytes alive across the call
        check(self.lib.ws_ingest_text(self.h, c_void_p(data), size, flags), "ws_ingest_text")

    def ingest_words(self, words: list[bytes]) -> None:
        lens = np.fromiter((len(w) for w in words), dtype=np.uint32, count=len(words))
        concat = b"".join(words)
        buf = np.frombuffer(concat, dtype=np.uint8) if concat else np.zeros(1, np.uint8)
        check(self.lib.ws_ingest_words(self.h, c_void_p(ptr(buf)), c_void_p(ptr(lens)),
                                       len(words)), "ws_ingest_words")

    def buckets(self) -> tuple[list[int], list[int], int]:
        n = ctypes.c_int32(0)
        words = ctypes.c_uint64(0)
        check(self.lib.ws_buckets(self.h, None, None, 0, ctypes.byref(n), ctypes.byref(words)),
              "ws_buckets")
        L = np.zeros(max(n.value, 1), dtype=np.int64)
        C = np.zeros(max(n.value, 1), dtype=np.int64)
        check(self.lib.ws_buckets(self.h, c_void_p(ptr(L)), c_void_p(ptr(C)), n.value,
                                  ctypes.byref(n), ctypes.byref(words)), "ws_buckets")
        return L[: n.value].tolist(), C[: n.value].tolist(), int(words.value)

    def tokens(self) -> np.ndarray:
        _, _, words = self.buckets()
        out = np.zeros(max(words, 1) * 2, dtype=np.uint32)
        nw = ctypes.c_uint64(0)
        check(self.lib.ws_tokens(self.h, c_void_p(ptr(out)), words, ctypes.byref(nw)),
              "ws_tokens")
        return out[: 2 * words].reshape(words, 2)

    # -- sort ---------------------------------------------------------------
    def sort(self, want_stats: bool = False) -> None:
        check(self.lib.ws_sort(self.h, 1 if want_stats else 0), "ws_sort")

    def bucket_stats(self, naive: bool) -> np.ndarray:
        L, _, _ = self.buckets()
        out = np.zeros((max(len(L), 1), 3), dtype=np.int64)
        check(self.lib.ws_bucket_stats(self.h, 1 if naive else 0, c_void_p(ptr(out)), len(L)),
              "ws_bucket_stats")
        return out[: len(L)]

    def permutation(self, bucket: int, count: int) -> np.ndarray:
        out = np.zeros(max(count, 1), dtype=np.uint32)
        check(self.lib.ws_permutation(self.h, int(bucket), c_void_p(ptr(out)), count),
              "ws_permutation")
        return out[:count]

    # -- emit -----------------------------------------------------------------
    def _emit(self, fn, out: np.ndarray | None) -> np.ndarray:
        size = ctypes.c_uint64(0)
        check(fn(self.h, None, 0, ctypes.byref(size)), fn.__name__)
        if out is None:
            out = np.empty(max(size.value, 1), dtype=np.uint8)
        if size.value:
            check(fn(self.h, c_void_p(ptr(out)), out.nbytes, ctypes.byref(size)), fn.__name__)
        return out[: size.value]

    def emit_lines(self, out: np.ndarray | None = None) -> np.ndarray:
        return self._emit(self.lib.ws_emit_lines, out)

    def emit_rows(self, out: np.ndarray | None = None) -> np.ndarray:
        return self._emit(self.lib.ws_emit_rows, out)

    def sort_text(self, text: np.ndarray, out: np.ndarray) -> int:
        """Fused ingest + sort + emit: host text in, host payload out (sizes in bytes)."""
        written = ctypes.c_uint64(0)
        check(self.lib.ws_sort_text(self.h, c_void_p(ptr(text)), text.nbytes,
                                    c_void_p(ptr(out)), out.nbytes, ctypes.byref(written)),
              "ws_sort_text")
        return int(written.value)

    def sort_texts(self, texts: list, outs: list, inflight: int = 0) -> list[int]:
        """Batch of corpora, up to `inflight` in flight (ws_sort_texts): texts[i]
        and outs[i] are uint8 numpy arrays (pinned for full PCIe speed);
        returns the payload sizes."""
        k = len(texts)
        if len(outs) != k:
            raise ValueError("texts and outs differ in length")
        tp = (ctypes.c_void_p * max(k, 1))(*[ptr(t) for t in texts])
        op = (ctypes.c_void_p * max(k, 1))(*[ptr(o) for o in outs])
        sz = np.array([t.nbytes for t in texts] or [0], dtype=np.uint64)
        cp = np.array([o.nbytes for o in outs] or [0], dtype=np.uint64)
        wr = np.zeros(max(k, 1), dtype=np.uint64)
        check(self.lib.ws_sort_texts(self.h, k, ctypes.cast(tp, c_void_p), c_void_p(ptr(sz)),
                                     ctypes.cast(op, c_void_p), c_void_p(ptr(cp)),
                                     c_void_p(ptr(wr)), int(inflight)), "ws_sort_texts")
        return [int(x) for x in wr[:k]]

    def sort_resident(self, n: int) -> int:
        """Ingest + sort + emit of the text already on the device; payload stays in HBM."""
        written = ctypes.c_uint64(0)
        check(self.lib.ws_sort_resident(self.h, int(n), ctypes.byref(written)), "ws_sort_resident")
        return int(written.value)

    def output_device(self) -> tuple[int, int]:
        p = c_void_p()
        size = ctypes.c_uint64(0)
        check(self.lib.ws_output_device(self.h, ctypes.byref(p), ctypes.byref(size)))
        return int(p.value or 0), int(size.value)

    # -- profiling --------------------------------------------------------------
    def set_profiling(self, on: bool | int) -> None:
        """True / 1: CUDA events around every phase; 2: also serialise the
        kernels on the main stream (one launch per event pair)."""
        check(self.lib.ws_set_profiling(self.h, int(on)))

    def profile(self, reset: bool = True) -> list[dict]:
        n = ctypes.c_int32(0)
        check(self.lib.ws_profile(self.h, None, 0, ctypes.byref(n)))
        arr = (WsPhase * max(n.value, 1))()
        check(self.lib.ws_profile(self.h, arr, n.value, ctypes.byref(n)))
        res = [dict(name=arr[i].name.decode(), launches=arr[i].launches, kind=arr[i].kind,
                    ms=arr[i].ms, bytes=arr[i].bytes, start_ms=arr[i].start_ms)
               for i in range(n.value)]
        if reset:
            check(self.lib.ws_profile_reset(self.h))
        return res

    def launch_count(self) -> int:
        v = ctypes.c_uint64(0)
        check(self.lib.ws_launch_count(self.h, ctypes.byref(v)))
        return int(v.value)

    def counted_classes(self) -> int:
        """Bit c set: the last fused sort counted lane class c's distinct words
        instead of sorting every occurrence (same payload bytes)."""
        m = ctypes.c_int32(0)
        check(self.lib.ws_counted_classes(self.h, ctypes.byref(m)))
        return int(m.value)

    def stream(self) -> int:
        s = c_void_p()
        check(self.lib.ws_stream(self.h, ctypes.byref(s)))
        return int(s.value or 0)


def sort_blocks(blocks: list[np.ndarray], naive: bool, want_perms: bool = False):
    """In-place batched _bubble_rows over C-contiguous uint8 (n, w) arrays.

    Returns (stats (k, 3) int64, perms list or None).
    """
    lib = load_library()
    k = len(blocks)
    for b in blocks:
        if b.dtype != np.uint8 or b.ndim != 2 or not b.flags["C_CONTIGUOUS"]:
            raise ValueError("blocks must be C-contiguous uint8 (n, width) arrays")
        if not b.flags["WRITEABLE"]:
            raise ValueError("blocks must be writeable (sorted in place)")
    rows = (c_void_p * max(k, 1))(*[b.ctypes.data for b in blocks])
    counts = np.array([b.shape[0] for b in blocks] or [0], dtype=np.int64)
    widths = np.array([b.shape[1] for b in blocks] or [0], dtype=np.int32)
    stats = np.zeros((max(k, 1), 3), dtype=np.int64)
    perms = None
    perm_ptrs = None
    if want_perms:
        perms = [np.zeros(max(b.shape[0], 1), dtype=np.uint32) for b in blocks]
        perm_ptrs = (c_void_p * max(k, 1))(*[p.ctypes.data for p in perms])
    check(lib.ws_sort_blocks(k, rows, c_void_p(ptr(counts)), c_void_p(ptr(widths)),
                             1 if naive else 0, c_void_p(ptr(stats)),
                             perm_ptrs if want_perms else None), "ws_sort_blocks")
    if perms is not None:
        perms = [p[: b.shape[0]] for p, b in zip(perms, blocks)]
    return stats[:k], perms


def stats_closed_form(n: int, inversions: int, kmax: int, naive: bool) -> tuple[int, int, int]:
    out = np.zeros(3, dtype=np.int64)
    check(load_library().ws_stats_closed_form(int(n), int(inversions), int(kmax),
                                              1 if naive else 0, c_void_p(ptr(out))))
    return int(out[0]), int(out[1]), int(out[2])
