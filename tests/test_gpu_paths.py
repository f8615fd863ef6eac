"""Every alternative device path selected by a diagnostic knob produces the
same payload and stats as the default path (each knob is read once per
process, so every case runs in a fresh interpreter)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
from oracle import oracle
from paper_1407_6603_b200 import synth
from paper_1407_6603_b200.pipeline import DeviceCorpus, sort_text
text = synth.generate(4, words={words}, seed=5) + b" " + b"x" * 70 + b" " + b"Zq" * 20
want, info = oracle.sort_text(text, mode="fast")
assert sort_text(text) == want, "payload"
dc = DeviceCorpus()
dc.ingest(text)
dc.sort(want_stats=True)
naive = dc.stats(naive=True)
for L, (n, inv, K, c, s, p) in info.items():
    assert naive[L] == (c, s, p), L
assert dc.payload() == want, "stats-mode payload"
print("ok")
"""


@pytest.mark.parametrize("knob", [
    "WSORT_NO_RADIX",         # class 0 by tile + merge path in payload mode
    "WSORT_NO_SAMPLE",        # multi-lane classes by tile + merge path in payload mode
    "WSORT_RADIX_RTS",        # class-0 radix by upsweep + scan + downsweep (no look-back)
    "WSORT_NO_FUSED_PAYLOAD", # payload by the emit kernels after the last radix pass / slot sorts
    "WSORT_NO_FUSED_SLOTS",   # multi-lane payload by the emit kernels after the slot sorts
    "WSORT_NO_JOINT",         # 1-2 character buckets by radix passes instead of whole-key counts
    "WSORT_NO_EARLY_HIST",    # class-0 histogram launched after the host plan, not by the ingest
    "WSORT_NO_EARLY_SPLIT",   # multi-lane split launches after the host plan, not by the ingest
    "WSORT_NO_EARLY_COUNT",   # multi-lane count passes after the host plan (split still early)
    "WSORT_LOOKBACK",         # ordered ingest by the decoupled look-back
    "WSORT_TWO_PASS",         # count + scan + scatter ingest
    "WSORT_NO_CHUNKED_H2D",   # one host->device copy before the ingest
    "WSORT_SERIAL",           # every kernel on the main stream
    "WSORT_D2H_PER_CLASS",    # one emit + copy per lane class
    "WSORT_INGEST=reserve",   # payload ingest by reserve_ingest_kernel (round-1 default)
    "WSORT_INGEST=6",         # payload ingest by ingest6_kernel (word-parallel, measured slower)
    # A/B knobs used in the measurements (profiles/r01_ab_*.txt)
    "WSORT_CLASS_ORDER=3,2,1,0,4",
    "WSORT_CLASS_PRIO=0,-5,-5,-5,0",
    "WSORT_FUSED_SLOT_CLASSES=2",
    "CUDA_DEVICE_MAX_CONNECTIONS=32",
])
def test_diagnostic_paths_agree(knob):
    """The sort paths themselves: distinct-word counting off (a text that
    repeats its vocabulary would otherwise never reach them in payload mode)."""
    words = 2_600_000 if knob == "WSORT_NO_CHUNKED_H2D" else 300_000  # > 16 MiB for the H2D knob
    name, _, value = knob.partition("=")
    env = dict(os.environ, **{name: value or "1"}, WSORT_NO_DEDUPE="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), words=words)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("knob", [
    "WSORT_NO_DEDUPE",        # every class sorted (no distinct-word counting)
    "WSORT_DEDUPE_MIN=0",     # counting from the smallest text that skips the small-corpus kernel
    "WSORT_NO_RADIX", "WSORT_NO_SAMPLE", "WSORT_NO_EARLY_HIST", "WSORT_NO_EARLY_SPLIT",
    "WSORT_NO_EARLY_COUNT", "WSORT_NO_CHUNKED_H2D", "WSORT_SERIAL", "WSORT_NO_JOINT",
    "WSORT_INGEST=reserve",
])
def test_diagnostic_paths_agree_with_counting(knob):
    """The same knobs with distinct-word counting on (the default): the
    distinct keys go through the knob's sort path."""
    words = 2_600_000 if knob == "WSORT_NO_CHUNKED_H2D" else 300_000
    name, _, value = knob.partition("=")
    env = dict(os.environ, **{name: value or "1"})
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), words=words)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
