"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

usage: python tools/sanitize_driver.py CFG [WORDS]

Exercises every device path of the library once on a prefix of config CFG
(WORDS words, default: the whole config) and checks each result against the
oracle, so a sanitizer run is also a parity run:
  payload mode  sort_resident (unordered ingest, radix / sample sort, fused records)
  host e2e      ws_sort_text (H2D + kernels + D2H), ws_sort_texts (batch, 2 in flight)
  stats mode    ordered ingest + merge sort with inversion / K counts + SortStats
  tokens        ingest with corpus-order tokens (look-back ingest)
  rows          ws_sort_rows / ws_sort_blocks on raw-byte rows (both variants)
The WSORT_* environment knobs select the alternative paths (tools/sanitize.sh).
"""
import sys

sys.path.insert(0, '.')
import numpy as np

from oracle import oracle
from paper_1407_6603_b200 import _native, synth
from paper_1407_6603_b200._native import Handle
from paper_1407_6603_b200.pipeline import payload_bound

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
words = int(sys.argv[2]) if len(sys.argv) > 2 else 0
text = synth.generate(cfg)
if words:
    text = synth.prefix(text, words)
want, info = oracle.sort_text(text, mode="fast")

h = Handle(0)
h.ingest_text(text, unordered=True)
w = h.sort_resident(len(text))
dptr, dsize = h.output_device()
buf = _native.device_bytes(dptr, dsize)
assert buf == want, "resident payload differs"

src = np.frombuffer(text, dtype=np.uint8)
out = np.empty(payload_bound(len(text)), dtype=np.uint8)
n = h.sort_text(src, out)
assert out[:n].tobytes() == want, "sort_text payload differs"
outs = [np.empty(payload_bound(len(text)), dtype=np.uint8) for _ in range(3)]
sizes = h.sort_texts([src, src, src], outs, inflight=2)
assert all(o[:s].tobytes() == want for o, s in zip(outs, sizes)), "sort_texts payload differs"

hs = Handle(0)
hs.ingest_text(text)
hs.sort(True)
st = hs.bucket_stats(True)
lengths, counts, _ = hs.buckets()
for i, L in enumerate(lengths):
    c, s, p = info[L][3:6]
    assert tuple(int(x) for x in st[i]) == (c, s, p), (L, st[i], (c, s, p))
assert hs.emit_lines().tobytes() == want, "stats-mode payload differs"

ht = Handle(0)
ht.ingest_text(text, keep_tokens=True)
toks = ht.tokens()
assert len(toks) == sum(v[0] for v in info.values())

rows = synth.bucket_case(5, 1500, 11, "random")
for naive in (True, False):
    r = rows.copy()
    ref = rows.copy()
    st_ref = oracle.bubble_rows(ref, naive=naive)
    stats, _ = _native.sort_blocks([r], naive=naive)
    assert tuple(int(x) for x in stats[0]) == st_ref and np.array_equal(r, ref)
for x in (h, hs, ht):
    x.close()
print(f"sanitize driver ok: config {cfg}, {len(text)} bytes")
