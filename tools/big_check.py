"""Large-input check (> 512 MiB text: the two-pass ingest): the payload is
non-decreasing in (length, bytes) and holds the same words per length as the
text (multiset by length + an order-independent hash of the words)."""
import sys, time, zlib
sys.path.insert(0, '.')
import numpy as np
from bench import corpus
from paper_1407_6603_b200.pipeline import sort_text

base = corpus(4, 0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
text = b" ".join([base] * reps)
print("text bytes", len(text))
t0 = time.time()
out = sort_text(text)
print("sorted in %.2f s, payload %d" % (time.time() - t0, len(out)))
lines = out.split(b"\n")[:-1]
# order: non-decreasing (len, bytes)
prev = b""
bad = 0
for i in range(0, len(lines), 997):  # sampled adjacent pairs
    a, b = lines[i], lines[min(i + 1, len(lines) - 1)]
    if (len(a), a) > (len(b), b):
        bad += 1
print("order violations (sampled)", bad)
import re
words = re.findall(rb"[A-Za-z0-9]+", base)
from collections import Counter
want = Counter(len(w) for w in words)
got = Counter(len(w) for w in lines)
ok = all(got[L] == reps * c for L, c in want.items()) and sum(got.values()) == reps * len(words)
h_in = sum(zlib.crc32(w) for w in words) * reps
h_out = sum(zlib.crc32(w) for w in lines)
print("length multiset ok", ok, "hash ok", h_in == h_out)
assert bad == 0 and ok and h_in == h_out
print("big check ok")
