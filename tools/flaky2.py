"""Reuse of freed device memory: dirty a handle's buffers, free it, then run
the raw-byte payload sort on a fresh handle and compare."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_1407_6603_b200 import synth, _native
from paper_1407_6603_b200.pipeline import sort_text

def raw_case(seed):
    rng = np.random.default_rng(seed)
    words = []
    for L, n in ((1, 3000), (3, 9000), (4, 40000), (5, 30000), (8, 20000), (9, 25000),
                 (12, 20000), (17, 8000), (24, 6000), (31, 5000), (32, 4000), (40, 500)):
        rows = rng.integers(0, 256, size=(n, L), dtype=np.uint8)
        rows[::5] = rows[0]
        rows[::7, : min(L, 9)] = 0xFF
        rows[::11, : min(L, 8)] = 0x00
        words += [bytes(r) for r in rows]
    rng.shuffle(words)
    return words

bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    # dirty: a big payload sort on a throwaway handle
    d = _native.Handle(0)
    t = synth.generate(4, words=2_000_000, seed=it)
    d.ingest_words([bytes([255]) * (i % 40 + 1) for i in range(200000)])
    d.sort(False); d.emit_lines()
    d.close()
    words = raw_case(90 + it)
    h = _native.Handle(0)
    h.ingest_words(words)
    h.sort(False)
    got = h.emit_lines().tobytes()
    want = b"".join(w + b"\n" for w in sorted(words, key=lambda w: (len(w), w)))
    if got != want:
        bad += 1
        # locate the first differing line / length
        gl, wl = got.split(b"\n"), want.split(b"\n")
        for i, (a, b) in enumerate(zip(gl, wl)):
            if a != b:
                print("first diff at line", i, "len", len(b), a[:16].hex(), b[:16].hex())
                break
    h.close()
print("mismatches", bad)
