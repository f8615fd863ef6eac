"""Repro loop for test_fused_payload_sort_then_emit_needs_sort (one failure
on a fresh box): ws_sort_text (fused), then ws_sort(h, 0) + ws_emit_lines on
the same handle. Varies seeds, sleeps (clock ramp-down), and reports the
first differing line and its length."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle
from paper_1407_6603_b200 import synth, _native

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = 0
for it in range(iters):
    if it % 4 == 3:
        time.sleep(2.0)  # let the clocks drop
    text = synth.generate(4, words=200_000, seed=8 + (it // 2))
    want, _ = oracle.sort_text(text, mode="fast")
    h = _native.Handle(0)
    src = np.frombuffer(text, dtype=np.uint8)
    out = np.empty(len(text) + 64, dtype=np.uint8)
    n = h.sort_text(src, out)
    first = out[:n].tobytes() == want
    h.sort(False)
    got = h.emit_lines().tobytes()
    second = got == want
    if not (first and second):
        bad += 1
        g = (out[:n].tobytes() if not first else got).split(b"\n")
        w = want.split(b"\n")
        for i, (a, b) in enumerate(zip(g, w)):
            if a != b:
                print(f"it {it} first_ok={first} second_ok={second} line {i} len {len(b)}: got {a!r} want {b!r}",
                      flush=True)
                break
    h.close()
print("mismatches", bad, "of", iters, flush=True)
