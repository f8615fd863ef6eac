"""Repeat a payload-mode sort of a duplicate-heavy word mix and count mismatches."""
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle
from paper_1407_6603_b200 import synth, _native
from paper_1407_6603_b200.pipeline import sort_text

rng = np.random.default_rng(5)
words = []
for L, alphabet, count in ((3, b"ab", 40), (12, b"ab", 30), (7, b"aZ09", 25), (25, b"ab", 20), (1, b"q", 10), (33, b"ab", 5)):
    al = np.frombuffer(alphabet, dtype=np.uint8)
    words += [bytes(r) for r in al[rng.integers(0, len(al), size=(count * 37, L))]]
rng.shuffle(words)
text = b" ".join(words)
want, _ = oracle.sort_text(text, mode="fast")
bad = 0
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
    if sort_text(text) != want:
        bad += 1
print("mismatches", bad)
