"""Randomised stress: texts and word lists of mixed lengths / alphabets /
separators, payload and stats mode, fresh and reused handles, compared with
the oracle; runs for the given number of seconds."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle
from paper_1407_6603_b200 import synth, _native
from paper_1407_6603_b200.pipeline import DeviceCorpus, sort_text

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
alphabets = [b"ab", b"aZ09", synth.ALNUM, b"q", b"xyz"]
seps = [b" ", b"\n", b"., ", b"\x00", b"\xff-"]
t0, cases, fails = time.time(), 0, 0
shared = _native.Handle(0)
while time.time() - t0 < budget:
    words = []
    small = rng.random() < 0.35  # <= 512 KiB texts also take the small-corpus kernel (tiny_sort_kernel)
    for _ in range(rng.integers(1, 14)):
        L = int(rng.integers(1, 60)); al = np.frombuffer(alphabets[rng.integers(0, len(alphabets))], dtype=np.uint8)
        n = int(rng.integers(1, (3000 if small else 30000) if L < 33 else 2000))
        words += [bytes(r) for r in al[rng.integers(0, len(al), size=(n, L))]]
    rng.shuffle(words)
    text = seps[rng.integers(0, len(seps))].join(words)
    want, info = oracle.sort_text(text, mode="fast", max_len=64)
    ok = sort_text(text) == want
    if rng.random() < 0.5:
        dc = DeviceCorpus(shared if rng.random() < 0.5 else None)
        dc.ingest(text); dc.sort(want_stats=True)
        naive = dc.stats(naive=True)
        ok = ok and all(naive[L] == (c, s, p) for L, (n, inv, K, c, s, p) in info.items())
        ok = ok and dc.payload() == want
    if rng.random() < 0.15:  # a batch of several corpora through ws_sort_texts
        texts = [text] + [synth.generate(0, seed=int(rng.integers(1 << 30))) for _ in range(int(rng.integers(1, 5)))]
        wants = [want] + [oracle.sort_text(t, mode="fast")[0] for t in texts[1:]]
        arrs = [np.frombuffer(t, dtype=np.uint8) if t else np.zeros(0, np.uint8) for t in texts]
        outs = [np.empty(len(t) + 1, dtype=np.uint8) for t in texts]
        sizes = shared.sort_texts(arrs, outs, int(rng.integers(1, 5)))
        ok = ok and all(o[:z].tobytes() == w for o, z, w in zip(outs, sizes, wants))
    if rng.random() < 0.05:  # > 16 MiB: chunked upload overlapped with the ingest
        big = synth.generate(4, words=int(rng.integers(2_200_000, 3_000_000)), seed=int(rng.integers(1 << 30)))
        ok = ok and sort_text(big) == oracle.sort_text(big, mode="fast")[0]
    cases += 1
    if not ok:
        fails += 1
        print("FAIL case", cases, "words", len(words))
print(f"stress: {cases} cases, {fails} failures, {time.time() - t0:.0f} s")
