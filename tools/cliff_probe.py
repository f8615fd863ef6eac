"""Resident-step time on adversarial inputs (performance cliffs), payload
checked against the oracle: python tools/cliff_probe.py [--phases] [names...]
(--phases: also the per-phase device times of one profiled step)"""
import json, statistics, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from oracle import oracle
from paper_1407_6603_b200._native import Handle, device_bytes

rng = np.random.default_rng(7)
AL = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", dtype=np.uint8)


def words(n, L, alphabet=AL):
    w = alphabet[rng.integers(0, len(alphabet), size=(n, L))]
    sep = np.full((n, 1), 32, dtype=np.uint8)
    return np.concatenate([w, sep], axis=1).tobytes()


CASES = {
    "one_word_16M": lambda: b"hello " * 16_000_000,
    "unique5_8M": lambda: words(8_000_000, 5),
    "len32_3M": lambda: words(3_000_000, 32),
    "len1_2_16M": lambda: words(8_000_000, 1) + words(8_000_000, 2),
    "long40_1M": lambda: words(1_000_000, 40),
    "one_huge_word_64MB": lambda: b"x" * (64 << 20),
    "descending6_4M": lambda: b" ".join(sorted({bytes(r) for r in AL[rng.integers(0, 26, size=(4_200_000, 6))]}, reverse=True)[:4_000_000]),
}


def run(name, text):
    h = Handle(0)
    h.ingest_text(text, unordered=True)
    for _ in range(3):
        h.sort_resident(len(text))
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); h.sort_resident(len(text)); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    got = device_bytes(*h.output_device())
    phases = None
    if PHASES:
        h.profile(reset=True)
        h.set_profiling(True)
        h.sort_resident(len(text))
        h.set_profiling(False)
        phases = {}
        for p in h.profile(reset=True):
            phases[p["name"]] = round(phases.get(p["name"], 0) + p["ms"], 4)
    t0 = time.time()
    want, _ = oracle.sort_text(text, mode="fast", max_len=1 << 27)
    print(json.dumps({"case": name, "bytes": len(text), "ms": round(statistics.median(ts), 4),
                      "parity": got == want, "oracle_s": round(time.time() - t0, 1),
                      **({"phases": phases} if phases else {})}), flush=True)


PHASES = "--phases" in sys.argv
for name in [a for a in sys.argv[1:] if a != "--phases"] or CASES:
    run(name, CASES[name]())
