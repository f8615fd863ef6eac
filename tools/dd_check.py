"""Distinct-word counting on a bench config: the device-resident payload
byte-compared with the oracle, the classes that were counted, and the
per-phase timeline of one profiled step. usage: dd_check.py [config]"""
import sys
sys.path.insert(0, '.')
from bench import corpus
from oracle import oracle
from paper_1407_6603_b200 import _native
from paper_1407_6603_b200._native import Handle

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
text = corpus(cfg, 0)
h = Handle(0)
h.ingest_text(text)
for _ in range(3):
    n = h.sort_resident(len(text))
p, size = h.output_device()
got = _native.device_bytes(p, size)
want = oracle.sort_text(text, mode="fast")[0]
print("config", cfg, "bytes", len(text), "payload", size, "counted classes", bin(h.counted_classes()),
      "PARITY", got == want)
if got != want:
    import numpy as np
    a = np.frombuffer(got, np.uint8); b = np.frombuffer(want, np.uint8)
    m = min(len(a), len(b))
    d = np.nonzero(a[:m] != b[:m])[0]
    print("sizes", len(a), len(b), "first diff", d[:5], got[max(0, int(d[0]) - 40):int(d[0]) + 40] if len(d) else None,
          want[max(0, int(d[0]) - 40):int(d[0]) + 40] if len(d) else None)
h.profile(reset=True)
h.set_profiling(True)
h.sort_resident(len(text))
h.set_profiling(False)
ph = h.profile(reset=True)
t0 = min(q["start_ms"] for q in ph)
for q in sorted(ph, key=lambda q: q["start_ms"]):
    print(f'{q["name"]:16s} start={q["start_ms"]-t0:7.3f} dur={q["ms"]:6.3f} end={q["start_ms"]-t0+q["ms"]:7.3f} MB={q["bytes"]/1e6:7.1f}')
