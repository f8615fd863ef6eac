"""Per-phase timeline (CUDA events) of one device-resident pass on config 4."""
import sys
sys.path.insert(0, '.')
import torch
from bench import corpus
from paper_1407_6603_b200._native import Handle

text = corpus(int(sys.argv[1]) if len(sys.argv) > 1 else 4, 0)
h = Handle(0)
h.ingest_text(text)
for _ in range(3):
    h.sort_resident(len(text))
torch.cuda.synchronize()
h.profile(reset=True)
h.set_profiling(True)
h.sort_resident(len(text))
h.set_profiling(False)
ph = h.profile(reset=True)
t0 = min(p["start_ms"] for p in ph)
for p in sorted(ph, key=lambda p: p["start_ms"]):
    print(f'{p["name"]:12s} start={p["start_ms"]-t0:7.3f} dur={p["ms"]:6.3f} end={p["start_ms"]-t0+p["ms"]:7.3f} MB={p["bytes"]/1e6:7.1f}')
