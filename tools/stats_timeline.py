"""Per-phase timeline (CUDA events) of one stats-mode pass (ordered ingest +
merge sort with SortStats) on config 4, text already on the device."""
import sys
sys.path.insert(0, '.')
import torch
from bench import corpus
from paper_1407_6603_b200._native import Handle

text = corpus(4, 0)
d = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
h = Handle(0)
for _ in range(3):
    h.ingest_text(None, device_ptr=d.data_ptr(), n=len(text)); h.sort(True); h.bucket_stats(True)
torch.cuda.synchronize()
h.profile(reset=True)
h.set_profiling(True)
h.ingest_text(None, device_ptr=d.data_ptr(), n=len(text)); h.sort(True); h.bucket_stats(True)
h.set_profiling(False)
ph = h.profile(reset=True)
t0 = min(p["start_ms"] for p in ph)
agg = {}
for p in ph:
    a = agg.setdefault(p["name"], [0, 0.0, 1e9, 0.0])
    a[0] += 1; a[1] += p["ms"]; a[2] = min(a[2], p["start_ms"] - t0); a[3] = max(a[3], p["start_ms"] - t0 + p["ms"])
for k, (n, ms, st, en) in sorted(agg.items(), key=lambda x: x[1][2]):
    print(f"{k:12s} n={n:3d} sum={ms:7.3f} ms  span {st:7.3f} .. {en:7.3f}")
