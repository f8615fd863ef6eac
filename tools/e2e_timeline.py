"""Timeline of one ws_sort_text call (config 4): per-phase CUDA events + wall time."""
import sys, time
sys.path.insert(0, '.')
import torch
from bench import corpus
from paper_1407_6603_b200.pipeline import TextSorter

text = corpus(4, 0)
ts = TextSorter(len(text), device=0)
ts.load(text)
for _ in range(3):
    ts.run()
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); ts.run(); print(f"wall {1e3*(time.perf_counter()-t0):.3f} ms")
ts.handle.profile(reset=True)
ts.handle.set_profiling(True)
t0 = time.perf_counter(); ts.run(); wall = 1e3 * (time.perf_counter() - t0)
ts.handle.set_profiling(False)
ph = ts.handle.profile(reset=True)
t0e = min(p["start_ms"] for p in ph)
for p in sorted(ph, key=lambda p: p["start_ms"]):
    if p["name"].startswith(("d2h", "runs", "emit", "h2d", "ingest", "radix", "tile", "merge")):
        print(f'{p["name"]:12s} start={p["start_ms"]-t0e:7.3f} dur={p["ms"]:6.3f} MB={p["bytes"]/1e6:7.1f}')
print(f"wall(profiled) {wall:.3f} ms")
