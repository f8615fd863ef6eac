"""Run the device-resident pass (ingest + sort + emit) a few times on the
config-4 workload; a small driver for ncu captures of single kernels."""
import sys
sys.path.insert(0, '.')
from bench import corpus
from paper_1407_6603_b200._native import Handle

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
text = corpus(cfg, 0)
h = Handle(0)
h.ingest_text(text, unordered=True)  # setup only; the timed passes re-ingest
for _ in range(reps):
    h.sort_resident(len(text))
print("ok", len(text))
