"""Stats-mode passes (ordered ingest + merge sort with SortStats) on config 4,
text already on the device; a small driver for ncu captures."""
import sys
sys.path.insert(0, '.')
import torch
from bench import corpus
from paper_1407_6603_b200._native import Handle

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
text = corpus(4, 0)
d = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
h = Handle(0)
for _ in range(reps):
    h.ingest_text(None, device_ptr=d.data_ptr(), n=len(text))
    h.sort(True)
    h.bucket_stats(True)
torch.cuda.synchronize()
print("ok")
