"""Serving-loop period: wall time of ws_sort_texts batches of K corpora (config 4)."""
import sys, time
sys.path.insert(0, '.')
import torch
from bench import corpus
from paper_1407_6603_b200.pipeline import BatchSorter

text = corpus(4, 0)
for inflight in (2, 3, 4):
    bs = BatchSorter(len(text), inflight=inflight, device=0)
    bs.load(text)
    bs.run(4)
    res = []
    for k in (4, 8, 16, 32):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bs.run(k)
        res.append((k, (time.perf_counter() - t0) * 1e3))
    (k1, t1), (k2, t2) = res[-2], res[-1]
    print(f"inflight={inflight}", " ".join(f"K={k}:{t/k:.2f}ms/job" for k, t in res),
          f"period={(t2 - t1) / (k2 - k1):.3f}ms")
    bs.close()
