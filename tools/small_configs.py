"""Device-resident step time (median of CUDA-event timed steps, L2 flushed)
of configs 0-3, payload checked against the oracle once per config.
usage: python tools/small_configs.py [configs...]   (env knobs apply, e.g. WSORT_NO_TINY=1)"""
import json, os, statistics, sys
sys.path.insert(0, '.')
import torch
from bench import corpus
from oracle import oracle
from paper_1407_6603_b200._native import Handle, device_bytes

cfgs = [int(c) for c in sys.argv[1:]] or [0, 1, 2, 3]
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for cfg in cfgs:
    text = corpus(cfg, 0)
    h = Handle(0)
    h.ingest_text(text, unordered=True)
    for _ in range(5):
        h.sort_resident(len(text))
    want, _ = oracle.sort_text(text, mode="fast")
    torch.cuda.synchronize()
    got = device_bytes(*h.output_device())
    ts = []
    for _ in range(30):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); h.sort_resident(len(text)); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ok = None
    if got is not None:
        ok = got == want
    print(json.dumps({"config": cfg, "bytes": len(text), "ms": round(statistics.median(ts), 4),
                      "min": round(min(ts), 4), "parity": ok,
                      "knobs": {k: v for k, v in os.environ.items() if k.startswith("WSORT_")}}), flush=True)
