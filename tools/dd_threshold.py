"""Where counting starts to pay: device-resident step time of config-4-like
texts of several sizes with the counting path forced on (WSORT_DEDUPE_MIN=0)
and off (WSORT_NO_DEDUPE=1). usage: python tools/dd_threshold.py [words ...]"""
import json, os, subprocess, sys

CHILD = r'''
import sys, statistics, json
sys.path.insert(0, '.')
import torch
from paper_1407_6603_b200 import synth
from paper_1407_6603_b200._native import Handle
words = int(sys.argv[1])
text = synth.generate(4, words=words, seed=3)
h = Handle(0)
h.ingest_text(text)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
ts = []
for i in range(25):
    flush.zero_()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); h.sort_resident(len(text)); torch.cuda.synchronize(); b.record(); torch.cuda.synchronize()
    if i >= 5: ts.append(a.elapsed_time(b))
print(json.dumps({"words": words, "bytes": len(text), "ms": round(statistics.median(ts), 4), "counted": h.counted_classes()}))
'''

for w in [int(x) for x in sys.argv[1:]] or [1_000_000, 2_000_000, 4_000_000, 8_000_000]:
    row = {}
    for name, env in (("counting", {"WSORT_DEDUPE_MIN": "0"}), ("sorting", {"WSORT_NO_DEDUPE": "1"})):
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, "-c", CHILD, str(w)], env=e, capture_output=True, text=True).stdout.strip().splitlines()
        row[name] = json.loads(out[-1]) if out else None
    print(json.dumps(row), flush=True)
