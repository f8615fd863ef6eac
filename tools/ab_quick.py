"""Quick A/B of library variants on the device-resident step (config 4).

usage: python tools/ab_quick.py VARIANT... (default | env:NAME=VALUE | a build/variants/ name)
AB_STATS=1 times the stats-mode step (ordered ingest + merge sort + SortStats) instead.
Each variant runs in its own process (WSORT_LIB); prints the median step time
(CUDA events on the library stream, 256 MiB L2 flush between steps) and the
per-phase times of one profiled step. Two rounds, interleaved.
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, statistics
sys.path.insert(0, '.')
import torch
from bench import corpus
from paper_1407_6603_b200._native import Handle
text = corpus(4, 0)
h = Handle(0)
h.ingest_text(text)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
st = torch.cuda.ExternalStream(h.stream_ptr()) if hasattr(h, 'stream_ptr') else torch.cuda.current_stream()
import os
stats = os.environ.get("AB_STATS") == "1"
if stats:
    d = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
def step():
    if stats:  # ordered ingest + merge sort with SortStats
        h.ingest_text(None, device_ptr=d.data_ptr(), n=len(text)); h.sort(True); h.bucket_stats(True)
    else:
        h.sort_resident(len(text))
ts = []
for i in range(25):
    flush.zero_()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    step()
    torch.cuda.synchronize()
    b.record(); torch.cuda.synchronize()
    if i >= 5: ts.append(a.elapsed_time(b))
h.profile(reset=True)
h.set_profiling(True)
step()
h.set_profiling(False)
ph = h.profile(reset=True)
agg = {}
for p in ph:
    agg[p["name"]] = agg.get(p["name"], 0) + p["ms"]
print(json.dumps({"ms": statistics.median(ts), "min": min(ts), "phases": {k: round(v, 4) for k, v in agg.items()}}))
'''


def main(variants):
    for rnd in range(2):
        for v in variants:
            env = dict(os.environ)
            env.pop("WSORT_LIB", None)
            if v.startswith("env:"):  # env:NAME=VALUE on the default library
                k, _, val = v[4:].partition("=")
                env[k] = val
            elif v != "default":
                env["WSORT_LIB"] = f"build/variants/{v}/libwsort_b200.so"
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
            print(f"[{rnd}] {v:14s} {line}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["default"])
