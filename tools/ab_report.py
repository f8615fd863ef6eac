"""Condense tools/ab_quick.py output: median step and selected phases per arm.
usage: python tools/ab_report.py AB_TXT [phase ...]"""
import json
import re
import sys

want = sys.argv[2:] or ["ingest", "radix_l0", "sample_l1", "sample_l2", "sample_l3"]
for line in open(sys.argv[1]):
    m = re.match(r"\[(\d)\] (\S+)\s+(\{.*\})", line)
    if not m:
        if line.strip() and not line.startswith(" "):
            print(line.rstrip()[:200])
        continue
    d = json.loads(m.group(3))
    ph = d["phases"]
    print(m.group(1), f"{m.group(2):12s}", f"{d['ms']:.4f}", {k: ph[k] for k in want if k in ph})
