"""Instruction share per source-line range (phases) from ncu_lines output."""
import subprocess, sys, re, collections
rep, kern = sys.argv[1], sys.argv[2]
ranges = [tuple(x.split(':')) for x in sys.argv[3:]]  # name:file:lo-hi
out = subprocess.run([sys.executable, 'tools/ncu_lines.py', rep, kern, '100000'], capture_output=True, text=True).stdout
agg = collections.Counter(); tot = 0
for line in out.splitlines()[1:]:
    m = re.match(r'\s*([\d.]+)% inst\s+([\d.]+)% stall\s+(\S+):(\d+)', line)
    if not m: continue
    pct, f, ln = float(m.group(1)), m.group(3), int(m.group(4))
    tot += pct
    name = 'other'
    for nm, fn, rg in ranges:
        lo, hi = map(int, rg.split('-'))
        if fn in f and lo <= ln <= hi:
            name = nm; break
    agg[name] += pct
for k, v in agg.most_common():
    print(f'{k:12s} {v:5.1f}%')
