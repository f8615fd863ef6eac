"""WSORT_TRACE timeline of a ws_sort_texts batch (config 4)."""
import os, re, sys, subprocess
if os.environ.get("WSORT_TRACE") != "1":
    env = dict(os.environ, WSORT_TRACE="1")
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    ev = {}
    order = []
    for line in r.stderr.splitlines():
        m = re.match(r"wsort-trace handle=(\S+) (.*)", line)
        if not m:
            continue
        h = m.group(1)
        kv = dict(x.split("=") for x in m.group(2).split())
        if h not in order:
            order.append(h)
        ev.setdefault(h, []).append({k: float(v) for k, v in kv.items()})
    rows = []
    for h in order:
        cur = {}
        for e in ev[h]:
            cur.update(e)
            if "done" in e:
                rows.append((order.index(h), dict(cur)))
                cur = {}
    rows.sort(key=lambda r: r[1]["begin"])
    t0 = rows[0][1]["begin"] if rows else 0
    for slot, r in rows:
        print(f"slot{slot} " + " ".join(f"{k}={r[k]-t0:8.2f}" for k in ("begin", "h2d_landed", "ingested", "enqueued", "done") if k in r))
    sys.exit(0)
sys.path.insert(0, '.')
from bench import corpus
from paper_1407_6603_b200.pipeline import BatchSorter
text = corpus(4, 0)
inflight = int(sys.argv[1]) if len(sys.argv) > 1 else 3
bs = BatchSorter(len(text), inflight=inflight, device=0)
bs.load(text)
bs.run(12)
