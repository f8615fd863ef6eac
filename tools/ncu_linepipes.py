"""Per CUDA source line: warp-instructions executed split by pipe (alu / fma /
xu / lsu / other) and the average active threads, from an ncu report with
-lineinfo (source page, cuda+sass). usage:
python tools/ncu_linepipes.py REP KERNEL_REGEX [TOP] [SKIP]"""
import collections
import csv
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_opcodes import pipe_of  # noqa: E402


def main(rep, kernel, top=40, skip=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", "regex:" + kernel, "--launch-skip", str(skip),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, cur = "?", None, None
    agg = collections.defaultdict(collections.Counter)
    thr = collections.Counter()
    src = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            te = hdr.index("Thread Instructions Executed")
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            src[cur] = r[1]
            continue
        text = r[3].strip()
        if not r[ie].isdigit() or text == "...":
            continue
        if text.startswith("@"):
            text = text.split(None, 1)[1] if " " in text else text
        op = text.split()[0] if text else "?"
        agg[cur][pipe_of(op)] += int(r[ie])
        thr[cur] += int(r[te]) if r[te].isdigit() else 0
    tot = collections.Counter()
    for c in agg.values():
        tot.update(c)
    T = sum(tot.values()) or 1
    print("total", {k: f"{v} ({100 * v / T:.1f}%)" for k, v in tot.items()})
    rank = sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[: int(top)]
    for k, c in rank:
        n = sum(c.values())
        avg = thr[k] / n if n else 0
        print(f"{100 * n / T:5.1f}% alu {100 * c['alu'] / T:4.1f} fma {100 * c['fma'] / T:4.1f} "
              f"xu {100 * c['xu'] / T:4.1f} thr {avg:4.1f}  {k[0]}:{k[1]:<5d} {src.get(k, '').strip()[:70]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
