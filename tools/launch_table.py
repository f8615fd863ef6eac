"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel."""
import csv, sys, collections


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    out = []
    ik, im, iv, iid = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
    cur = {}
    for r in rows[1:]:
        d = cur.setdefault(r[iid], {'kernel': r[ik]})
        d[r[im]] = float(r[iv].replace(',', ''))
    return list(cur.values())


def main(path, skip=0):
    ls = load(path)[int(skip):]
    agg = collections.OrderedDict()
    for d in ls:
        k = d['kernel'].split('(')[0]
        a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get('gpu__time_duration.sum', 0) / 1e3
        a[2] += d.get('dram__bytes_read.sum', 0) / 1e6
        a[3] += d.get('dram__bytes_write.sum', 0) / 1e6
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':45s} {'n':>4s} {'us':>9s} {'share':>6s} {'MB rd':>8s} {'MB wr':>8s} {'GB/s':>7s}")
    for k, (n, us, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:45]:45s} {n:4d} {us:9.1f} {100*us/tot:5.1f}% {rd:8.1f} {wr:8.1f} {(rd+wr)/max(us,1e-9)*1e3:7.0f}")
    print(f"total {len(ls)} launches, {tot:.1f} us (serialised)")


if __name__ == '__main__':
    main(*sys.argv[1:])
