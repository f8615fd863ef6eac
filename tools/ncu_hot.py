"""Hot SASS regions of one kernel in an ncu report (instructions executed, stall samples)."""
import csv, subprocess, sys


def main(rep, kernel, top=25):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', kernel,
                          '--launch-count', '1', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) > 10]
    ia = hdr.index('Instructions Executed'); src = hdr.index('Source')
    st = hdr.index('Warp Stall Sampling (All Samples)')
    num = lambda x: int(x) if x.isdigit() else 0
    tot = sum(num(r[ia]) for r in data)
    samp = sum(num(r[st]) for r in data)
    print(f'{kernel}: total warp-inst {tot}, stall samples {samp}, sass {len(data)}')
    regions, prev, start, acc = [], None, 0, 0
    for i, r in enumerate(data + [['x'] * len(hdr)]):
        c = num(r[ia]) if i < len(data) else -1
        if c != prev:
            if prev is not None:
                regions.append((prev, i - start, acc, start))
            prev, start, acc = c, i, 0
        if i < len(data):
            acc += num(r[st])
    for c, n, s, i in sorted(regions, key=lambda x: -x[0] * x[1])[:int(top)]:
        print(f"exec={c:9d} x{n:4d} = {c*n:11d} ({100*c*n/max(tot,1):5.1f}%) stalls={s:6d} "
              f"@{i:4d} {data[i][src].strip()[:70]}")


if __name__ == '__main__':
    main(*sys.argv[1:])
