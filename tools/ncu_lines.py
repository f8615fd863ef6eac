"""Per-CUDA-source-line instructions executed and stall samples from an ncu
report (needs -lineinfo): python tools/ncu_lines.py REP KERNEL_REGEX [TOP]."""
import csv, subprocess, sys, collections


def main(rep, kernel, top=40, skip=0):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                          '--kernel-name', 'regex:' + kernel, '--launch-skip', str(skip), '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = collections.defaultdict(lambda: [0, 0])
    src, fname = {}, '?'
    hdr = None
    cur = None
    for r in rows:
        if len(r) == 2 and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:  # a CUDA source line row
            cur = (fname, int(r[0]))
            src[cur] = r[1]
            ie = hdr.index('Instructions Executed')
            ss = hdr.index('Warp Stall Sampling (All Samples)')
            num = lambda x: int(float(x)) if x.replace('.', '').isdigit() else 0
            agg[cur][0] += num(r[ie])
            agg[cur][1] += num(r[ss])
    tot = sum(a[0] for a in agg.values()) or 1
    stot = sum(a[1] for a in agg.values()) or 1
    print(f'total warp-inst {tot}, stall samples {stot}')
    for k, (ie, ss) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(top)]:
        print(f'{100*ie/tot:5.1f}% inst {100*ss/stot:5.1f}% stall  {k[0]}:{k[1]:<5d} {src[k].strip()[:90]}')


if __name__ == '__main__':
    main(*sys.argv[1:])
