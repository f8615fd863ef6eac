"""Warp-instructions executed per SASS address window of one kernel, with the
source lines the window's instructions come from, in address order (inlined
helpers show up where they are inlined):
python tools/ncu_sass_phases.py REP KERNEL_REGEX [WINDOW]."""
import csv, subprocess, sys


def main(rep, kernel, window=48):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kernel,
                          '--launch-count', '1', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, cur, fname = None, None, '?'
    sass = []
    for r in rows:
        if len(r) == 2 and r[0] == 'File Path':
            fname = r[1].split('/')[-1].replace('.cu', '').replace('.cuh', 'h')
            continue
        if r and r[0] == 'Line No':
            hdr = r
            ie, te = hdr.index('Instructions Executed'), hdr.index('Thread Instructions Executed')
            ss = hdr.index('Warp Stall Sampling (All Samples)')
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur = f'{fname}:{r[0]}'
            continue
        if r[2].startswith('0x'):
            num = lambda x: int(float(x)) if x.replace('.', '').isdigit() else 0
            sass.append((int(r[2], 16), num(r[ie]), num(r[te]), cur, r[3].strip(), num(r[ss])))
    sass.sort()
    tot = sum(x[1] for x in sass) or 1
    stot = sum(x[5] for x in sass) or 1
    print(f'{len(sass)} sass, total warp-inst {tot}, stall samples {stot}')
    w = int(window)
    for i in range(0, len(sass), w):
        blk = sass[i:i + w]
        c = sum(x[1] for x in blk)
        t = sum(x[2] for x in blk)
        st = sum(x[5] for x in blk)
        if c * 1000 < tot and st * 200 < stot:
            continue
        seen = []
        for x in blk:
            if x[3] not in seen:
                seen.append(x[3])
        print(f'{i:5d} {100 * c / tot:5.1f}% stall {100 * st / stot:5.1f}% util {t / max(c, 1) / 32:4.2f}  {" ".join(seen)[:140]}')


if __name__ == '__main__':
    main(*sys.argv[1:])
