"""Warp-instructions executed per SASS opcode of one kernel in an ncu report,
grouped by the pipe that executes them (alu / fma / xu / lsu / other), so an
integer kernel's real bound shows: on Blackwell the alu and fma pipes each
take 2 cycles per warp-instruction per SMSP, the xu pipe (FLO, BREV, POPC,
...) more. usage: python tools/ncu_opcodes.py REP KERNEL_REGEX [SKIP]"""
import collections
import csv
import subprocess
import sys

PIPE = {
    "alu": ("IADD3", "LOP3", "SHF", "PRMT", "ISETP", "SEL", "MOV", "LEA", "VIMNMX", "IABS",
            "PLOP3", "FSEL", "P2R", "R2P", "LOP", "SHL", "SHR", "IMNMX", "BMSK", "SGXT", "CS2R"),
    "fma": ("IMAD", "VIADD", "FFMA", "FMUL", "FADD", "IMUL", "HFMA2", "IADD", "IMADSP"),
    "xu": ("FLO", "BREV", "POPC", "MUFU", "I2F", "F2I", "FRND"),
    "lsu": ("LDS", "STS", "LDG", "STG", "ATOMS", "ATOMG", "RED", "LD", "ST", "LDC", "SHFL",
            "MATCH", "REDUX", "LDSM", "ATOM", "REDG"),
}


def pipe_of(op):
    base = op.split(".")[0]
    for p, ops in PIPE.items():
        if base in ops:
            return p
    return "other"


def main(rep, kernel, skip="0"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          "regex:" + kernel, "--launch-skip", str(skip), "--launch-count", "1",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if "Instructions Executed" in r)
    ia, src = hdr.index("Instructions Executed"), hdr.index("Source")
    per_op = collections.Counter()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= max(ia, src) or not r[ia].isdigit():
            continue
        text = r[src].strip()
        if text.startswith("@"):
            text = text.split(None, 1)[1] if " " in text else text
        op = text.split()[0] if text else "?"
        per_op[op] += int(r[ia])
    tot = sum(per_op.values()) or 1
    per_pipe = collections.Counter()
    for op, c in per_op.items():
        per_pipe[pipe_of(op)] += c
    print(f"total warp-inst {tot}")
    for p, c in per_pipe.most_common():
        print(f"  {p:6s} {c:12d} {100 * c / tot:5.1f}%")
    for op, c in per_op.most_common(30):
        print(f"    {op:24s} {pipe_of(op):5s} {c:12d} {100 * c / tot:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
