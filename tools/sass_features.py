"""Per-kernel counts of selected SASS instruction classes in the built library
objects (cuobjdump -sass): bulk copies (TMA, UBLKCP), mbarrier waits (SYNCS),
MATCH, REDUX, VOTE, shared / global atomics, LDS/STS, plus the register count.
usage: python tools/sass_features.py [build/*.o ...] > profiles/r02_sass_features.txt"""
import re, subprocess, sys, glob

PATS = {"UBLKCP(TMA)": r"\bUBLKCP", "SYNCS(mbar)": r"\bSYNCS", "MATCH": r"\bMATCH\.", "REDUX": r"\bREDUX",
        "VOTE": r"\bVOTE", "ATOMS": r"\bATOMS", "ATOMG/RED": r"\b(ATOMG|RED)\.", "LDS": r"\bLDS", "STS": r"\bSTS",
        "BAR": r"\bBAR\.", "SHFL": r"\bSHFL"}


def main(objs):
    print(f"{'kernel':70s} " + " ".join(f"{k:>11s}" for k in PATS) + "  total")
    for o in objs:
        out = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
        for m in re.finditer(r"Function : (\S+)\n(.*?)(?=\n\s*Function : |\Z)", out, re.S):
            name, body = m.group(1), m.group(2)
            lines = [l for l in body.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            dem = re.sub(r"\(.*", "", dem).replace("ws::", "").replace("(anonymous namespace)::", "")
            cnt = [sum(1 for l in lines if re.search(p, l)) for p in PATS.values()]
            print(f"{dem[:70]:70s} " + " ".join(f"{c:11d}" for c in cnt) + f"  {len(lines)}")


if __name__ == "__main__":
    main(sys.argv[1:] or sorted(glob.glob("build/*.o")))
