"""Per-phase time of the counting launches' tiles on a bench config (library
built with -DWS_DD_PROF=1: tools/build_variants.sh "ddprof:-DWS_DD_PROF=1").
usage: WSORT_LIB=build/variants/ddprof/libwsort_b200.so python tools/dd_phases.py [config]"""
import ctypes, sys
sys.path.insert(0, '.')
from bench import corpus
from paper_1407_6603_b200 import _native
from paper_1407_6603_b200._native import Handle

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
text = corpus(cfg, 0)
h = Handle(0)
h.ingest_text(text)
lib = _native.load_library()
buf = (ctypes.c_ulonglong * 16)()
for _ in range(3):
    h.sort_resident(len(text))
lib.dd_prof_read(buf)  # warm-up steps discarded
reps = 5
for _ in range(reps):
    h.sort_resident(len(text))
lib.dd_prof_read(buf)
names = ["clear", "count", "compact", "flush", "append"]
for g, gname in enumerate(["uint32 keys (lengths 1-5)", "wider keys"]):
    tiles = buf[8 * g + 7] / reps
    print(f"{gname}: {tiles:.0f} tiles per step")
    tot = 0
    for k in range(1, 5):
        us = buf[8 * g + k] / 1e3 / max(buf[8 * g + 7], 1)
        tot += us
        print(f"  {names[k]:8s} {us:7.2f} us per tile")
    print(f"  sum      {tot:7.2f} us per tile")
