#!/bin/bash
# A/B of radix variants: class-0 radix span in the resident timeline + bench value.
# usage: tools/ab_radix.sh VARIANT... (default | rts | a build/variants/ name)
radix_span() { python tools/resident_timeline.py | python -c "
import re, sys
rows=[(l.split()[0], *map(float, re.findall(r'=\s*([0-9.]+)', l))) for l in sys.stdin if '=' in l]
r=[x for x in rows if x[0]=='radix_l0']
print('radix span %.3f  end %.3f' % (max(x[3] for x in r) - r[0][1], max(x[3] for x in rows)))"; }
for rep in 1 2; do
for v in "$@"; do
  unset WSORT_LIB WSORT_RADIX_RTS
  if [ $v = rts ]; then export WSORT_RADIX_RTS=1; elif [ $v != default ]; then export WSORT_LIB=build/variants/$v/libwsort_b200.so; fi
  echo "== $v $(radix_span) bench $(python bench.py --steps 20 --warmup 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["value"]/1e9,2), round(d["ms_per_step"],4))')"
done
done
