#!/bin/bash
# A/B of environment settings: resident timeline end + bench value, two rounds.
# usage: tools/ab_env.sh "NAME=VALUE ..." ...   ("-" = no extra setting)
for rep in 1 2; do
for spec in "$@"; do
  envs=(); [ "$spec" != "-" ] && envs=($spec)
  end=$(env "${envs[@]}" python tools/resident_timeline.py | python -c "
import re, sys
rows=[(l.split()[0], *map(float, re.findall(r'=\s*([0-9.]+)', l))) for l in sys.stdin if '=' in l]
print('%.3f' % max(x[3] for x in rows))")
  b=$(env "${envs[@]}" python bench.py --steps 20 --warmup 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["value"]/1e9,2), round(d["ms_per_step"],4))')
  echo "== [$spec] timeline_end $end bench $b"
done
done
