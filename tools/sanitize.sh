#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck, synccheck and initcheck over
# every device path (tools/sanitize_driver.py) on configs 0 and 1 (a 60k-word
# prefix of config 1 for the slow racecheck), then memcheck on each WSORT_*
# knob path. Writes gpurun_out/sanitize/*.log and a summary table.
# usage (on the GPU box): bash tools/sanitize.sh [quick]
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
SUMMARY=$OUT/summary.txt
: > $SUMMARY
run() {  # name tool env... -- args
  local name=$1 tool=$2; shift 2
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done
  shift
  local log=$OUT/$name.log
  local t0=$(date +%s)
  env "${envs[@]}" timeout 1500 $CS --tool $tool --error-exitcode 99 --print-limit 50 \
      --target-processes all python tools/sanitize_driver.py "$@" > $log 2>&1
  local rc=$?
  local errs=$(grep -Eo "ERROR SUMMARY: [0-9]+ error" $log | tail -1)
  local haz=$(grep -Eo "RACECHECK SUMMARY: [0-9]+ hazard[s]? displayed \([0-9]+ error" $log | tail -1)
  printf "%-28s %-10s rc=%-3s %-28s %s %ss %s\n" "$name" "$tool" "$rc" "${errs:-no summary}" \
      "${haz}" "$(( $(date +%s) - t0 ))" "$(grep -c 'sanitize driver ok' $log) ok" | tee -a $SUMMARY
}
for cfg in 0 1; do
  W=0; [ $cfg = 1 ] && W=60000
  run memcheck_c$cfg memcheck -- $cfg
  run racecheck_c$cfg racecheck -- $cfg $W
  run synccheck_c$cfg synccheck -- $cfg $W
  run initcheck_c$cfg initcheck -- $cfg $W
done
[ "${1:-}" = quick ] && exit 0
for knob in WSORT_NO_RADIX WSORT_NO_SAMPLE WSORT_LOOKBACK WSORT_TWO_PASS WSORT_NO_FUSED_SLOTS \
            WSORT_NO_JOINT WSORT_NO_EARLY_HIST WSORT_NO_EARLY_SPLIT WSORT_SERIAL WSORT_D2H_PER_CLASS \
            WSORT_NO_FUSED_PAYLOAD; do
  run memcheck_c1_$knob memcheck $knob=1 -- 1
  run racecheck_c0_$knob racecheck $knob=1 -- 0 20000
done
