#!/bin/bash
# Plan-time / threshold knobs re-swept after the round-2 kernel changes (one
# process per setting, interleaved twice): S22 task budget and taper, S26
# direct / hashed-summary thresholds.
tag=${1:-ab_knobs}
{
for rep in 1 2; do
  for e in "SSB_TASK_BUDGET=256" "SSB_TASK_BUDGET=128" "SSB_TASK_BUDGET=512" "SSB_TASK_TAPER=80" "SSB_TASK_TAPER_DIV=8"; do
    echo "env=[$e] rep=$rep $(env $e python scripts/iter_profile.py --scale 22 --roots 64 2>/dev/null)"
  done
done
for rep in 1 2; do
  for e in "SSB_DIRECT_THR=262144" "SSB_DIRECT_THR=524288 SSB_HASH_THR=524288" "SSB_DIRECT_THR=1048576 SSB_HASH_THR=1048576" "SSB_HASH_THR=131072"; do
    echo "env=[$e] rep=$rep $(env $e python scripts/iter_profile.py --scale 26 --roots 64 2>/dev/null)"
  done
done
} > gpurun_out/${tag}.txt 2>&1
