#!/bin/bash
# SSB_DIRECT_THR sweep (|F| above which the early-exit sweeps probe the exact
# frontier directly instead of the summary); default = the summary's bit count.
for t in 65536 131072 262144 524288 65536 131072 262144 524288; do
  echo "thr=$t S26 $(SSB_DIRECT_THR=$t python scripts/iter_profile.py --scale 26 2>/dev/null)"
done
for t in 16384 32768 65536 131072 16384 32768 65536 131072; do
  echo "thr=$t S22 $(SSB_DIRECT_THR=$t python scripts/iter_profile.py --scale 22 2>/dev/null)"
done
