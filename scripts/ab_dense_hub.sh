#!/bin/bash
# Early-exit switch point on hub-heavy graphs with the hashed summary (S26, 64 roots, twice)
{
for rep in 1 2; do
  for e in "SSB_DENSE_DIV_HUB=32768" "SSB_DENSE_DIV_HUB=65536" "SSB_DENSE_DIV_HUB=131072" "SSB_DENSE_DIV_HUB=16384"; do
    echo "env=[$e] rep=$rep $(env $e python scripts/iter_profile.py --scale 26 --roots 64 2>/dev/null)"
  done
done
} > gpurun_out/ab_dense_hub.txt 2>&1
