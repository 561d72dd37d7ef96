#!/bin/bash
# Frontier-image budget re-swept with the hashed summary (S26 64 roots, S22 64 roots, twice)
{
for rep in 1 2; do
  for e in "SSB_SMEM_KB=160" "SSB_SMEM_KB=144" "SSB_SMEM_KB=176" "SSB_SMEM_KB=192"; do
    echo "env=[$e] rep=$rep $(env $e python scripts/iter_profile.py --scale 26 --roots 64 2>/dev/null)"
    echo "env=[$e] rep=$rep $(env $e python scripts/iter_profile.py --scale 22 --roots 64 2>/dev/null)"
  done
done
} > gpurun_out/ab_smem.txt 2>&1
