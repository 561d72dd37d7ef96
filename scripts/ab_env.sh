#!/bin/bash
# ab_env.sh TAG "VAR=a VAR2=b" "VAR=c" ... : per-iteration A/B of runtime knobs (S22 64 roots,
# S26 and Erdős–Rényi 2^26 16 roots), each setting run twice, interleaved, on one box.
tag=$1; shift
mkdir -p gpurun_out
for args in "--scale 22 --roots 64" "--scale 26 --roots 16" "--scale 26 --graph er --roots 16"; do
  for rep in 1 2; do
    for e in "$@"; do
      echo "env=[$e] rep=$rep $(env $e python scripts/iter_profile.py $args 2>/dev/null)"
    done
  done
done > gpurun_out/${tag}.txt 2>&1
