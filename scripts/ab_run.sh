#!/bin/bash
# ab_run.sh TAG lib1.so lib2.so ... : per-iteration A/B (S22 64 roots, S26 and ER 2^26 16 roots)
# over the listed libraries ("base" = the in-tree build), interleaved twice on one box.
tag=$1; shift
mkdir -p gpurun_out
{
  bash scripts/ab_libs.sh "--scale 22 --roots 64" "$@"
  bash scripts/ab_libs.sh "--scale 26 --roots 16" "$@"
  bash scripts/ab_libs.sh "--scale 26 --graph er --roots 16" "$@"
} > gpurun_out/${tag}.txt 2>&1
