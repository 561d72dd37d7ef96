#!/bin/bash
# ab/bc1.so: scripts/build_variant.sh $PWD/ab/bc1.so at commit 0ed113d (before the hashed summary)
# A/B of the tree against ab/bc1.so (the kernel before the hashed summary), then the GPU suite
{
bash scripts/ab_libs.sh "--scale 22 --roots 64" $PWD/ab/bc1.so base
bash scripts/ab_libs.sh "--scale 26 --roots 64" $PWD/ab/bc1.so base
bash scripts/ab_libs.sh "--scale 26 --roots 16 --variant 0" $PWD/ab/bc1.so base
} > gpurun_out/ab_hash4.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_hash4_gputest.txt 2>&1; echo rc=$? >> gpurun_out/ab_hash4_gputest.txt
