#!/bin/bash
# ab/dz1.so: scripts/build_variant.sh $PWD/ab/dz1.so -DSSB_LEAN_DECIDED_ZERO=1
{
bash scripts/ab_libs.sh "--scale 26 --roots 64" base $PWD/ab/dz1.so
bash scripts/ab_libs.sh "--scale 22 --roots 64" base $PWD/ab/dz1.so
bash scripts/ab_libs.sh "--scale 26 --roots 16 --variant 0" base $PWD/ab/dz1.so
} > gpurun_out/ab_decided_zero.txt 2>&1
SSB_LIB=$PWD/ab/dz1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ab_decided_zero_parity.txt 2>&1; echo rc=$? >> gpurun_out/ab_decided_zero_parity.txt
