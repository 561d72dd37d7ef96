#!/bin/bash
# ab/hs1.so: scripts/build_variant.sh $PWD/ab/hs1.so -DSSB_HASH_SHIFT=1 (the A/B build of commit 386bcc6 + the macro; the shift is the only form since)
# shift vs high-multiply summary hash (S26 sel-max 64 roots, tropical 16), then parity of the shift build
{
bash scripts/ab_libs.sh "--scale 26 --roots 64" base $PWD/ab/hs1.so
bash scripts/ab_libs.sh "--scale 26 --roots 16 --variant 0" base $PWD/ab/hs1.so
} > gpurun_out/ab_hash_shift.txt 2>&1
SSB_LIB=$PWD/ab/hs1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sweep_modes or c32_golden or selftest" > gpurun_out/ab_hash_shift_parity.txt 2>&1; echo rc=$? >> gpurun_out/ab_hash_shift_parity.txt
