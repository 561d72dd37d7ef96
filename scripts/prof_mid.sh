#!/bin/bash
# ab/iters1.so: scripts/build_variant.sh $PWD/ab/iters1.so -DSSB_ITERS_PER_LAUNCH=1
# The mid-frontier early-exit iteration (S26 root 24490569, |F_2| = 16,482:
# dense + hashed summary at k = 3): per-iteration times with and without the
# hashed summary, and one ncu capture of that iteration alone (one launch per
# iteration build; the hashed-summary flag is carried across launches).
python scripts/prof_iter.py --scale 26 --iters 4 --L 2048 --root 24490569 > gpurun_out/mid_hash.txt 2>&1
SSB_HASH_SUMMARY=0 python scripts/prof_iter.py --scale 26 --iters 4 --L 2048 --root 24490569 > gpurun_out/mid_nohash.txt 2>&1
SSB_LIB=$PWD/ab/iters1.so python scripts/prof_iter.py --scale 26 --iters 4 --L 2048 --root 24490569 > gpurun_out/mid_iters1.txt 2>&1
SSB_LIB=$PWD/ab/iters1.so ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 5 -c 1 -o gpurun_out/mid_k3 \
  python scripts/prof_iter.py --scale 26 --iters 3 --L 2048 --root 24490569 > gpurun_out/mid_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/mid_parity.txt 2>&1; echo rc=$? >> gpurun_out/mid_parity.txt
