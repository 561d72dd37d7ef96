#!/bin/bash
# A/B of bfs.cu build variants (scripts/build_variant.sh): per-iteration times
# of a deep path BFS, three S22 Graph500 roots and one S26 root.
# usage: scripts/ab_split.sh NAME...   (build_old/NAME.so each)
for x in "$@"; do
  echo "== $x"
  export SSB_LIB=$PWD/build_old/$x.so
  python scripts/iter_overhead.py 2>&1 | tail -2
  for i in 0 1 2; do python scripts/prof_iter.py --scale 22 --g500 $i --iters 100 --L 2048 2>&1 | sed -n 3p | cut -c1-300; done
  python scripts/prof_iter.py --scale 26 --g500 0 --iters 100 --L 2048 2>&1 | sed -n 3p | cut -c1-300
  [ -n "$AB_ER" ] && python scripts/prof_iter.py --graph er --scale 26 --g500 0 --iters 100 --L 2048 2>&1 | sed -n 3p | cut -c1-300
done
