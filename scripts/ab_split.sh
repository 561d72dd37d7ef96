for x in 0 1 2 4; do
  echo "== split$x"
  export SSB_LIB=$PWD/build_old/split$x.so
  python scripts/iter_overhead.py 2>&1 | tail -2
  for i in 0 1 2; do python scripts/prof_iter.py --scale 22 --g500 $i --iters 100 --L 2048 2>&1 | sed -n 3p | cut -c1-300; done
  python scripts/prof_iter.py --scale 26 --g500 0 --iters 100 --L 2048 2>&1 | sed -n 3p | cut -c1-300
done
