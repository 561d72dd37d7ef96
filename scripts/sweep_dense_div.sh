for d in 4096 1024 16384 2048 4096; do
  echo "== SSB_DENSE_DIV=$d"
  SSB_DENSE_DIV=$d python scripts/iter_profile.py --scale 26
  SSB_DENSE_DIV=$d python scripts/k3_per_root.py | awk '{print $2, $5, $6}' | tr '\n' ';'
  echo
done
