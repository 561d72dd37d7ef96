for d in 4096 8192 16384 32768 4096 8192 16384; do
  echo "div=$d S26 $(SSB_DENSE_DIV=$d python scripts/iter_profile.py --scale 26 2>/dev/null)"
  echo "div=$d S22 $(SSB_DENSE_DIV=$d python scripts/iter_profile.py --scale 22 2>/dev/null)"
done
