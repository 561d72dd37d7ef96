for d in 128 512 2048 8192 128 512 2048; do
  echo "div=$d ER $(SSB_DENSE_DIV=$d python scripts/iter_profile.py --scale 26 --graph er --roots 16 2>/dev/null)"
done
