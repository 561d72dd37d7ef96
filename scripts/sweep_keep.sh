for k in 0 32 64 96 0 32 64 96; do
  echo "keep=$k | S22 $(SSB_KEEP_MB=$k python scripts/iter_profile.py --scale 22 2>/dev/null)"
  echo "keep=$k | S26 $(SSB_KEEP_MB=$k python scripts/iter_profile.py --scale 26 --roots 16 2>/dev/null)"
done
