# A/B: iteration profile + per-root k=3 for base vs variant libs
for lib in base "$@" base "$@"; do
  if [ "$lib" = base ]; then unset SSB_LIB; else export SSB_LIB=$lib; fi
  echo "lib=$lib S26 $(python scripts/iter_profile.py --scale 26 2>/dev/null)"
  echo "lib=$lib ER $(python scripts/iter_profile.py --scale 26 --graph er --roots 16 2>/dev/null)"
  echo "lib=$lib S22 $(python scripts/iter_profile.py --scale 22 2>/dev/null)"
done
