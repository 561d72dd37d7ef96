for cfg in "SSB_TASK_TAPER=100" "SSB_TASK_TAPER=90" "SSB_TASK_TAPER=75" "SSB_TASK_TAPER=90 SSB_TASK_TAPER_DIV=8" "SSB_TASK_TAPER=100" "SSB_TASK_TAPER=90" "SSB_TASK_TAPER=75"; do
  echo "$cfg | S26 $(env $cfg python scripts/iter_profile.py --scale 26 2>/dev/null)"
  echo "$cfg | S22 $(env $cfg python scripts/iter_profile.py --scale 22 2>/dev/null)"
done
