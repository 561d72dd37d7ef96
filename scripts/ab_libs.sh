#!/bin/bash
# ab_libs.sh "ARGS" lib1.so lib2.so ... : iter_profile.py per library, interleaved twice (same box)
args=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = base ]; then unset SSB_LIB; else export SSB_LIB=$lib; fi
    echo "lib=$lib rep=$rep $(python scripts/iter_profile.py $args 2>/dev/null)"
  done
done
