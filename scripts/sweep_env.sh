#!/bin/bash
# One process per value of a plan-time knob (the plan is cached per range):
# usage: scripts/sweep_env.sh NAME "v1 v2 ..." SCALE [GRAPH] ; REPS (default 2)
name=$1; vals=$2; s=$3; graph=${4:-kronecker}
for rep in $(seq ${REPS:-2}); do
  for v in $vals; do
    echo -n "$graph S$s $name=$v "
    env $name=$v python scripts/sweep_params.py --graph $graph --scale $s --roots 16 --L 2048 2>&1 | tail -1
  done
done
