#!/bin/bash
# Task budget sweep (SSB_TASK_BUDGET is read when the plan is built, so one
# process per value), 16 Graph500 roots, sel-max.
# env: SCALES (default "22 26"), BUDGETS (default "128 256 512 1024"), GRAPH (kronecker|er), REPS
for rep in $(seq ${REPS:-2}); do
for s in ${SCALES:-22 26}; do
  for b in ${BUDGETS:-128 256 512 1024}; do
    echo -n "${GRAPH:-kronecker} S$s budget=$b "
    SSB_TASK_BUDGET=$b python scripts/sweep_params.py --graph ${GRAPH:-kronecker} --scale $s --roots 16 --L 2048 2>&1 | tail -1
  done
done
done
