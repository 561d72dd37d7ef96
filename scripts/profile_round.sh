#!/bin/bash
# Round profile on the GPU box: bench (no profiler) -> launch list -> one
# --set full capture of bfs32_kernel on the bench workload. Outputs under
# gpurun_out/; copy the summaries into profiles/.
set -x
R=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_launches.log 2>&1
python scripts/prof_iter.py --iters 100 --L 2048 --root 2564265 > gpurun_out/${R}_prof_iter.txt 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 1 -c 1 -o gpurun_out/${R}_bfs32_full \
    python scripts/prof_iter.py --iters 100 --L 2048 --root 2564265 > gpurun_out/${R}_ncu_full.log 2>&1
tail -n 3 gpurun_out/${R}_ncu_full.log
