#!/bin/bash
# Round-2 measurement on the GPU box: bench lines (no profiler), then the ncu
# launch list of the bench command and one --set full capture of bfs32_kernel.
set -x
R=${1:-r2}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --scale 22 --no-cpu-baseline > gpurun_out/${R}_s22_selmax.json 2> gpurun_out/${R}_s22_selmax.err
python bench.py --scale 22 --variant tropical --no-cpu-baseline > gpurun_out/${R}_s22_tropical.json 2>> gpurun_out/${R}_s22_selmax.err
python bench.py --graph er --no-cpu-baseline > gpurun_out/${R}_er.json 2> gpurun_out/${R}_er.err
python bench.py --variant tropical --no-cpu-baseline > gpurun_out/${R}_s26_tropical.json 2> gpurun_out/${R}_s26_tropical.err
python bench.py --shard chunks --no-cpu-baseline > gpurun_out/${R}_chunks1.json 2> gpurun_out/${R}_chunks1.err
SSB_BENCH_BACKEND=gloo python bench.py --gpus 2 --shard chunks --steps 2 --warmup 1 > gpurun_out/${R}_gloo2_s26.json 2> gpurun_out/${R}_gloo2_s26.err
python scripts/time_spmv.py --scale 22 > gpurun_out/${R}_spmv.jsonl 2>&1
python scripts/time_spmv.py --scale 26 >> gpurun_out/${R}_spmv.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-validate --e2e-steps 0 > gpurun_out/${R}_ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 1 -c 1 -o gpurun_out/${R}_bfs32_full \
    python scripts/prof_iter.py --iters 100 --L 2048 --root 2564265 > gpurun_out/${R}_ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:bfs32 -s 1 -c 1 -o gpurun_out/${R}_bfs32_s22_full \
    python scripts/prof_iter.py --scale 22 --iters 100 --L 2048 --g500 0 > gpurun_out/${R}_ncu_s22.log 2>&1
ncu --set full --clock-control none -k regex:bfs32 -s 1 -c 1 -o gpurun_out/${R}_bfs32_er_full \
    python scripts/prof_iter.py --graph er --iters 100 --L 2048 --g500 0 > gpurun_out/${R}_ncu_er.log 2>&1
