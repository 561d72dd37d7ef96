#!/bin/bash
# Closing check of the round-2 tree (r2u): the GPU suite, smoke(), the
# driver's bench command, the secondary configuration lines and the launch list.
R=${R:-r2u}
python -m pytest tests -m gpu -q > gpurun_out/${R}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${R}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${R}_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --scale 22 --no-cpu-baseline > gpurun_out/${R}_s22_selmax.json 2> gpurun_out/${R}_s22.err
python bench.py --graph er --no-cpu-baseline > gpurun_out/${R}_er.json 2> gpurun_out/${R}_er.err
python bench.py --variant tropical --no-cpu-baseline > gpurun_out/${R}_s26_tropical.json 2> gpurun_out/${R}_s26t.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-validate --e2e-steps 0 > gpurun_out/${R}_ncu_launches.log 2>&1
