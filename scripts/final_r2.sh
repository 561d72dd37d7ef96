#!/bin/bash
# Closing check of round 2 on the committed tree: the GPU suite, smoke(), the
# driver's bench command and the secondary configuration lines.
R=${R:-r2z}
python -m pytest tests -m gpu -q > gpurun_out/${R}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${R}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${R}_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --scale 22 --no-cpu-baseline > gpurun_out/${R}_s22_selmax.json 2> gpurun_out/${R}_s22.err
python bench.py --graph er --no-cpu-baseline > gpurun_out/${R}_er.json 2> gpurun_out/${R}_er.err
python bench.py --variant tropical --no-cpu-baseline > gpurun_out/${R}_s26_tropical.json 2> gpurun_out/${R}_s26t.err
