# per-iteration ncu captures of S26 iteration 3 (one launch per iteration build)
export SSB_LIB=$PWD/build_variants/iters1.so
python scripts/prof_iter.py --scale 26 --iters 8 --L 2048 > gpurun_out/k3_iters.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 9 -c 1 -o gpurun_out/s26_sel_k3 python scripts/prof_iter.py --scale 26 --iters 8 --L 2048 > gpurun_out/ncu_k3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 9 -c 1 -o gpurun_out/s26_trop_k3 python scripts/prof_iter.py --scale 26 --iters 8 --L 2048 --variant 0 > gpurun_out/ncu_k3t.log 2>&1
