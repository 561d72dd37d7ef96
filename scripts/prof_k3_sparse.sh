export SSB_LIB=$PWD/build_variants/iters1.so
python scripts/prof_iter.py --scale 26 --iters 3 --L 2048 --root 22712927 > gpurun_out/k3s_iters.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 5 -c 1 -o gpurun_out/final_k3_sparse python scripts/prof_iter.py --scale 26 --iters 3 --L 2048 --root 22712927 > gpurun_out/ncu_k3s.log 2>&1
