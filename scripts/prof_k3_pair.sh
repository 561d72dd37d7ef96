export SSB_LIB=$PWD/build_variants/iters1.so
python scripts/prof_iter.py --scale 26 --iters 3 --L 2048 --root 24490569 > gpurun_out/k3p_iters.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 5 -c 1 -o gpurun_out/r2f_k3_mid python scripts/prof_iter.py --scale 26 --iters 3 --L 2048 --root 24490569 > gpurun_out/ncu_k3p1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 11 -c 1 -o gpurun_out/r2f_k4_direct python scripts/prof_iter.py --scale 26 --iters 8 --L 2048 --root 2564265 > gpurun_out/ncu_k3p2.log 2>&1
