set -x
export SSB_LIB=$PWD/build_variants/count.so
python scripts/prof_iter.py --scale 26 --iters 8 --L 2048 > gpurun_out/cnt_s26.txt 2>&1
python scripts/prof_iter.py --scale 26 --graph er --iters 10 --L 2048 --root 30478752 > gpurun_out/cnt_er.txt 2>&1
export SSB_LIB=$PWD/build_variants/iters1.so
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 10 -c 2 -o gpurun_out/s26_k34 python scripts/prof_iter.py --scale 26 --iters 8 --L 2048 > gpurun_out/ncu_s26.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 14 -c 3 -o gpurun_out/er_k567 python scripts/prof_iter.py --scale 26 --graph er --iters 10 --L 2048 --root 30478752 > gpurun_out/ncu_er.log 2>&1
ls -la gpurun_out/
