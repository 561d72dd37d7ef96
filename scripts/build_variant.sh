#!/bin/bash
# build_variant.sh OUT.so "-DFOO=1 ..." : libslimsell_b200.so with extra defines on bfs.cu (A/B experiments)
set -e
out=$1; shift
defs="$*"
cd "$(dirname "$0")/../paper_2010_09913_b200/csrc"
make -s >/dev/null
tmp=$(mktemp -d)
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I../../include \
  --expt-relaxed-constexpr $defs -c bfs.cu -o $tmp/bfs.o
objs=$(ls build/*.o | grep -v '/bfs.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs $tmp/bfs.o -lcudart
rm -rf $tmp
