#!/usr/bin/env bash
# Build the CUDA library (sm_100a) and the C oracle.  Usage: ./build.sh [-j]
set -euo pipefail
cd "$(dirname "$0")"
PKG=paper_1808_02950_b200
OUT=$PKG/libadct.so
mkdir -p build
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude -I$PKG/csrc --expt-relaxed-constexpr -Xptxas -v"
pids=()
for f in matrix basic fused stream tc sweep blockmajor jam greedy merit; do
  nvcc $FLAGS -c $PKG/csrc/$f.cu -o build/$f.o > build/$f.ptxas.log 2>&1 &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
if [ $rc -ne 0 ]; then cat build/*.ptxas.log | grep -v "^ptxas info" | head -50; exit 1; fi
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT.tmp build/matrix.o build/basic.o build/fused.o build/stream.o build/tc.o build/sweep.o build/blockmajor.o build/jam.o build/greedy.o build/merit.o
mv $OUT.tmp $OUT
gcc -O2 -fopenmp -shared -fPIC -o oracle/liboracle.so oracle/adct_oracle.c -lm
echo "built $OUT"
